cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -k edge_tau 2>&1 | tail -3 > $O/tests.log
for l in ns ew; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 $O/prof_$l.json > $O/prof_$l.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tau_edge -s 0 -c 1 -o $O/etau_ns python scripts/profile_vcycle.py 512 3 1 edge_ns > $O/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tau_edge -s 0 -c 1 -o $O/etau_ew python scripts/profile_vcycle.py 512 3 1 edge_ew > $O/ncu2.log 2>&1
