cd $GRAFT_REPO_ROOT
O=gpurun_out/r02r; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -k edge_tau 2>&1 | tail -3 > $O/tests.log
for l in ns ew tb; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_${l}.txt 2>&1; done
