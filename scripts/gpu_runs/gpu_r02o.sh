cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -k edge_tau 2>&1 | tail -30 > $O/tests.log
timeout 300 python scripts/vcycle_prof.py 512 ns 5 $O/prof_ns.json > $O/prof_ns.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 tb 5 $O/prof_tb.json > $O/prof_tb.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 ew 5 $O/prof_ew.json > $O/prof_ew.txt 2>&1
