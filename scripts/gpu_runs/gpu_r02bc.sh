cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bc; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py tests/test_solve_loop_gpu.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $O/tests.log
for l in cell ew; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_$l.txt 2>&1; done
