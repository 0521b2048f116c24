cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bl; mkdir -p $O
timeout 1200 python -m pytest tests/test_wave_gpu.py tests/test_gpu_parity.py tests/test_solve_loop_gpu.py -q -x 2>&1 | tail -3 > $O/tests.log
for l in ew cell; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_$l.txt 2>&1; done
