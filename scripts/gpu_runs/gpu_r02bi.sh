cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bi; mkdir -p $O
timeout 900 python -m pytest tests/test_solve_loop_gpu.py -q 2>&1 | tail -15 > $O/tests.log
