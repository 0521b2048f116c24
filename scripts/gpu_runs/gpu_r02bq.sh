cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bq; mkdir -p $O
timeout 1800 python -m pytest tests/test_slab_gpu.py tests/test_ns_slab_gpu.py tests/test_solve_loop_gpu.py -q 2>&1 | tail -6 > $O/tests.log
