cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bn; mkdir -p $O
timeout 900 python -m pytest tests/test_solve_loop_gpu.py tests/test_ns_gpu.py -q -x 2>&1 | tail -3 > $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
