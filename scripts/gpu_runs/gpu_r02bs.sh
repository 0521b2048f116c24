cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bs; mkdir -p $O
timeout 1200 python -m pytest tests/test_solve_loop_gpu.py tests/test_slab_gpu.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
