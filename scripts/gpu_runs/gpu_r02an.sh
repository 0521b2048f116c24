cd $GRAFT_REPO_ROOT
O=gpurun_out/r02an; mkdir -p $O
timeout 900 python -m pytest tests/test_solve_loop_gpu.py tests/test_wave_gpu.py -q -x 2>&1 | tail -15 > $O/tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-numba-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ns_gpu.py tests/test_heat_gpu.py tests/test_cli_gpu.py tests/test_batch_gpu.py tests/test_fuzz_gpu.py -q -x 2>&1 | tail -5 > $O/tests2.log
