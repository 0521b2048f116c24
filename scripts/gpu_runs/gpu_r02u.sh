cd $GRAFT_REPO_ROOT
O=gpurun_out/r02u; mkdir -p $O
timeout 1200 python -m pytest tests/test_ns_gpu.py tests/test_arena_gpu.py tests/test_wave_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -4 > $O/tests.log
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
timeout 1500 python bench.py --workload ns1024 --steps 2 --warmup 3 --no-cpu-baseline > $O/ns1024.json 2> $O/ns1024.err
