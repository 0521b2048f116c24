cd $GRAFT_REPO_ROOT
O=gpurun_out/r02af; mkdir -p $O
timeout 1700 python -m pytest tests/test_ns_gpu.py tests/test_ns_slab_gpu.py tests/test_heat_gpu.py tests/test_cli_gpu.py -q -x 2>&1 | tail -2 > $O/tests.log
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
