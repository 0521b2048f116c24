cd $GRAFT_REPO_ROOT
O=gpurun_out/r02n; mkdir -p $O
timeout 300 python bench.py --workload ns --grid 64 --gpus 2 --steps 2 --warmup 3 > $O/ns64_g2.json 2> $O/ns64_g2.err
timeout 300 python bench.py --workload ns --grid 64 --gpus 4 --steps 2 --warmup 3 > $O/ns64_g4.json 2> $O/ns64_g4.err
timeout 1200 python -m pytest tests/test_ns_gpu.py tests/test_arena_gpu.py tests/test_ns_slab_gpu.py -q -x 2>&1 | tail -4 > $O/ns_tests.log
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
