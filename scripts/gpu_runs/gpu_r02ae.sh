cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ae; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_ns_gpu.py tests/test_slab_cpu.py tests/test_batch_gpu.py tests/test_ns_slab_gpu.py -q -x 2>&1 | tail -2 > $O/tests.log
timeout 600 python scripts/ns_prof.py 512 2 2 > $O/nsprof.txt 2>&1
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
