cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bp; mkdir -p $O
timeout 1500 python -m pytest tests/test_slab_gpu.py tests/test_ns_slab_gpu.py -q -x 2>&1 | tail -25 > $O/tests.log
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_g2.json 2> $O/bench_g2.err; echo "rc=$?" >> $O/bench_g2.err
