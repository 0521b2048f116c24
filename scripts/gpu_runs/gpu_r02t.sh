cd $GRAFT_REPO_ROOT
O=gpurun_out/r02t; mkdir -p $O
timeout 1700 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -8 > $O/gpu_tests.log
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
