cd $GRAFT_REPO_ROOT
O=gpurun_out/r02y; mkdir -p $O
timeout 600 python bench.py --gpus 8 --grid 128 --steps 2 --warmup 3 --no-cpu-baseline --no-numba-baseline > $O/heat_g8.json 2> $O/heat_g8.err; echo "rc=$?" >> $O/heat_g8.err
timeout 900 python bench.py --workload ns --grid 64 --gpus 8 --steps 2 --warmup 3 > $O/ns_g8.json 2> $O/ns_g8.err; echo "rc=$?" >> $O/ns_g8.err
