cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aj; mkdir -p $O
timeout 2400 python bench.py --workload ns512 --gpus 8 --steps 1 --warmup 3 > $O/ns512_g8.json 2> $O/ns512_g8.err; echo "rc=$?" >> $O/ns512_g8.err
