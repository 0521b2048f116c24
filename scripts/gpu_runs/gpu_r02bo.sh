cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bo; mkdir -p $O
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_g2.json 2> $O/bench_g2.err; echo "rc=$?" >> $O/bench_g2.err
