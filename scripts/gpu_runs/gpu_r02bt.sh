cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bt; mkdir -p $O
timeout 900 python bench.py --workload ns --grid 64 --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ns64_g2.json 2> $O/ns64_g2.err; echo "rc=$?" >> $O/ns64_g2.err
timeout 900 python bench.py --workload ns --grid 64 --steps 2 --warmup 3 --no-cpu-baseline > $O/ns64_g1.json 2> $O/ns64_g1.err; echo "rc=$?" >> $O/ns64_g1.err
