cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ai; mkdir -p $O
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > $O/mem.txt
timeout 2400 python bench.py --workload ns1024 --gpus 8 --steps 1 --warmup 3 > $O/ns1024_g8.json 2> $O/ns1024_g8.err; echo "rc=$?" >> $O/ns1024_g8.err
