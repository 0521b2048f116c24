#!/bin/bash
# r02c: validate the slab NS stepper, probe the 8-virtual-rank hang with more
# hardware queues, run compute-sanitizer over the core kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests/test_ns_slab_gpu.py -x -q 2>&1 | tail -30 > $O/ns_slab_tests.log
for c in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 120 python scripts/virtual_slab_repro.py 512 8 > $O/vrepro_conn$c.log 2>&1
  echo "rc=$?" >> $O/vrepro_conn$c.log
done
for tool in memcheck racecheck synccheck initcheck; do
  for case in tma edge d2 ns; do
    timeout 400 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py $case > $O/san_${tool}_${case}.log 2>&1
    echo "rc=$?" >> $O/san_${tool}_${case}.log
  done
done
for tool in memcheck synccheck; do
  SELFTEST_N=64 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29655 --no-python \
    compute-sanitizer --tool $tool --print-limit 20 python scripts/dist_selftest.py > $O/san_${tool}_dist2.log 2>&1
  echo "rc=$?" >> $O/san_${tool}_dist2.log
done
SELFTEST_N=64 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29656 scripts/dist_selftest.py > $O/dist4.log 2>&1; echo "rc=$?" >> $O/dist4.log
