#!/bin/bash
# r02bf: racecheck / synccheck of the kernels with the host loop
# (FASMG_DEVICE_LOOP=0), and of the bare conditional-WHILE probe to see
# whether the tools handle device-side cudaGraphSetConditional at all.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bf; mkdir -p $O
for tool in racecheck synccheck memcheck; do
  timeout 300 compute-sanitizer --tool $tool scripts/micro/cond_probe > $O/san_${tool}_condprobe.log 2>&1
  echo "rc=$?" >> $O/san_${tool}_condprobe.log
done
for tool in racecheck synccheck; do
  for case in tma edge; do
    FASMG_DEVICE_LOOP=0 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py $case > $O/san_${tool}_${case}.log 2>&1
    echo "rc=$?" >> $O/san_${tool}_${case}.log
  done
done
