#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bg; mkdir -p $O
for tool in synccheck racecheck; do
  for case in tma edge; do
    timeout 600 compute-sanitizer --tool $tool --num-cuda-barriers 4 --print-limit 20 python scripts/sanitize_cases.py $case > $O/san_${tool}_${case}_dl.log 2>&1
    echo "rc=$?" >> $O/san_${tool}_${case}_dl.log
  done
done
