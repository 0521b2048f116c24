#!/bin/bash
# r02be: compute-sanitizer over the fused edge correction and the device
# solve loop (sanitize_cases.py solves through FasSolver.solve: the
# conditional-WHILE graph), plus the 2D and NS cases.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02be; mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  for case in tma edge; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py $case > $O/san_${tool}_${case}.log 2>&1
    echo "rc=$?" >> $O/san_${tool}_${case}.log
  done
done
for case in d2 ns; do
  timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py $case > $O/san_memcheck_${case}.log 2>&1
  echo "rc=$?" >> $O/san_memcheck_${case}.log
done
