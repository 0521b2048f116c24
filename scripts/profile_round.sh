#!/usr/bin/env bash
# Run on the GPU box (via gpurun): tests, bench, ncu launch list and a full
# ncu capture of the finest half-sweep.  Outputs under gpurun_out/$TAG*.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1
tail -3 gpurun_out/${TAG}_gpu_tests.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json | head -c 600; echo
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_smem -s 2 -c 1 \
    -o gpurun_out/${TAG}_sweep python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_tau_fast -s 0 -c 1 \
    -o gpurun_out/${TAG}_tau python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ls -la gpurun_out/ | grep ${TAG}
