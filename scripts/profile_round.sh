#!/usr/bin/env bash
# Run on the GPU box (via gpurun): tests, smoke, bench, ncu launch list and a
# full ncu capture of the finest half-sweep.  Outputs under gpurun_out/$TAG*.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1
tail -3 gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2>> gpurun_out/${TAG}_bench.err
head -c 400 gpurun_out/${TAG}_bench.json; echo
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 2 -c 1 \
    -o gpurun_out/${TAG}_sweep python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_resid_tma -s 0 -c 1 \
    -o gpurun_out/${TAG}_tau python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ls -la gpurun_out/ | grep ${TAG}
