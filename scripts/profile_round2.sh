#!/usr/bin/env bash
# Round-2 GPU validation + profiles (run via gpurun): GPU tests, smoke, bench
# (heat, reference arm, NS 512^3), the ncu launch list of one eager cell and
# edge V-cycle, and full captures of the finest sweep, tau, corrected sweep
# and edge tau.  Outputs under gpurun_out/$TAG*.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1
tail -3 gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --workload ns512 --steps 5 --warmup 3 > gpurun_out/${TAG}_ns512.json 2>> gpurun_out/${TAG}_bench.err
head -c 300 gpurun_out/${TAG}_bench.json; echo
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}edge_launches.csv \
    python scripts/profile_vcycle.py 512 3 1 edge_ns > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 2 -c 1 \
    -o gpurun_out/${TAG}_sweep python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resid_tma -s 0 -c 1 \
    -o gpurun_out/${TAG}_tau python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 24 -c 1 \
    -o gpurun_out/${TAG}_corr python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resid_tma -s 2 -c 1 \
    -o gpurun_out/${TAG}_spec python scripts/profile_vcycle.py 512 3 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tau_edge -s 0 -c 1 \
    -o gpurun_out/${TAG}_etau python scripts/profile_vcycle.py 512 3 1 edge_ns > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 24 -c 1 \
    -o gpurun_out/${TAG}_ecorr python scripts/profile_vcycle.py 512 3 1 edge_ns > /dev/null 2>&1
# summaries on the box (the .ncu-rep captures exceed gpurun's copy-back cap)
mkdir -p gpurun_out/${TAG}_prof
PROF_OUT=gpurun_out/${TAG}_prof python scripts/summarize_profiles.py ${TAG}edge > /dev/null 2>&1
mv gpurun_out/${TAG}_prof/ncu_sweep_traffic.json gpurun_out/${TAG}_prof/ncu_sweep_traffic_edge.json 2>/dev/null
PROF_OUT=gpurun_out/${TAG}_prof python scripts/summarize_profiles.py ${TAG} > /dev/null 2>&1
for k in sweep tau corr etau spec ecorr; do
  ncu -i gpurun_out/${TAG}_${k}.ncu-rep --page details --csv > gpurun_out/${TAG}_prof/${k}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${k}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_prof/${k}_source.csv 2>/dev/null
done
gzip -f gpurun_out/${TAG}_prof/*_source.csv
rm -f gpurun_out/${TAG}_*.ncu-rep
ls -la gpurun_out/ gpurun_out/${TAG}_prof | head -40
