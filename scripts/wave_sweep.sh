#!/usr/bin/env bash
# Launch-list timing of the wavefront smoothing kernel for a few configs
# (run on the GPU box).  Usage: scripts/wave_sweep.sh TAG "T K LAG MIN" ...
TAG=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  out=gpurun_out/${TAG}_T$1_K$2_L$3_M$4.csv
  FASMG_WAVE_T=$1 FASMG_WAVE_K=$2 FASMG_WAVE_LAG=$3 FASMG_WAVE_MIN=$4 \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_smooth_wave|k_sweep" --csv --log-file $out python scripts/profile_vcycle.py 512 3 1 > /dev/null 2>&1
  echo "T=$1 K=$2 LAG=$3 MIN=$4"
  FASMG_WAVE_T=$1 FASMG_WAVE_K=$2 FASMG_WAVE_LAG=$3 FASMG_WAVE_MIN=$4 timeout 120 python scripts/probe_perf.py 512x3
done
