#!/usr/bin/env bash
# V-cycle+norm times (cell and edge) under FASMG_NORM_SMEM (CTAs/SM of the norm march)
for v in 0 58000 76000; do
  echo "== FASMG_NORM_SMEM=$v"
  FASMG_NORM_SMEM=$v python scripts/edge_perf.py 512 2>&1 | grep -v "^$"
done
