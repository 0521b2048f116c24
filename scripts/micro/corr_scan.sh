#!/usr/bin/env bash
# 512^3 V-cycle time vs the corrected half-sweep's chunk and the coarse cluster size
for env in "FASMG_CORR_CHUNK=4" "FASMG_CORR_CHUNK=8" "FASMG_CORR_CHUNK=2" "FASMG_COARSE_CS=16" "FASMG_CORR_CHUNK=4"; do
  echo "== $env"
  for r in 1 2; do env $env python scripts/sweep_bench.py 512x3 2>&1 | grep -v "^$"; done
done
