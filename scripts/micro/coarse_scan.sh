#!/usr/bin/env bash
# edge/cell V-cycle times at 512^3 vs the coarse-cluster knobs
for env in "FASMG_COARSE_MAX=0" "FASMG_COARSE_MAX=64" "FASMG_COARSE_MAX=512" "FASMG_COARSE_MAX=4096" "FASMG_COARSE_CS=16" "FASMG_COARSE_MAX=512 FASMG_COARSE_CS=4"; do
  echo "== $env"
  env $env python scripts/edge_perf.py 512 2>&1 | grep -v "^$"
done
