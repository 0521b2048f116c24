#!/usr/bin/env bash
# cell V-cycle time at 512^3 (and 2D 8192^2) vs the coarse-cluster threshold / size
for env in "FASMG_COARSE_MAX=4096" "FASMG_COARSE_MAX=32768" "FASMG_COARSE_MAX=32768 FASMG_COARSE_CS=16" "FASMG_COARSE_MAX=4096 FASMG_COARSE_CS=16" "FASMG_COARSE_MAX=16384"; do
  echo "== $env"
  env $env python scripts/sweep_bench.py 512x3 8192x2 2>&1 | grep -v "^$"
  env $env python scripts/sweep_bench.py 512x3 2>&1 | grep -v "^$"
done
