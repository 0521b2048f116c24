#!/usr/bin/env bash
# V-cycle and per-level half-sweep times at 512^3 under march/corr chunk knobs
for env in "" "FASMG_CORR_CHUNK=2" "FASMG_CORR_CHUNK=8" "FASMG_CORR_CHUNK=16" "FASMG_MARCH_CHUNK=2" "FASMG_MARCH_CHUNK=8"; do
  echo "== $env"
  env $env python - <<'PY'
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N
n = 512
g = P.unit_grid((n,) * 3)
p = P.Field(g, P.Location.CELL); f = P.Field(g, P.Location.CELL)
p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device='cuda')
f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device='cuda')
S = P.FasSolver(P.make_hierarchy(g, 8), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                P.make_plan('x', 3), P.OperatorCoeffs(1.0, 1.0))
e = S.engine(2, p.device); e.load(p, f)
out = []
for k in (0, 1, 2):
    e.time_sweeps(k, 4)
    out.append(e.time_sweeps(k, 40) * 1e3)
e.run(3, True)
st = torch.cuda.ExternalStream(e.stream.value)
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record(st); e.run(20, True); b.record(st); torch.cuda.synchronize()
print("sweep us L0 %.1f L1 %.1f L2 %.1f | cycle %.3f ms" % (*out, a.elapsed_time(b) / 20), flush=True)
PY
done
