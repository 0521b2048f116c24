"""V-cycle time of an edge-centred field at N^3 (the NS momentum solves) vs
the cell-centred one.  Usage: python scripts/edge_perf.py N"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.unit_grid((n,) * 3)
ml = int(np.log2(n)) - 1
for loc in (P.Location.CELL, P.Location.EDGE_EW, P.Location.EDGE_NS, P.Location.EDGE_TB):
    p = P.Field(g, loc); f = P.Field(g, loc)
    p.interior = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
    f.interior = torch.rand(f.interior.shape, dtype=torch.float64, device="cuda")
    S = P.FasSolver(P.make_hierarchy(g, ml), loc, P.BoundaryCondition.dirichlet(3),
                    P.make_plan("x", 3), P.OperatorCoeffs(1.0, 0.05))
    e = S.engine(2, p.device); e.load(p, f); e.run(3, True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e.run(10, True); torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    print(f"{loc.name:8s} {n}^3: {ms:.3f} ms/V-cycle, kernels/cycle {e.kernels_per_vcycle()}", flush=True)
    del e, S, p, f
    torch.cuda.empty_cache()
