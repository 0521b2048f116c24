"""Virtual-rank slab decomposition on ONE GPU: P slab engines on P streams
running the multi-GPU protocol (halo push per half-sweep, coarse gather,
rank-ordered norm).  The wall time per V-cycle vs the single engine bounds
the exchange + synchronization overhead the real 1..8-GPU runs carry
(the slabs share this GPU's SMs and HBM, so it is NOT a scaling number).
Usage: python scripts/virtual_slab_perf.py N P [P ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.slab import VirtualSlabSolver

n = int(sys.argv[1])
g = P.unit_grid((n,) * 3)
ml = int(np.log2(n)) - 1
bc = P.BoundaryCondition.dirichlet(3)
plan = P.make_plan("x", 3)
co = P.OperatorCoeffs(1.0, 1.0)
p = P.Field(g, P.Location.CELL); f = P.Field(g, P.Location.CELL)
p.interior = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
f.interior = torch.rand(f.interior.shape, dtype=torch.float64, device="cuda")
for parts in [int(x) for x in sys.argv[2:]]:
    if parts == 1:
        S = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, co)
        e = S.engine(2, p.device); e.load(p, f); e.run(3, True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e.run(10, True)
        torch.cuda.synchronize(); ms = (time.perf_counter() - t0) / 10 * 1e3
        print(f"{n}^3 single engine: {ms:.3f} ms/V-cycle (+norm)", flush=True)
        continue
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, co, parts)
    es = vs.engines(2, p.device)
    vs._load(es, p, f)
    for _ in range(3):
        vs.launch_all(es, 1, True)
        for e in es: e.result()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10):
        vs.launch_all(es, 1, True)
        for e in es: e.result()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    print(f"{n}^3 {parts} virtual ranks on one GPU: {ms:.3f} ms/V-cycle (+norm)", flush=True)
