import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np, torch
import cases as C
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.slab import VirtualSlabSolver

def run(n, dim, parts, minpl, ml=None, kmax=1):
    shape = (n,) * dim
    ml = ml or int(np.log2(n)) - 1
    bc = P.BoundaryCondition.dirichlet(dim)
    p0 = C.rand_field(21, shape, "cell", 1); f0 = C.rand_field(22, shape, "cell", 1)
    g = P.unit_grid(shape); coeffs = P.OperatorCoeffs(1.0, 0.5); plan = P.make_plan("x", dim)
    params = P.FasParams(1e-30, kmax, 2, ml)
    p1 = P.Field(g, P.Location.CELL, 1, p0.copy()); f1 = P.Field(g, P.Location.CELL, 1, f0.copy())
    r1 = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs).solve(p1, f1, params)
    p2 = P.Field(g, P.Location.CELL, 1, p0.copy()); f2 = P.Field(g, P.Location.CELL, 1, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs, parts, min_planes=minpl)
    es = vs.engines(2, p2.device)
    r2 = vs.solve(p2, f2, params)
    d = (p1.data - p2.data).abs()
    # per-slab max error along axis 0
    per = d.amax(dim=tuple(range(1, dim))).cpu().numpy()
    bad = np.nonzero(per)[0]
    print(f"n={n} dim={dim} P={parts} minpl={minpl} ml={ml} kg={es[0].kg}: maxdiff {float(d.max()):.3e} "
          f"hist {r1.residual_history[-1]:.6e} vs {r2.residual_history[-1]:.6e} bad planes {bad[:8]}..{bad[-4:] if len(bad) else ''}", flush=True)

for cfg in [(64,3,2,4), (64,3,4,4), (64,3,4,8), (64,3,4,16), (128,3,4,16), (128,3,4,4), (32,2,4,4), (64,3,4,8,1), (64,3,2,4,1)]:
    n, dim, parts, minpl = cfg[:4]
    ml = cfg[4] if len(cfg) > 4 else None
    try:
        run(n, dim, parts, minpl, ml)
    except Exception as e:
        print(cfg, "ERROR", e)
