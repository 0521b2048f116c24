import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np, torch
import cases as C
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N
from paper_2510_11152_b200.slab import VirtualSlabSolver

def level(h, k, which, dim):
    g = (ctypes.c_long * 9)()
    N.call("fasmg_engine_level_geom", h, k, g)
    cls, s0, s1, E0, E1, E2, B0, off0, G0 = list(g)
    nc = 1 << dim
    t = torch.empty(cls * nc, dtype=torch.float64, device="cuda")
    N.call("fasmg_engine_level_copy", h, k, which, N.ptr(t))
    torch.cuda.synchronize()
    a = t.cpu().numpy().reshape(nc, cls)
    if dim == 3:
        a = a[:, :E0 * s0].reshape(nc, E0, E1, s1)[:, :, :, 3:3 + E2]
    else:
        a = a[:, :E0 * s0].reshape(nc, E0, s0)[:, :, 3:3 + E1]
    return a, B0, off0

def main(n, dim, parts, minpl, ml, kmax=1):
    shape = (n,) * dim
    bc = P.BoundaryCondition.dirichlet(dim)
    p0 = C.rand_field(21, shape, "cell", 1); f0 = C.rand_field(22, shape, "cell", 1)
    g = P.unit_grid(shape); coeffs = P.OperatorCoeffs(1.0, 0.5); plan = P.make_plan("x", dim)
    params = P.FasParams(1e-30, kmax, 2, ml)
    S = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs)
    p1 = P.Field(g, P.Location.CELL, 1, p0.copy()); f1 = P.Field(g, P.Location.CELL, 1, f0.copy())
    S.solve(p1, f1, params)
    e1 = S.engine(2, p1.device)
    p2 = P.Field(g, P.Location.CELL, 1, p0.copy()); f2 = P.Field(g, P.Location.CELL, 1, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs, parts, min_planes=minpl)
    es = vs.engines(2, p2.device)
    vs.solve(p2, f2, params)
    print(f"n={n} P={parts} ml={ml} kg={es[0].kg} field maxdiff {float((p1.data-p2.data).abs().max()):.3e}")
    for k in range(ml + 1):
        for which in (0, 1):
            ref, B0g, _ = level(e1.handle, k, which, dim)
            msg = []
            for e in es:
                loc, B0, off0 = level(e.handle, k, which, dim)
                if B0 == B0g:  # replicated
                    d = np.abs(loc[:, 1:B0 + 1] - ref[:, 1:B0 + 1]).max()
                else:
                    d = np.abs(loc[:, 1:B0 + 1] - ref[:, off0 + 1:off0 + B0 + 1]).max()
                msg.append(f"r{e.rank}:{d:.1e}")
                if d > 1e-3 and k == 1 and which == 1 and B0 != B0g:
                    dd = np.abs(loc[:, 1:B0 + 1] - ref[:, off0 + 1:off0 + B0 + 1])
                    print("    rank", e.rank, "per plane", dd.max(axis=(0, 2, 3)), "per class", dd.max(axis=(1, 2, 3)))
                    idx = np.argwhere(dd > 1e-3)[:6]
                    print("    first bad (class, plane, b1, b2):", idx.tolist())
            print(f"  level {k} {'PF'[which]}: " + " ".join(msg))

main(64, 3, 4, 4, 2)
main(128, 3, 4, 4, 2)
main(128, 3, 8, 4, 2)
