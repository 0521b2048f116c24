"""Compare fused (FASMG_FUSE bits) vs unfused engines on one V-cycle: field
differences per level/class and the residual sum."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P

def run(fuse, n, cycles, with_norm):
    os.environ["FASMG_FUSE"] = str(fuse)
    os.environ["FASMG_TMA_MIN"] = "0"
    g = P.unit_grid((n,) * 3)
    rng = np.random.default_rng(5)
    p0 = np.zeros((n + 2,) * 3); p0[1:-1, 1:-1, 1:-1] = rng.standard_normal((n,) * 3)
    f0 = np.zeros((n + 2,) * 3); f0[1:-1, 1:-1, 1:-1] = rng.standard_normal((n,) * 3)
    p = P.Field(g, P.Location.CELL, 1, p0); f = P.Field(g, P.Location.CELL, 1, f0)
    S = P.FasSolver(P.make_hierarchy(g, 3), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                    P.make_plan("x", 3), P.OperatorCoeffs(1.0, 0.5))
    e = S.engine(2, p.device); e.load(p, f)
    ss = e.run(cycles, with_norm, use_graph=False)
    out = []
    from paper_2510_11152_b200 import _native as N
    import ctypes
    for k in range(4):
        geo = (ctypes.c_long * 9)()
        N.lib().fasmg_engine_level_geom(e.handle, k, geo)
        tot = geo[0] * 8
        buf = torch.empty(tot, dtype=torch.float64, device="cuda")
        N.lib().fasmg_engine_level_copy(e.handle, k, 0, ctypes.c_void_p(buf.data_ptr()))
        out.append(buf.cpu().numpy().reshape(8, -1))
    return ss, out

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for fuse, wn in ((1, False), (2, True), (3, True)):
    a = run(0, n, 1, wn)
    b = run(fuse, n, 1, wn)
    print(f"fuse={fuse} norm: {a[0]!r} vs {b[0]!r}")
    for k in range(4):
        d = np.abs(a[1][k] - b[1][k])
        bad = [(c, int((d[c] > 0).sum())) for c in range(8) if (d[c] > 0).any()]
        print(f"  level {k}: classes differing {bad}")
