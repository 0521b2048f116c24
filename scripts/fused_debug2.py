"""Per-point check of the fused residual (FASMG_FUSE_DEBUG) against the
engine's own unfused residual recomputed on the host from the blocked P/F."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["FASMG_FUSE"] = "2"; os.environ["FASMG_TMA_MIN"] = "0"; os.environ["FASMG_FUSE_DEBUG"] = "1"
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = P.unit_grid((n,) * 3)
rng = np.random.default_rng(5)
p0 = np.zeros((n + 2,) * 3); p0[1:-1, 1:-1, 1:-1] = rng.standard_normal((n,) * 3)
f0 = np.zeros((n + 2,) * 3); f0[1:-1, 1:-1, 1:-1] = rng.standard_normal((n,) * 3)
p = P.Field(g, P.Location.CELL, 1, p0); f = P.Field(g, P.Location.CELL, 1, f0)
S = P.FasSolver(P.make_hierarchy(g, 3), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                P.make_plan("x", 3), P.OperatorCoeffs(1.0, 0.5))
e = S.engine(2, p.device); e.load(p, f)
ss = e.run(1, True, use_graph=False)
geo = (ctypes.c_long * 9)(); N.lib().fasmg_engine_level_geom(e.handle, 0, geo)
cls, s0, s1, E0, E1, E2 = geo[0], geo[1], geo[2], geo[3], geo[4], geo[5]
def get(which):
    buf = torch.empty(cls * 8, dtype=torch.float64, device="cuda")
    assert N.lib().fasmg_engine_level_copy(e.handle, 0, which, ctypes.c_void_p(buf.data_ptr())) == 0
    return buf.cpu().numpy()
Pb, Fb, Rb = get(0), get(1), get(2)
B = n // 2; OFF = 3
h = 1.0 / n; inv_h2 = 1.0 / (h * h); a, b = 1.0, 0.5
def at(c, b0, b1, b2): return c * cls + b0 * s0 + b1 * s1 + b2 + OFF
bad = 0; tot = 0.0
for c in range(8):
    q = [(c >> 2) & 1, (c >> 1) & 1, c & 1]
    b0, b1, b2 = np.meshgrid(np.arange(1, B + 1), np.arange(1, B + 1), np.arange(1, B + 1), indexing="ij")
    o = at(c, b0, b1, b2)
    pc = Pb[o]
    ns = None
    for ax in range(3):
        bit = 1 << (2 - ax)
        d = [0, 0, 0]
        dcls = ((c ^ bit) - c) * cls
        sa = [s0, s1, 1][ax]
        e_ = Pb[o + dcls + (0 if q[ax] else sa)]
        w_ = Pb[o + dcls - (sa if q[ax] else 0)]
        ns = (e_ + w_) if ns is None else ((ns + e_) + w_)
    lap = (ns - 6.0 * pc) * inv_h2
    r = Fb[o] - (a * pc - b * lap)
    got = Rb[o]
    diff = got != r
    tot += float((r * r).sum())
    if diff.any():
        idx = np.argwhere(diff)
        bad += len(idx)
        pl = idx[idx[:, 0] == idx[0, 0]] + 1
        print("  class", c, "plane", int(pl[0, 0]), "coords(b1,b2):", pl[:, 1:].tolist()[:70])
        print("class", c, "bad", len(idx), "planes", sorted(set((idx[:, 0] + 1).tolist())),
              "b1", sorted(set((idx[:, 1] + 1).tolist()))[:40], "b2", sorted(set((idx[:, 2] + 1).tolist()))[:40])
print("bad points", bad, "host sumsq", tot, "engine", ss)
