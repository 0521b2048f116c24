"""Trace one wavefront smoothing launch at 512^3 and summarize the latency
of each stage of an item and of each dependency hop (GPU box)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.unit_grid((n,) * 3)
p = P.Field(g, P.Location.CELL); f = P.Field(g, P.Location.CELL)
p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device="cuda")
S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), P.Location.CELL,
                P.BoundaryCondition.dirichlet(3), P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0))
e = S.engine(2, p.device); e.load(p, f); e.run(1, True)
lib = N.lib()
fn = lib.fasmg_engine_wave_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_long, ctypes.POINTER(ctypes.c_long)]
B = n // 2; T = int(os.environ.get("FASMG_WAVE_T", "4")); nt = (B // 32) * (B // 8)
cap = 6 * T * B * nt
buf = np.zeros(cap, dtype=np.uint64); cnt = ctypes.c_long()
for rep in range(2):
    st = fn(e.handle, 0, buf.ctypes.data, cap, ctypes.byref(cnt))
    assert st == 0, lib.fasmg_last_error()
tr = buf.reshape(T, B, nt, 6).astype(np.int64)
t0 = tr[..., 0].min()
tr = tr - t0
tot = tr[..., 5].max() / 1e3
print(f"T={T} launch span {tot:.1f} us, items {cnt.value}")
names = ["poll->deps", "deps->tma issued", "issued->landed", "landed->computed", "computed->published"]
for i, nm in enumerate(names):
    d = (tr[..., i + 1] - tr[..., i]) / 1e3
    print(f"  {nm:22s} mean {d.mean():7.3f} us  p50 {np.median(d):7.3f}  p90 {np.percentile(d, 90):7.3f}")
# hop: deps met of (t,b) minus max publish of (t-1, b-1..b+1)
pub = tr[..., 5].max(axis=2)  # per (t, b): last tile published
hops = []
for t in range(1, T):
    for b in range(B):
        lo, hi = max(0, b - 1), min(B - 1, b + 1)
        ready = pub[t - 1, lo:hi + 1].max()
        hops.append((tr[t, b, :, 1].min() - ready) / 1e3)
hops = np.array(hops)
print(f"  detect (deps met - last dep published) mean {hops.mean():.3f} us p50 {np.median(hops):.3f}")
# per-wave span: plane completion spread
spread = (tr[..., 5].max(axis=2) - tr[..., 5].min(axis=2)) / 1e3
print(f"  plane publish spread (first->last tile) mean {spread.mean():.2f} us")
first = tr[..., 3].min(axis=2); last = tr[..., 5].max(axis=2)
print(f"  plane life (first landed -> last published) mean {((last-first)/1e3).mean():.2f} us")
print(f"  per-wave period {tot / (B + 2 * (T - 1)):.2f} us")
