"""One weno3_convect of each target component at N^3 (halo-2 random winds),
for ncu: python scripts/weno_prof.py N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.ns import LOC_OF
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.unit_grid((n,) * 3)
vel = []
for c in ("u", "v", "w"):
    F = P.Field(g, LOC_OF[c], 2)
    F.data.copy_(torch.rand(F.data.shape, dtype=torch.float64, device="cuda") - 0.5)
    F.ghosts_fresh = True
    vel.append(F)
for t in range(3):
    out = P.weno3_convect(tuple(vel), t)
torch.cuda.synchronize()
print("done")
if len(sys.argv) > 2:  # timing mode
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for t in range(3):
        P.weno3_convect(tuple(vel), t, out=out)
        st.record()
        for _ in range(5):
            P.weno3_convect(tuple(vel), t, out=out)
        en.record(); torch.cuda.synchronize()
        print(f"target {t}: {st.elapsed_time(en) / 5:.3f} ms per weno3_convect at {n}^3")
