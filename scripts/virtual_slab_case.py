"""One VirtualSlabSolver solve vs the single-engine solve (bitwise):
    python scripts/virtual_slab_case.py N PARTS BC(dirichlet|neumann) LOC [k_max]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.slab import VirtualSlabSolver
n, parts, bcn, loc = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
kmax = int(sys.argv[5]) if len(sys.argv) > 5 else 3
L = getattr(P.Location, loc.upper())
g = P.unit_grid((n,) * 3)
ml = int(np.log2(n)) - 1
torch.manual_seed(0)
p0 = P.Field(g, L); f0 = P.Field(g, L)
p0.interior = torch.rand(p0.interior.shape, dtype=torch.float64, device="cuda")
f0.interior = torch.rand(f0.interior.shape, dtype=torch.float64, device="cuda")
bc = P.BoundaryCondition.neumann(3) if bcn == "neumann" else P.BoundaryCondition.dirichlet(3)
co = P.OperatorCoeffs(0.0 if bcn == "neumann" else 1.0, 1.0)
args = (P.make_hierarchy(g, ml), L, bc, P.make_plan("x", 3), co)
prm = P.FasParams(1e-30, kmax, 2, ml)
outs = []
for k in (1, parts):
    p = P.Field(g, L); f = P.Field(g, L)
    p.data.copy_(p0.data); f.data.copy_(f0.data)
    t0 = time.time()
    rep = (P.FasSolver(*args) if k == 1 else VirtualSlabSolver(*args, parts)).solve(p, f, prm)
    torch.cuda.synchronize()
    print(f"parts {k}: {rep.iterations} cycles {time.time() - t0:.2f}s last {rep.residual_history[-1]:.6e}",
          flush=True)
    outs.append(p.data.clone())
print("bitwise", torch.equal(outs[0], outs[1]), flush=True)
