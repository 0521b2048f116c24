"""Multi-process slab solve (one process per "GPU"; all may share one device):
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/dist_selftest.py
Each rank compares its slab of the solution with a single-engine solve of
the same problem (bitwise) and prints one line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np, torch
import torch.distributed as dist
import cases as C
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.slab import DistSlabSolver, slab_view

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ndev = torch.cuda.device_count()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % ndev)
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
n = int(os.environ.get("SELFTEST_N", "64"))
loc = os.environ.get("SELFTEST_LOC", "cell")          # cell | edge_ew | edge_ns | edge_tb
LOC = getattr(P.Location, loc.upper())
ea = LOC.edge_axis
dim = 3
shape = (n,) * dim
ml = int(np.log2(n)) - 1
p0 = C.rand_field(21, shape, loc, 1)
f0 = C.rand_field(22, shape, loc, 1)
g = P.unit_grid(shape)
singular = os.environ.get("SELFTEST_BC", "dirichlet") == "neumann"  # pressure-like: a=0
bc = P.BoundaryCondition.neumann(dim) if singular else P.BoundaryCondition.dirichlet(dim)
coeffs = P.OperatorCoeffs(0.0 if singular else 1.0, 0.5 if ea is None else 0.05)
plan = P.make_plan("x", dim)
params = P.FasParams(1e-30, 3, 2, ml)
# reference: single engine
p1 = P.Field(g, LOC, 1, p0.copy(), device=dev)
f1 = P.Field(g, LOC, 1, f0.copy(), device=dev)
rep1 = P.FasSolver(P.make_hierarchy(g, ml), LOC, bc, plan, coeffs).solve(p1, f1, params)
# distributed
ds = DistSlabSolver(P.make_hierarchy(g, ml), LOC, bc, plan, coeffs, 2, dev,
                    min_planes=4)
p2 = torch.from_numpy(p0.copy()).to(dev)
f2 = torch.from_numpy(f0.copy()).to(dev)
pv = slab_view(p2, 1, n, world, rank)
fv = slab_view(f2, 1, n, world, rank)
rep2 = ds.solve(pv, fv, params)  # singular: distributed ordered means of f and p
torch.cuda.synchronize()
lo, hi = 2 * rank * (n // 2 // world) + 1, 2 * (rank + 1) * (n // 2 // world)
if ea == 0:
    hi = min(hi, n - 1)  # the wall node n is not an unknown
sl = (slice(lo, hi + 1),) + tuple(slice(1, n if a == ea else n + 1) for a in range(1, dim))
mine = p2[sl]
ref = p1.data[sl]
ok = torch.equal(mine, ref) and torch.equal(f2[sl], f1.data[sl])
hist_ok = np.allclose(rep2.residual_history, rep1.residual_history, rtol=1e-12, atol=0)
print(f"rank {rank}/{world} {loc} kg={ds.engine.kg} slab cells {lo}..{hi}: field bitwise {ok}, "
      f"history {hist_ok} {rep2.residual_history[-1]:.6e} vs {rep1.residual_history[-1]:.6e}", flush=True)
ds.close()
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if (ok and hist_ok) else 1)
