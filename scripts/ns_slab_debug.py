"""Progress trace of the virtual-rank slab NS stepper (which solve stalls):
    python scripts/ns_slab_debug.py N PARTS ORDER"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.ns import NSParams
from paper_2510_11152_b200.ns_slab import SlabProjectionStepper, VirtualRanks
from paper_2510_11152_b200 import slab as S
n, parts, order = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
orig = S.VirtualSlabSolver.solve_views
def traced(self, pvs, fvs, params, halo_p=1, halo_f=1):
    es = self.engines(params.s, pvs[0].device)
    print(f"  solve {self.location.name} kg={[e.kg if hasattr(e, 'kg') else '?' for e in es]} ...", flush=True)
    t0 = time.time()
    rep = orig(self, pvs, fvs, params, halo_p, halo_f)
    torch.cuda.synchronize()
    print(f"  ... {rep.iterations} cycles {time.time() - t0:.2f}s", flush=True)
    return rep
S.VirtualSlabSolver.solve_views = traced
g = P.unit_grid((n, n, n))
sl = SlabProjectionStepper(g, NSParams(re=100.0, dt=1e-3, order=order, tol=1e-10, k_max=20),
                           VirtualRanks(parts))
sl.set_state({})
for k in range(2):
    print("step", k, flush=True)
    sl.step()
print("done", flush=True)
