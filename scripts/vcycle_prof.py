"""Per-kernel device time of graph-replayed V-cycles (torch.profiler / CUPTI).
Usage: python scripts/vcycle_prof.py N LOC(cell|ew|ns|tb) [cycles]"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2510_11152_b200 as P
n = int(sys.argv[1]); loc = {"cell": "CELL", "ew": "EDGE_EW", "ns": "EDGE_NS", "tb": "EDGE_TB"}[sys.argv[2]]
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = P.unit_grid((n,) * 3); L = getattr(P.Location, loc)
p = P.Field(g, L); f = P.Field(g, L)
p.interior = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), L, P.BoundaryCondition.dirichlet(3),
                P.make_plan("x", 3), P.OperatorCoeffs(1.0, 0.05))
e = S.engine(2, p.device); e.load(p, f); e.run(2, True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e.run(cyc, True)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        nm = ev.name.split("(")[0].replace("void ", "").replace("fasmg::", "")[:46]
        a = agg[nm]; a[0] += 1; a[1] += ev.device_time_total / 1e3
tot = sum(a[1] for a in agg.values())
print(f"{loc} {n}^3: device kernel time {tot / cyc:.3f} ms per V-cycle")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"  {nm:46s} x{c / cyc:6.1f} {t / cyc:7.3f} ms")
