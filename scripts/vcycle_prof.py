"""Per-kernel device time of graph-replayed V-cycles (torch.profiler / CUPTI,
live, warm caches), grouped by kernel name and grid (so the levels of one
kernel show separately), plus the idle gaps between kernels.
Usage: python scripts/vcycle_prof.py N LOC(cell|ew|ns|tb) [cycles] [out.json]"""
import collections, json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import paper_2510_11152_b200 as P
n = int(sys.argv[1]); loc = {"cell": "CELL", "ew": "EDGE_EW", "ns": "EDGE_NS", "tb": "EDGE_TB"}[sys.argv[2]]
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dim = int(os.environ.get("PROF_DIM", "3"))
g = P.unit_grid((n,) * dim); L = getattr(P.Location, loc)
p = P.Field(g, L); f = P.Field(g, L)
p.interior = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), L, P.BoundaryCondition.dirichlet(dim),
                P.make_plan("x", dim), P.OperatorCoeffs(1.0, 1.0 if loc == "CELL" else 0.05))
e = S.engine(2, p.device); e.load(p, f); e.run(2, True)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record(); e.run(cyc, True); en.record(); torch.cuda.synchronize()
live = st.elapsed_time(en) / cyc
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e.run(cyc, True)
    torch.cuda.synchronize()
tr = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(tr)
evs = [x for x in json.load(open(tr))["traceEvents"] if x.get("cat") == "kernel"]
evs.sort(key=lambda x: x["ts"])
agg = collections.defaultdict(lambda: [0, 0.0])
gaps = 0.0
for i, ev in enumerate(evs):
    nm = ev["name"].split("(")[0].replace("void ", "").replace("fasmg::", "")
    nm = nm.split("<")[0] + ("<" + nm.split("<")[1][:18] if "<" in nm else "")
    grid = tuple(ev.get("args", {}).get("grid", []))
    a = agg[(nm, grid)]; a[0] += 1; a[1] += ev["dur"] / 1e3
    if i:
        gaps += max(0.0, ev["ts"] - (evs[i - 1]["ts"] + evs[i - 1]["dur"])) / 1e3
tot = sum(a[1] for a in agg.values())
print(f"{loc} {n}^3: live {live:.3f} ms per V-cycle (events); profiled kernel time {tot / cyc:.3f} ms, "
      f"gaps {gaps / cyc:.3f} ms, {len(evs) / cyc:.0f} kernels per V-cycle")
rows = []
for (nm, grid), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    rows.append({"kernel": nm, "grid": list(grid), "per_cycle": c / cyc, "ms_per_cycle": t / cyc,
                 "us_per_launch": 1e3 * t / c})
    print(f"  {nm:44s} {str(grid):18s} x{c / cyc:5.1f} {t / cyc:7.3f} ms  {1e3 * t / c:8.1f} us/launch")
if len(sys.argv) > 4:
    json.dump({"loc": loc, "n": n, "live_ms": live, "kernel_ms": tot / cyc, "gaps_ms": gaps / cyc,
               "rows": rows}, open(sys.argv[4], "w"), indent=1)
