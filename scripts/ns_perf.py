"""3D lid-driven cavity projection steps on the B200 path: per-step device
time, V-cycles per solve, per-V-cycle MDOF/s and memory footprint.
Usage: python scripts/ns_perf.py N [order] [steps] [mode]   (prints one JSON line)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.ns import NSParams, ProjectionStepper, cavity_bcs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
mode = sys.argv[4] if len(sys.argv) > 4 else "efficient"
ml = n.bit_length() - 2
g = P.unit_grid((n,) * 3)
free0, total = torch.cuda.mem_get_info()
prm = NSParams(re=100.0, dt=1e-3, order=order, mode=mode, tol=1e-10, k_max=20, s=2, mesh_level=ml)
st = ProjectionStepper(g, prm, cavity_bcs(3))
st.set_state({})
rows = []
for k in range(steps):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    rep = st.step()
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    cyc = {c: r.iterations for c, r in rep.momentum.items()}
    cyc["p"] = rep.pressure.iterations
    rows.append({"step": k + 1, "ms": wall, "cycles": cyc, "div": st.divergence(),
                 "p_res": rep.pressure.final_residual})
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
free1, _ = torch.cuda.mem_get_info()
steady = rows[1:] if len(rows) > 1 else rows
ms = sum(r["ms"] for r in steady) / len(steady)
cycles = sum(sum(r["cycles"].values()) for r in steady) / len(steady)
dof_cell = n ** 3
dof_edge = (n - 1) * n * n
dof_cycle = (sum(sum(v for c, v in r["cycles"].items() if c != "p") for r in steady) * dof_edge
             + sum(r["cycles"]["p"] for r in steady) * dof_cell) / len(steady)
print(json.dumps({
    "grid": [n] * 3, "order": order, "mode": mode, "re": 100.0, "dt": 1e-3, "mesh_level": ml,
    "steps": steps, "ms_per_step": ms, "vcycles_per_step": cycles,
    "mdof_vcycles_per_s": dof_cycle / (ms * 1e-3) / 1e6,
    "resident_slots": st.resident_count(),
    "device_mem_gb": (free0 - free1) / 1e9, "max_abs_divergence": max(abs(r["div"]) for r in rows),
    "per_step": rows}))
