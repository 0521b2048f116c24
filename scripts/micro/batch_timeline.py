"""Timeline of FasSolver.solve_host_batch at 512^3 (torch.profiler/CUPTI):
memcpy and kernel spans per stream, to check the H2D/solve/D2H overlap."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2510_11152_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = P.unit_grid((n,) * 3)
ml = int(np.log2(n)) - 1
S = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0))
shape = (n + 2,) * 3
ph = torch.rand(shape, dtype=torch.float64).pin_memory()
fh = torch.rand(shape, dtype=torch.float64).pin_memory()
outs = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in range(2)]
prm = P.FasParams(1e-9, 1, 2, ml)
wk = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ballast = torch.empty(int(sys.argv[4]) if len(sys.argv) > 4 else 0, dtype=torch.uint8, device='cuda')
S.solve_host_batch([ph] * wk, [fh] * wk, prm, out=outs[:wk])
torch.cuda.synchronize()
for rep in range(int(sys.argv[5]) if len(sys.argv) > 5 else 2):
    t = time.perf_counter()
    S.solve_host_batch([ph] * k, [fh] * k, prm, out=[outs[i % 2] for i in range(k)])
    torch.cuda.synchronize()
    print(f"batch of {k}: {(time.perf_counter() - t) * 1e3 / k:.2f} ms/problem", flush=True)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    S.solve_host_batch([ph] * k, [fh] * k, prm, out=[outs[i % 2] for i in range(k)])
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
spans = {}
for e in ev:
    key = ("memcpy " if "emcpy" in e.name else "kern ") + str(getattr(e, "device_resource_id", "?"))
    s, t = (e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3
    if "emcpy" in e.name:
        print(f"{e.name[:40]:40s} stream {getattr(e, 'device_resource_id', '?')} {s:9.2f} -> {t:9.2f} ms")
    else:
        a = spans.setdefault(key, [1e18, 0, 0])
        a[0] = min(a[0], s); a[1] = max(a[1], t); a[2] += t - s
for kk, a in spans.items():
    print(f"{kk}: first {a[0]:.2f} last {a[1]:.2f} busy {a[2]:.2f} ms")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and
       ("Synchronize" in e.name or "Malloc" in e.name or "cudaMemcpy" in e.name)]
for e in cpu[:40]:
    print(f"cpu {e.name[:40]:40s} {(e.time_range.start - t0) / 1e3:9.2f} dur {(e.time_range.end - e.time_range.start) / 1e3:8.2f} ms")
