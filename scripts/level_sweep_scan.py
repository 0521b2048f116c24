"""Half-sweep time per level and V-cycle time at 3D 512^3 for engine knobs
given as env strings, e.g.
    python scripts/level_sweep_scan.py "" "FASMG_MARCH_CHUNK=2" "FASMG_TMA_MIN=0"
(knobs are read when an engine is created)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N
n = int(os.environ.get("SCAN_N", "512"))
loc = getattr(P.Location, os.environ.get("SCAN_LOC", "CELL"))
g = P.unit_grid((n,) * 3)
p = P.Field(g, loc); f = P.Field(g, loc)
torch.manual_seed(0)
p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device="cuda")
f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device="cuda")
base = dict(os.environ)
for cfg in sys.argv[1:]:
    os.environ.clear(); os.environ.update(base)
    for kv in cfg.split():
        k, v = kv.split("=")
        os.environ[k] = v
    S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), loc, P.BoundaryCondition.dirichlet(3),
                    P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0 if loc is P.Location.CELL else 0.05))
    e = S.engine(2, p.device); e.load(p, f)
    out = []
    ms = ctypes.c_double()
    for k in range(4):
        N.call("fasmg_engine_time_sweeps", e.handle, k, 4, ctypes.byref(ms))
        N.call("fasmg_engine_time_sweeps", e.handle, k, 32, ctypes.byref(ms))
        nk = n >> k
        out.append(f"L{k} {ms.value * 1e3:6.1f}us ({12.0 * nk ** 3 / ms.value / 1e6:5.0f} GB/s)")
    e.run(3, True)
    st = torch.cuda.ExternalStream(e.stream.value)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(st); e.run(20, True); b.record(st); torch.cuda.synchronize()
    print(f"[{cfg or 'default'}] V-cycle+norm {a.elapsed_time(b) / 20:.3f} ms | " + " | ".join(out), flush=True)
    del e, S
    torch.cuda.synchronize()
