"""Time finest-level half-sweeps + full cycles for sweep variants (env)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200 import _native as N
peak = 6550.7
for arg in sys.argv[1:]:
    n, dim = map(int, arg.split('x'))
    shape = (n,) * dim
    g = P.unit_grid(shape)
    p = P.Field(g, P.Location.CELL); f = P.Field(g, P.Location.CELL)
    p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device='cuda')
    f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device='cuda')
    S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), P.Location.CELL,
                    P.BoundaryCondition.dirichlet(dim), P.make_plan('x', dim), P.OperatorCoeffs(1.0, 1.0))
    e = S.engine(2, p.device); e.load(p, f)
    ms = ctypes.c_double()
    N.call("fasmg_engine_time_sweeps", e.handle, 0, 4, ctypes.byref(ms))
    N.call("fasmg_engine_time_sweeps", e.handle, 0, 40, ctypes.byref(ms))
    byts = 12.0 * n ** dim
    e.run(3, True)
    st = torch.cuda.ExternalStream(e.stream.value)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(st); e.run(10, True); b.record(st); torch.cuda.synchronize()
    cyc = a.elapsed_time(b) / 10
    print(f"{os.environ.get('FASMG_SWEEP_VARIANT','2')}/{os.environ.get('FASMG_MARCH_CHUNK','32')} {dim}D {n}: half-sweep {ms.value*1e3:7.1f} us = {byts/ms.value/1e6:7.0f} GB/s ({byts/ms.value/1e6/peak*100:4.1f}%)  cycle {cyc:.3f} ms {n**dim/cyc/1e3:8.0f} MDOF/s", flush=True)
