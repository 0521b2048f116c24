"""Quick perf probe: time FAS V-cycles (+norm) of the engine at a size."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P

def run(n, dim, cycles=10):
    shape = (n,) * dim
    g = P.unit_grid(shape)
    ml = int(np.log2(n)) - 1
    p = P.Field(g, P.Location.CELL)
    f = P.Field(g, P.Location.CELL)
    p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device='cuda')
    f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device='cuda')
    S = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, P.BoundaryCondition.dirichlet(dim),
                    P.make_plan('x', dim), P.OperatorCoeffs(1.0, 1.0))
    e = S.engine(2, p.device)
    e.load(p, f)
    e.run(3, True)
    st = torch.cuda.ExternalStream(e.stream.value)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    e.run(cycles, True)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / cycles
    N = n ** dim
    print(f"{dim}D {n}: {ms:.3f} ms/cycle  {N/ms/1e3:.1f} MDOF/s  kernels/cycle {e.kernels_per_vcycle()}  "
          f"model {259.4 if dim==3 else 306.7} B/DOF -> {N*(259.4 if dim==3 else 306.7)/ms/1e6:.0f} GB/s", flush=True)

for arg in sys.argv[1:]:
    n, dim = map(int, arg.split('x'))
    run(n, dim)
