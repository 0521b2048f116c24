"""Run a few eager (non-graph) V-cycles at a given size for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_11152_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 2
loc = P.Location[sys.argv[4].upper()] if len(sys.argv) > 4 else P.Location.CELL
halo = 2 if loc.edge_axis is not None else 1
shape = (n,) * dim
g = P.unit_grid(shape)
p = P.Field(g, loc, halo)
f = P.Field(g, loc, halo)
p.interior[...] = torch.rand(p.interior.shape, dtype=torch.float64, device='cuda')
f.interior[...] = torch.rand(f.interior.shape, dtype=torch.float64, device='cuda')
S = P.FasSolver(P.make_hierarchy(g, int(np.log2(n)) - 1), loc,
                P.BoundaryCondition.dirichlet(dim), P.make_plan('x', dim),
                P.OperatorCoeffs(1.0, 1.0 if loc is P.Location.CELL else 0.05))
e = S.engine(2, p.device)
e.load(p, f)
for _ in range(cycles):
    e.run(1, True, use_graph=False)
torch.cuda.synchronize()
print("done")
