"""One warm NS projection step at N^3 (for ncu launch lists): step 1 from rest,
then the profiled step 2.  Usage: python scripts/ns_step_once.py N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.ns import NSParams, ProjectionStepper, cavity_bcs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.unit_grid((n,) * 3)
st = ProjectionStepper(g, NSParams(re=100.0, dt=1e-3, order=2, tol=1e-10, k_max=20, s=2,
                                   mesh_level=n.bit_length() - 2), cavity_bcs(3))
st.set_state({})
st.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
