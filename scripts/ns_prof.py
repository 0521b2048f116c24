"""Kernel-time breakdown of NS projection steps with torch.profiler (CUPTI
activity records: device-side kernel durations, no replay).
Usage: python scripts/ns_prof.py N [order] [steps]"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2510_11152_b200 as P
from paper_2510_11152_b200.ns import NSParams, ProjectionStepper, cavity_bcs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = P.unit_grid((n,) * 3)
st = ProjectionStepper(g, NSParams(re=100.0, dt=1e-3, order=order, tol=1e-10, k_max=20, s=2,
                                   mesh_level=n.bit_length() - 2), cavity_bcs(3))
st.set_state({})
st.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        st.step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        nm = ev.name.split("(")[0].replace("void ", "").replace("fasmg::", "")[:48]
        a = agg[nm]
        a[0] += 1
        a[1] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1e3
tot = sum(a[1] for a in agg.values())
print(f"{n}^3 order {order}: {steps} steps, device kernel time {tot / steps:.1f} ms/step")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
    print(f"  {nm:48s} x{c / steps:7.1f}/step {t / steps:8.2f} ms/step")
