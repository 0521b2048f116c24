"""Multi-process slab NS step (one process per "GPU"; all may share one device):
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ns_slab_selftest.py
Each rank runs the same 2 projection steps on its slab (DistRanks) and
compares the gathered fields with a single-GPU stepper (bitwise)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2510_11152_b200 as P  # noqa: E402
from paper_2510_11152_b200.ns import NSParams, ProjectionStepper  # noqa: E402
from paper_2510_11152_b200.ns_slab import DistRanks, SlabProjectionStepper  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ndev = torch.cuda.device_count()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % ndev)
torch.cuda.set_device(dev)
shared = world > ndev
dist.init_process_group("gloo" if shared else "nccl", **({} if shared else {"device_id": dev}))
n = int(os.environ.get("NS_SLAB_N", "32"))
order = int(os.environ.get("NS_SLAB_ORDER", "2"))
g = P.unit_grid((n, n, n))
prm = NSParams(re=100.0, dt=1e-3, order=order, tol=1e-10, k_max=20)
ref = ProjectionStepper(g, prm, device=dev)
ref.set_state({})
sl = SlabProjectionStepper(g, prm, DistRanks(), device=dev)
sl.set_state({})
ok = True
for k in range(2):
    a = ref.step()
    b = sl.step()
    for c in ref.comps:
        ok &= np.allclose(b.momentum[c].residual_history, a.momentum[c].residual_history,
                          rtol=1e-12, atol=0)
        ok &= bool(torch.equal(sl.velocity_global(c), ref.velocity(c).interior))
    ok &= np.allclose(b.pressure.residual_history, a.pressure.residual_history, rtol=1e-12,
                      atol=0)
    ok &= bool(torch.equal(sl.pressure_global(), ref.pressure().interior))
ok &= sl.divergence() == ref.divergence()
print(f"rank {rank}/{world} n={n} order {order}: 2 steps bitwise {ok}", flush=True)
sl.close()
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
