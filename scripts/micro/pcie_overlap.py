"""PCIe copy concurrency on the box: H2D alone, D2H alone, H2D || D2H on two
streams, H2D || device work.  Sizes: one 514^3 fp64 field (1.09 GB)."""
import time, torch
n = 514 ** 3
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device=dev)
d_b = torch.empty(n, dtype=torch.float64, device=dev)
d_c = torch.empty(n, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3

def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
def work():
    for _ in range(20):
        d_c.mul_(1.0000001)
def h2d_work():
    h2d(); work()
gb = n * 8 / 1e9
for name, fn in [("h2d", h2d), ("d2h", d2h), ("h2d||d2h", both), ("work", work), ("h2d||work", h2d_work)]:
    ms = timed(fn)
    print(f"{name:10s} {ms:8.2f} ms  ({gb / ms * 1e3:.1f} GB/s per 1.09 GB)", flush=True)
