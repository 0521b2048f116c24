"""Benchmark: MDOF/s per FAS V-cycle, 3D heat 512^3, % of HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--grid 512] [--dim 3] [--no-cpu-baseline]

Workload (BASELINE.json configs[2], the config the metric is quoted on):
one backward-Euler heat step p - dt*Lap(p) = f with dt = 1 (a = b = 1) on a
512^3 cell-centered grid, Dirichlet 0, X-MCGS 'ff' smoother, s = 2,
meshLevel = log2(n) - 1 = 8, f = L_h(exact manufactured solution)
(PKG/manufactured.py:76-84), p0 = default_rng(0).random --
the paper's timing problem.  Synthetic data.

A "step" is one outer iteration of FasSolver.solve (PKG/fas.py:147-154):
one FAS V-cycle followed by the outer residual norm read back for the tol
test -- the paper's per-"iteration" time.

* value: steps timed on the device (CUDA events on the engine stream) with
  p and f resident in HBM, K steps after W warm-up steps.  Each field is
  1.09 GB, far larger than the 126 MB L2, so no flush is needed between
  steps.
* e2e: the same metric through the public API with HOST buffers: each step
  is one problem of ``FasSolver.solve_host_batch`` -- copy p0 and f from
  pinned host memory to the device, ``solve(..., FasParams(tol, k_max=1,
  s=2, mesh_level=8))`` (the paper's kMax = 1 timing call: pack, V-cycle,
  residual norm, unpack, ghost fill), copy p back to pinned host memory.
  The batch call overlaps the H2D copy of problem i+1 and the D2H copy of
  problem i-1 with the solve of problem i; ``e2e.serial`` reports the same
  calls one problem at a time with nothing overlapped.
* roofline: the dominant kernel, the finest-level smoothing half-sweep,
  re-timed live with CUDA events on its launch stream; algorithmic bytes =
  12 B per fine DOF per half-sweep (read the opposite-parity half of p and
  this half of f, write this half of p).
* cpu_baseline: the CPU oracle port of the reference (oracle/, C, all host
  threads) timed on one V-cycle + norm of the same inputs, rank 0, N = 1.
* --impl reference: the same metric from the oracle port alone (the
  reference is pure Python+numba and does not travel to the GPU box).

Multi-GPU (torchrun, one process per GPU): the SAME 512^3 problem is split
into axis-0 slabs (paper_2510_11152_b200/slab.py DistSlabSolver): halo
planes are pushed into the neighbours' memory after every smoothing
half-sweep over CUDA IPC / NVLink, coarse levels are all-gathered and
solved redundantly, the residual is reduced in rank order.  Strong
scaling: value = 512^3 / max-over-ranks time per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MDOF/s per FAS V-cycle, 3D heat 512³ (1–8 B200), % of HBM roofline"
PAPER_4090_MDOFS = 289.7  # RTX 4090, 3D 512^3, 0.4633 s per V-cycle
BYTES_PER_DOF_HALF_SWEEP = 12.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--grid", dest="n", type=int, default=512)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_dict(n, dim, parallelism):
    ml = int(np.log2(n)) - 1
    fb = (n + 2) ** dim * 8  # bytes of one field
    return {
        "workload": f"heat{dim}d_{n}: backward-Euler step p - dt*Lap(p) = f, dt=1 (a=b=1), "
                    f"cell-centered {n}^{dim}, Dirichlet 0, FAS V-cycle, X-MCGS ff, s=2, "
                    f"meshLevel={ml}, f=L_h(manufactured), p0=U[0,1)",
        "grid": [n] * dim, "mesh_level": ml, "smoother": "X-MCGS ff", "s": 2,
        "step": "one FAS V-cycle + outer residual norm (PKG/fas.py:147-154)",
        "l2_flush": ("not needed: each field is %.2f GB >> 126 MB L2" % (fb / 1e9) if fb > 4 * 126e6
                     else "none: each field is %.3f GB, not >> 126 MB L2 (functional size, not a "
                          "bench configuration)" % (fb / 1e9)),
        "parallelism": parallelism,
    }


def make_inputs(n, dim):
    """Host arrays (reference layout, halo 1) of the timing problem."""
    from paper_2510_11152_b200 import manufactured as M
    import paper_2510_11152_b200 as P
    g = P.unit_grid((n,) * dim)
    shape = (n + 2,) * dim
    inner = (slice(1, -1),) * dim
    p0 = np.zeros(shape)
    p0[inner] = np.random.default_rng(0).random((n,) * dim)
    return g, p0, shape, inner


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampler of SM clocks and throttle reasons."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        inwin = [s for t, s in self.samples if any(a - 0.06 <= t <= b + 0.06 for a, b in self.windows)]
        use = inwin if inwin else [s for _, s in self.samples]
        sm, smax, reasons, power = [], None, set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in use:
            parts = [x.strip() for x in s.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "samples_in_timed_region": len(inwin),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------- CPU oracle
def cpu_oracle_vcycle(p0, f_int, n, dim, threads, cycles=1):
    """One (or more) V-cycle(s) + residual norm of the same problem on the
    CPU oracle port; returns seconds per step."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    O.set_threads(threads)
    op = O.OField((n,) * dim, "cell", 1, p0.copy())
    of = O.OField((n,) * dim, "cell", 1)
    of.interior[...] = f_int
    t0 = time.perf_counter()
    O.fas_solve(op, of, 1.0, 1.0, O.uniform_bc(dim, "dirichlet"), O.plan_colors("x", dim),
                1e-300, cycles, 2, int(np.log2(n)) - 1)
    return (time.perf_counter() - t0) / cycles


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------- reference arm
def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n, dim = args.n, args.dim
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    shape = (n + 2,) * dim
    p0 = np.zeros(shape)
    p0[(slice(1, -1),) * dim] = np.random.default_rng(0).random((n,) * dim)
    f_int = O.poisson_rhs_discrete((n,) * dim)
    threads = host_threads()
    budget_s = 150.0
    t_first = cpu_oracle_vcycle(p0, f_int, n, dim, threads)  # warm-up step (also a sample)
    steps = max(1, min(args.steps, int(budget_s / max(t_first, 1e-3))))
    t = cpu_oracle_vcycle(p0, f_int, n, dim, threads, cycles=steps)
    value = n ** dim / t / 1e6
    sample = (f"{steps} V-cycle(s)+norm of the full {n}^{dim} workload after 1 warm-up cycle, "
              f"oracle/ C port of the reference, OpenMP {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MDOF/s",
        "n_gpus": world, "steps": steps, "warmup": 1, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(n, dim, "cpu"),
        "cpu_baseline": {"value": value, "unit": "MDOF/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "MDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm
def b200_arm(args):
    import torch
    import paper_2510_11152_b200 as P
    from paper_2510_11152_b200.grid import Field, Location

    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"[bench] warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    ndev = torch.cuda.device_count()
    shared = world > ndev  # functional test: several ranks on one device
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n, dim = args.n, args.dim
    K, W = args.steps, max(args.warmup, 3)
    g, p0, shape, inner = make_inputs(n, dim)
    from paper_2510_11152_b200 import manufactured as M
    f_dev = M.poisson_rhs_discrete(g, device=dev)  # f = L_h(p_exact) on the device
    coeffs = P.OperatorCoeffs(1.0, 1.0)
    ml = int(np.log2(n)) - 1
    plan = P.make_plan("x", dim, "ff")
    bc = P.BoundaryCondition.dirichlet(dim)
    hier = P.make_hierarchy(g, ml)
    dof = n ** dim

    if world == 1:
        p = Field(g, Location.CELL, 1, p0, device=dev)
        f = Field(g, Location.CELL, 1, f_dev.data.clone())
        solver = P.FasSolver(hier, Location.CELL, bc, plan, coeffs)
        eng = solver.engine(2, dev)
        eng.load(p, f)
        run_step = lambda: eng.run(1, with_norm=True)  # noqa: E731
        stream_handle = eng.stream.value
        local_dof = dof
        parallelism = "single"
    else:
        from paper_2510_11152_b200.slab import DistSlabSolver, slab_view
        ds = DistSlabSolver(hier, Location.CELL, bc, plan, coeffs, 2, dev)
        pg = torch.from_numpy(p0).to(dev)
        fg = f_dev.data.clone()
        pv = slab_view(pg, 1, n, world, rank)
        fv = slab_view(fg, 1, n, world, rank)
        ds.load(pv, fv)
        eng = ds.engine

        def run_step():
            eng.launch(1, True)
            return eng.result()
        stream_handle = eng.stream.value
        local_dof = dof // world
        parallelism = (f"z-slab x{world} (axis-0 slabs, halo push per half-sweep over "
                       f"CUDA IPC/NVLink, coarse levels >= {eng.kg} gathered)"
                       + (" [ranks sharing one device: functional test only]" if shared else ""))
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)

    # --- device-resident timed region: K outer iterations (V-cycle + norm,
    #     host reads the residual each step exactly as FasSolver.solve does)
    for _ in range(W):
        run_step()
    st = torch.cuda.ExternalStream(stream_handle, device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    ev0.record(st)
    hist = []
    for _ in range(K):
        hist.append(run_step())
    ev1.record(st)
    torch.cuda.synchronize()
    t1 = time.time()
    clocks.mark(t0, t1)
    ms_step = max_over_ranks(ev0.elapsed_time(ev1) / K)
    if dist is not None:
        dist.barrier()
    value = dof / (ms_step * 1e-3) / 1e6

    # --- live per-launch timing of the dominant kernel (finest half-sweep)
    sweep_ms = eng.time_sweeps(0, 16)
    achieved = BYTES_PER_DOF_HALF_SWEEP * local_dof / (sweep_ms * 1e-3) / 1e9
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        try:
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    if os.path.exists(prof) and world == 1:
        try:
            d = json.load(open(prof))
            if d.get("n") == n and d.get("dim") == dim:
                traffic = float(d["dram_bytes_per_launch"])
        except Exception:
            pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": ("k_sweep_tma" if dim == 3 else "k_sweep_fast")
                          + " (finest-level X-MCGS half-sweep)",
                "kernel_ms": sweep_ms,
                "algorithmic_bytes_per_launch": BYTES_PER_DOF_HALF_SWEEP * local_dof,
                "peak_source": peak_src,
                "vcycle_model_GBps_per_gpu": (259.4 if dim == 3 else 306.7) * local_dof
                                             / (ms_step * 1e-3) / 1e9}

    from paper_2510_11152_b200 import _native as N
    kernels = int(N.lib().fasmg_engine_kernels_per_vcycle(eng.handle, 1))

    # --- e2e through the public API with host buffers (single GPU: Field +
    #     solve(kMax=1); slabs: per-rank slab copies + DistSlabSolver)
    e2e_steps = args.e2e_steps or max(3, K)
    cur = torch.cuda.current_stream(dev)
    serial = None
    if world == 1:
        ph = torch.from_numpy(p0).pin_memory()
        fh = torch.empty(shape, dtype=torch.float64).pin_memory()
        fh.copy_(f_dev.data.cpu())
        outs = [torch.empty(shape, dtype=torch.float64).pin_memory() for _ in range(2)]
        params1 = P.FasParams(1e-9, 1, 2, ml)
        pe = Field(g, Location.CELL, 1, device=dev)
        fe = Field(g, Location.CELL, 1, device=dev)

        def serial_step():
            pe.data.copy_(ph, non_blocking=True)
            fe.data.copy_(fh, non_blocking=True)
            solver.solve(pe, fe, params1)
            outs[0].copy_(pe.data, non_blocking=True)

        # the timed e2e region: e2e_steps independent problems through the
        # public host-batch API (H2D of problem i+1 and D2H of problem i-1
        # overlap the solve of problem i)
        def e2e_run(k):
            solver.solve_host_batch([ph] * k, [fh] * k, params1,
                                    out=[outs[i % 2] for i in range(k)])
        h2d = 2 * int(np.prod(shape)) * 8
        d2h = int(np.prod(shape)) * 8 + 8
        api = ("FasSolver.solve_host_batch(host pinned p_i, f_i, FasParams(k_max=1)) over "
               f"{e2e_steps} problems: H2D p,f -> solve -> D2H p per problem, copies "
               "pipelined on two streams against the solves")
        # the same call sequence one problem at a time (no overlap), reported beside it
        serial_step()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for _ in range(e2e_steps):
            serial_step()
        b.record(cur)
        torch.cuda.synchronize()
        serial = {"ms_per_step": a.elapsed_time(b) / e2e_steps,
                  "api": "Field(host pinned -> device) + solve(kMax=1) + p -> host, one "
                         "problem at a time"}
        serial["value"] = dof / (serial["ms_per_step"] * 1e-3) / 1e6
    else:
        ph = pv.cpu().pin_memory()
        fh = fv.cpu().pin_memory()
        out_h = torch.empty_like(ph).pin_memory()

        def e2e_step():
            pv.copy_(ph, non_blocking=True)
            fv.copy_(fh, non_blocking=True)
            ds.load(pv, fv)
            ds.run(1)
            ds.store(pv)
            out_h.copy_(pv, non_blocking=True)
        h2d = 2 * ph.numel() * 8
        d2h = ph.numel() * 8 + 8
        api = "rank slab (host pinned -> device) + DistSlabSolver load/run(1)/store + slab -> host"

        def e2e_run(k):
            for _ in range(k):
                e2e_step()
    e2e_run(2)  # warm-up (allocates the batch API's two staging buffers)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    t2 = time.time()
    a.record(cur)
    if os.environ.get("BENCH_E2E_TRACE"):
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            e2e_run(e2e_steps)
            torch.cuda.synchronize()
        evs = sorted(prof.events(), key=lambda e: e.time_range.start)
        t00 = evs[0].time_range.start
        for e in evs:
            if "emcpy" in e.name or "ynchronize" in e.name or "alloc" in e.name.lower():
                print(f"[trace] {e.name[:40]:40s} {(e.time_range.start - t00) / 1e3:9.2f} "
                      f"{(e.time_range.end - e.time_range.start) / 1e3:9.2f}", file=sys.stderr)
    else:
        e2e_run(e2e_steps)
    b.record(cur)
    torch.cuda.synchronize()
    clocks.mark(t2, time.time())
    e2e_ms = max_over_ranks(a.elapsed_time(b) / e2e_steps)
    e2e = {"value": dof / (e2e_ms * 1e-3) / 1e6, "unit": "MDOF/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_ms, "steps": e2e_steps, "api": api}
    if serial is not None:
        e2e["serial"] = serial
    clocks.stop()

    # --- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        t_cpu = cpu_oracle_vcycle(p0, f_dev.interior.cpu().numpy(), n, dim, threads)
        cpu = {"value": dof / t_cpu / 1e6, "unit": "MDOF/s", "cores": threads, "kind": "port",
               "sample": f"1 V-cycle + residual norm of the same {n}^{dim} inputs on the oracle/ "
                         f"C port of the reference (OpenMP, {threads} threads)",
               "cpu": cpu_model(), "s_per_step": t_cpu}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": value / PAPER_4090_MDOFS,
            "vs_baseline_ref": "RTX 4090, 0.4633 s per V-cycle at 3D 512^3 (PAPER.md:510)",
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(n, dim, parallelism),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks.summary(), "gpu_launches": kernels * K,
            "kernels_per_step": kernels,
            "residual_last": (g.h ** (dim / 2.0)) * float(np.sqrt(hist[-1])) if hist else None,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        if world > 1:
            ds.close()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
