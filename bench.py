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
* cpu_baseline_reference_1core: the UNMODIFIED reference package
  (baseline/_ref, numba backend, NUMBA_NUM_THREADS=1 -- its parallel
  Gauss-Seidel is unusable) timed on one outer
  iteration of the same inputs in a subprocess: the paper's own
  single-core baseline configuration.
* --impl reference: the same metric, config, K and W from the oracle port
  alone on all host threads.
* --workload ns512|ns1024: one Navier-Stokes projection step (BASELINE
  configs[3]/[4]) per bench step: steps/s, per-solve MDOF/s per V-cycle,
  the edge-field half-sweep against the roofline.
* --gpus N > 1 outside torchrun relaunches itself under
  torch.distributed.run with N processes.

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
    ap.add_argument("--workload", default="heat", choices=("heat", "ns512", "ns1024", "ns"),
                    help="heat: the headline V-cycle metric; ns512/ns1024: one Navier-Stokes "
                         "projection step of BASELINE configs[3]/[4] per bench step")
    ap.add_argument("--no-numba-baseline", action="store_true",
                    help="skip the single-core run of the real reference (baseline/_ref)")
    ap.add_argument("--numba-child", action="store_true", help=argparse.SUPPRESS)
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
        "pack_unpack": "excluded from value (p and f stay in the engine's parity-blocked "
                       "layout between steps), included in e2e",
    }


def parallelism_of(world: int) -> str:
    return "single" if world == 1 else f"z-slab x{world}"


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
    """The reference's CPU path on the box's host cores: the oracle/ C port of
    the reference V-cycle (pinned bitwise to the reference's own outputs) on
    all host threads, W warm-up steps then K timed steps of the SAME
    workload and config as the GPU arm.  Rank 0 only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    if args.workload != "heat":
        return ns_reference_arm(args)
    n, dim = args.n, args.dim
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    shape = (n + 2,) * dim
    p0 = np.zeros(shape)
    p0[(slice(1, -1),) * dim] = np.random.default_rng(0).random((n,) * dim)
    f_int = O.poisson_rhs_discrete((n,) * dim)
    threads = host_threads()
    K, W = args.steps, max(args.warmup, 3)
    t_w = cpu_oracle_vcycle(p0, f_int, n, dim, threads, cycles=W)  # warm-up steps
    budget_s = 240.0
    steps = K if t_w * K <= budget_s else max(1, int(budget_s / max(t_w, 1e-3)))
    t = cpu_oracle_vcycle(p0, f_int, n, dim, threads, cycles=steps)
    value = n ** dim / t / 1e6
    sample = (f"{steps} V-cycle(s)+norm of the full {n}^{dim} workload after {W} warm-up "
              f"cycles, oracle/ C port of the reference, OpenMP {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MDOF/s",
        "n_gpus": world, "steps": steps, "warmup": W, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(n, dim, parallelism_of(world)),
        "cpu_baseline": {"value": value, "unit": "MDOF/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "MDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------- the real reference, one core
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def numba_child(args):
    """Runs in a subprocess with NUMBA_NUM_THREADS=1 and baseline/_ref on the
    path: the UNMODIFIED reference package (numba backend) times one outer
    iteration (V-cycle + residual norm, FasSolver.solve with kMax=1) of the
    same workload after a JIT warm-up on a 16^d grid; prints one JSON line."""
    import fasmg as fm
    from fasmg import manufactured as M
    n, dim = args.n, args.dim
    ml = int(np.log2(n)) - 1

    def problem(m):
        g = fm.unit_grid((m,) * dim)
        p = fm.Field(g, fm.Location.CELL, 1)
        p.interior[...] = np.random.default_rng(0).random((m,) * dim)
        f = M.poisson_rhs_discrete(g)
        S = fm.FasSolver(fm.make_hierarchy(g, int(np.log2(m)) - 1), fm.Location.CELL,
                         fm.BoundaryCondition.dirichlet(dim), fm.make_plan("x", dim, "ff"),
                         fm.OperatorCoeffs(1.0, 1.0))
        return p, f, S

    t0 = time.perf_counter()
    p, f, S = problem(16)
    S.solve(p, f, fm.FasParams(1e-300, 2, 2, 3))  # JIT compile
    t_jit = time.perf_counter() - t0
    p, f, S = problem(n)
    t0 = time.perf_counter()
    rep = S.solve(p, f, fm.FasParams(1e-300, 1, 2, ml))
    t = time.perf_counter() - t0
    print(json.dumps({"s_per_step": t, "jit_s": t_jit, "residual": rep.residual_history[-1],
                      "backend": os.environ.get("FASMG_BACKEND", "numba"),
                      "numba_threads": os.environ.get("NUMBA_NUM_THREADS")}), flush=True)
    return 0


def numba_baseline(n, dim):
    """Single-core timing of the real reference (the
    numba backend, 1 core -- its parallel Gauss-Seidel is unusable, SURVEY.md
    section 0 item 2) or None when baseline/_ref is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "fasmg")):
        return None
    env = dict(os.environ, NUMBA_NUM_THREADS="1", OMP_NUM_THREADS="1",
               NUMBA_CACHE_DIR="/tmp/fasmg_numba_cache", PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=REF_DIR + os.pathsep + os.environ.get("PYTHONPATH", ""))
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    try:
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--numba-child",
                              "--grid", str(n), "--dim", str(dim)], env=env,
                             capture_output=True, text=True, timeout=600)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 -- reported, never fatal to the GPU line
        return {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}
    t = d["s_per_step"]
    return {"value": n ** dim / t / 1e6, "unit": "MDOF/s", "cores": 1, "kind": "reference",
            "sample": f"1 V-cycle + residual norm (FasSolver.solve, kMax=1) of the same {n}^{dim} "
                      "inputs by the unmodified reference package (baseline/_ref, numba "
                      "backend, NUMBA_NUM_THREADS=1) after a 16^d JIT warm-up",
            "s_per_step": t, "cpu": cpu_model()}


# ------------------------------------------------------------------ B200 arm
def b200_arm(args):
    import torch
    import paper_2510_11152_b200 as P
    from paper_2510_11152_b200.grid import Field, Location

    rank, world, local = dist_env()
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
        scale_res = g.h ** (dim / 2.0)
        # K outer iterations as FasSolver.solve runs them: one graph launch,
        # the residual test on the device (tol -1: never met, so exactly K)
        def run_steps(k):  # (in launches of at most 4096 iterations, the loop's cap)
            out = []
            while k > 0:
                out += eng.solve_loop(min(k, 4096), -1.0, scale_res)
                k -= min(k, 4096)
            return out
        stream_handle = eng.stream.value
        local_dof = dof
        slab_detail = None
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

        def run_steps(k):  # the device loop on every rank, as DistSlabSolver.solve runs it
            out = []
            while k > 0:
                out += ds.solve_loop(min(k, 4096), -1.0)
                k -= min(k, 4096)
            return out
        stream_handle = eng.stream.value
        local_dof = dof // world
        slab_detail = (f"axis-0 slabs, halo push per half-sweep over CUDA IPC/NVLink, "
                       f"coarse levels >= {eng.kg} gathered"
                       + (" [ranks sharing one device: functional test only]" if shared else ""))
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)

    # --- device-resident timed region: K outer iterations (V-cycle + norm +
    #     convergence test), issued the way FasSolver.solve issues them:
    #     single GPU -> one graph launch with the test on the device
    #     (fasmg_engine_solve); slabs -> per-iteration launch + host read
    run_steps(1)      # builds the graph entered from a fresh load
    run_steps(W - 1)  # ... and the one entered with a speculation pending
    st = torch.cuda.ExternalStream(stream_handle, device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    ev0.record(st)
    hist = run_steps(K)
    ev1.record(st)
    torch.cuda.synchronize()
    t1 = time.time()
    clocks.mark(t0, t1)
    ms_step = max_over_ranks(ev0.elapsed_time(ev1) / K)
    if dist is not None:
        dist.barrier()
    value = dof / (ms_step * 1e-3) / 1e6
    host_loop = None
    if world == 1:  # the per-iteration host loop (launch + read), beside it
        for _ in range(2):  # its graph variants captured outside the timing
            run_step()
        torch.cuda.synchronize()
        ev0.record(st)
        for _ in range(K):
            run_step()
        ev1.record(st)
        torch.cuda.synchronize()
        host_loop = {"ms_per_step": ev0.elapsed_time(ev1) / K,
                     "api": "engine.run(1, with_norm=True) per iteration: graph launch + "
                            "host read of the norm + host-side test"}

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
    # kernels per timed step: one device-loop iteration (V-cycle + norm +
    # k_conv, the WHILE body)
    kernels = int(N.lib().fasmg_engine_kernels_per_vcycle(eng.handle, 2))

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
    numba = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.no_numba_baseline:
        numba = numba_baseline(n, dim)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": value / PAPER_4090_MDOFS,
            "vs_baseline_ref": "RTX 4090, 0.4633 s per V-cycle at 3D 512^3 (PAPER.md:510)",
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(n, dim, parallelism_of(world)),
            "slab": slab_detail,
            "roofline": roofline, "cpu_baseline": cpu,
            "cpu_baseline_reference_1core": numba, "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": kernels * K,
            "kernels_per_step": kernels,
            "solve_loop": "one graph launch per rank for the K iterations (conditional WHILE "
                          "node, device-side residual test k_conv)",
            "host_loop": host_loop,
            "residual_last": hist[-1] if hist else None,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        if world > 1:
            ds.close()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------- Navier-Stokes workload
NS_METRIC = "NS projection steps/s, 3D lid-driven cavity {n}³, 2nd order, 8-slot schedule (f64)"


def ns_config(n, world):
    ml = int(np.log2(n)) - 1
    return {
        "workload": f"ns3d_{n}: lid-driven cavity (u=1 on zhi), Re 100, dt 1e-3, 2nd-order MAC "
                    f"projection, memory-efficient 8-slot schedule (PAPER.md Table 5), FAS "
                    f"X-MCGS ff s=2 tol 1e-10 kMax 20 meshLevel {ml}, from rest after the "
                    f"warm-up steps",
        "grid": [n] * 3, "mesh_level": ml, "order": 2, "schedule": "efficient (8 slots)",
        "step": "one projection step: 3 momentum rhs (WENO3) + 3 edge-field FAS solves + "
                "divergence + singular pressure FAS solve + correction + p update",
        "l2_flush": "not needed: each field is %.2f GB >> 126 MB L2" % ((n + 2) ** 3 * 8 / 1e9),
        "parallelism": parallelism_of(world),
        "pack_unpack": "included (each solve packs p, f into the blocked layout and unpacks p)",
    }


def ns_size(args):
    return {"ns512": 512, "ns1024": 1024}.get(args.workload, args.n)


def ns_arm(args):
    """One NS projection step per bench step (BASELINE configs[3] at 512^3,
    configs[4] at 1024^3), single GPU: steps/s, per-solve MDOF/s per V-cycle
    from CUDA events around every schedule Step, the edge-field finest
    half-sweep against the HBM roofline."""
    import torch
    import paper_2510_11152_b200 as P
    from paper_2510_11152_b200.ns import NSParams, ProjectionStepper

    rank, world, local = dist_env()
    if world > 1:
        return ns_slab_arm(args)
    n = ns_size(args)
    K, W = args.steps, max(args.warmup, 3)
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    ml = int(np.log2(n)) - 1
    st = ProjectionStepper(P.unit_grid((n,) * 3), NSParams(re=100.0, dt=1e-3, order=2,
                                                           mode="efficient", tol=1e-10, k_max=20,
                                                           s=2, mesh_level=ml), device=dev)
    st.set_state({})
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    for _ in range(W):
        st.step()
    torch.cuda.synchronize()
    st.timing = []
    cur = torch.cuda.current_stream(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    a.record(cur)
    reps = [st.step() for _ in range(K)]
    b.record(cur)
    torch.cuda.synchronize()
    clocks.mark(t0, time.time())
    ms_step = a.elapsed_time(b) / K
    # per formula/component device time, and V-cycles per solve
    per = {}
    for formula, comp, e0, e1 in st.timing:
        key = formula if formula in ("copy", "rotate2", "p_update") else f"{formula}:{comp or 'p'}"
        per[key] = per.get(key, 0.0) + e0.elapsed_time(e1) / K
    st.timing = None
    cyc = {c: sum(r.momentum[c].iterations for r in reps) / K for c in st.comps}
    cyc["p"] = sum(r.pressure.iterations for r in reps) / K
    solves = {}
    for c in st.comps + ("p",):
        key = f"solve_momentum:{c}" if c != "p" else "solve_pressure:p"
        dofs = n ** 3 if c == "p" else (n - 1) * n * n
        ms = per.get(key, 0.0)
        solves[c] = {"ms_per_step": ms, "vcycles_per_step": cyc[c],
                     "mdofs_per_vcycle": dofs * cyc[c] / (ms * 1e-3) / 1e6 if ms else None}
    # dominant kernel: finest half-sweep of an edge-field (momentum) solve
    eng = st.solvers["u"].engine(2, dev)
    sweep_ms = eng.time_sweeps(0, 16)
    edofs = (n - 1) * n * n
    achieved = BYTES_PER_DOF_HALF_SWEEP * edofs / (sweep_ms * 1e-3) / 1e9
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    # e2e: the same steps through the public API with host state: set_state
    # from pinned host arrays, K steps, velocities and pressure back to host
    hvel = {c: torch.zeros(tuple(st.velocity(c).interior.shape), dtype=torch.float64).pin_memory()
            for c in st.comps}
    hp = torch.zeros(tuple(st.pressure().interior.shape), dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    a.record(cur)
    t2 = time.time()
    st.set_state({c: hvel[c] for c in st.comps}, hp)
    for _ in range(K):
        st.step()
    for c in st.comps:
        hvel[c].copy_(st.velocity(c).interior, non_blocking=True)
    hp.copy_(st.pressure().interior, non_blocking=True)
    b.record(cur)
    torch.cuda.synchronize()
    clocks.mark(t2, time.time())
    e2e_ms = a.elapsed_time(b) / K
    state_bytes = (sum(v.numel() for v in hvel.values()) + hp.numel()) * 8
    clocks.stop()
    mem = torch.cuda.max_memory_allocated(dev)
    free_b, total_b = torch.cuda.mem_get_info(dev)
    line = {
        "metric": NS_METRIC.format(n=n), "value": 1e3 / ms_step, "unit": "steps/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (cavity from rest)", "config": ns_config(n, world),
        "solves": solves, "ms_per_step_by_formula": per,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "k_sweep_tma (finest edge-field u half-sweep)",
                     "kernel_ms": sweep_ms, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": BYTES_PER_DOF_HALF_SWEEP * edofs},
        "e2e": {"value": 1e3 / e2e_ms, "unit": "steps/s",
                "h2d_bytes_per_step": state_bytes // K, "d2h_bytes_per_step": state_bytes // K,
                "ms_per_step": e2e_ms,
                "api": f"ProjectionStepper.set_state(host pinned) + {K} x step() + velocities "
                       "and pressure to host; the state copies amortised over the steps"},
        "cpu_baseline": None, "clocks": clocks.summary(),
        "torch_max_allocated_gb": mem / 1e9,
        "device_used_gb": (total_b - free_b) / 1e9,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = ns_cpu_sample(min(n, 256))
    print(json.dumps(line), flush=True)
    return 0


def ns_slab_arm(args):
    """NS projection steps on axis-0 slabs, one process per GPU (BASELINE
    configs[4]: the 1024^3 cavity across 8 B200; ns_slab.SlabProjectionStepper
    over DistRanks: NCCL row exchanges, DistSlabSolver peer-store halos).
    Total work is fixed (strong scaling); the step time is the max over ranks
    of CUDA events around K steps bracketed by barriers."""
    import torch
    import torch.distributed as dist
    import paper_2510_11152_b200 as P
    from paper_2510_11152_b200.ns import NSParams
    from paper_2510_11152_b200.ns_slab import DistRanks, SlabProjectionStepper

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    shared = world > ndev  # functional run: several ranks time-slice one device
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = ns_size(args)
    K, W = args.steps, max(args.warmup, 3)
    ml = int(np.log2(n)) - 1
    st = SlabProjectionStepper(P.unit_grid((n,) * 3),
                               NSParams(re=100.0, dt=1e-3, order=2, mode="efficient", tol=1e-10,
                                        k_max=20, s=2, mesh_level=ml), DistRanks(), device=dev)
    st.set_state({})
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    for _ in range(W):
        st.step()
    torch.cuda.synchronize()
    dist.barrier()
    cur = torch.cuda.current_stream(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    a.record(cur)
    reps = [st.step() for _ in range(K)]
    b.record(cur)
    torch.cuda.synchronize()
    dist.barrier()
    if clocks:
        clocks.mark(t0, time.time())
    ms_step = max_over_ranks(a.elapsed_time(b) / K)
    cyc = {c: sum(r.momentum[c].iterations for r in reps) / K for c in st.comps}
    cyc["p"] = sum(r.pressure.iterations for r in reps) / K
    # e2e through the public API: every rank loads its slab of the state from
    # pinned host memory, runs K steps and copies its slab back
    slabs = {q: st.field_of(f"{q}_n") for q in st.comps}
    slabs["p"] = st.field_of("p_n")
    host = {q: torch.zeros(tuple(F.interior(rank).shape), dtype=torch.float64).pin_memory()
            for q, F in slabs.items()}
    torch.cuda.synchronize()
    dist.barrier()
    t2 = time.time()
    a.record(cur)
    for q, F in slabs.items():
        F.interior(rank).copy_(host[q], non_blocking=True)
        if q != "p":
            st._refresh(F, st.bcs[q])
            st.field_of(f"{q}_nm1").copy_from(F)
    for _ in range(K):
        st.step()
    for q in host:
        host[q].copy_(st.field_of(f"{q}_n" if q != "p" else "p_n").interior(rank), non_blocking=True)
    b.record(cur)
    torch.cuda.synchronize()
    dist.barrier()
    if clocks:
        clocks.mark(t2, time.time())
    e2e_ms = max_over_ranks(a.elapsed_time(b) / K)
    state_bytes = torch.tensor([sum(h.numel() for h in host.values()) * 8.0], dtype=torch.float64,
                               device="cpu" if shared else dev)
    dist.all_reduce(state_bytes)
    mem = max_over_ranks(torch.cuda.max_memory_allocated(dev) / 1e9)
    if rank == 0:
        clocks.stop()
        line = {
            "metric": NS_METRIC.format(n=n), "value": 1e3 / ms_step, "unit": "steps/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (cavity from rest)", "config": ns_config(n, world),
            "slab": {"ranks": world, "planes_per_rank": n // world,
                     "exchange": "row blocks over torch.distributed (%s) + solver halos by "
                                 "peer stores from the sweep kernels" % ("gloo" if shared else "NCCL"),
                     "ranks_share_device": shared},
            "vcycles_per_step": cyc,
            "e2e": {"value": 1e3 / e2e_ms, "unit": "steps/s",
                    "h2d_bytes_per_step": int(state_bytes.item()) // K,
                    "d2h_bytes_per_step": int(state_bytes.item()) // K, "ms_per_step": e2e_ms,
                    "api": f"every rank: slab state from pinned host + {K} x "
                           "SlabProjectionStepper.step() + slab state to host; copies amortised "
                           "over the steps"},
            "cpu_baseline": None, "clocks": clocks.summary(), "torch_max_allocated_gb": mem,
        }
        print(json.dumps(line), flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def ns_cpu_sample(m):
    """One projection step of the pinned NS oracle (oracle/ns_oracle.py, C
    kernels on all host threads) at m^3, after one warm-up step."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import ns_oracle as NO
    threads = host_threads()
    O.set_threads(threads)
    orc = NO.NSOracle((m,) * 3, 100.0, 1e-3, 2, tol=1e-10, k_max=20, s=2,
                      mesh_level=int(np.log2(m)) - 1)
    orc.step()
    t0 = time.perf_counter()
    orc.step()
    t = time.perf_counter() - t0
    return {"value": 1.0 / t, "unit": "steps/s", "cores": threads, "kind": "port",
            "sample": f"step 2 of the {m}^3 cavity by the oracle/ NS port (C kernels, OpenMP "
                      f"{threads} threads); NOT the bench grid when m < n -- scale by (m/n)^3 "
                      "for a rough per-DOF comparison", "grid": m}


def ns_reference_arm(args):
    n = ns_size(args)
    K, W = args.steps, max(args.warmup, 3)
    base = ns_cpu_sample(n)
    line = {"impl": "reference", "metric": NS_METRIC.format(n=n), "value": base["value"],
            "unit": "steps/s", "n_gpus": 1, "steps": 1, "warmup": 1,
            "ms_per_step": 1e3 / base["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (cavity from rest)",
            "config": ns_config(n, 1), "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": f"requested K={K} W={W}; one timed step at this size (minutes of CPU)",
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def self_launch(args) -> int:
    """``--gpus N`` (N > 1) outside torchrun: relaunch this command under
    torch.distributed.run with N processes (127.0.0.1 rendezvous) instead of
    silently measuring one GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] --gpus {args.gpus} without torchrun: relaunching as {' '.join(cmd)}",
          file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.numba_child:
        return numba_child(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    rank, world, _ = dist_env()
    if world != args.gpus:
        print(f"[bench] error: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return reference_arm(args)
    if args.workload != "heat":
        return ns_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
