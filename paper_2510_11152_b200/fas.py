"""Full Approximation Storage multigrid: V-cycle and outer solve loop.

Same API and semantics as PKG/fas.py (Algorithm 1):
``FasSolver(hierarchy, location, bc, plan, coeffs)``, ``.vcycle(p, f, s)``,
``.solve(p, f, params) -> SolveReport``, and the ``solve``/``vcycle``
convenience wrappers.

Execution: a native engine (csrc/fasmg_engine.cu, one per smoothing count
``s``) holds every level in the parity-blocked layout, runs the V-cycle as
one CUDA graph (smoothing half-sweeps, fused residual+restriction+tau,
coarse source, fused prolongation+correction) and the outer residual norm,
and returns one scalar per cycle for the ``tol`` test.  ``p`` and ``f`` are
packed on entry and ``p`` unpacked on exit; the caller-visible state after
``solve`` (interior, ghosts, the singular-case mean shifts of ``f`` and
``p``) matches the reference bitwise.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _native as N
from .boundary import BoundaryCondition, fill_ghosts
from .errors import NativeError
from .grid import Field, GridHierarchy, Location, make_hierarchy, subtract_interior_mean
from .smoothers import SweepPlan
from .stencil import OperatorCoeffs

# FASMG_DEVICE_LOOP=0: the outer loop on the host, one graph launch per
# iteration (the device loop's conditional graph node is not supported by
# compute-sanitizer's racecheck / synccheck)
_DEVICE_LOOP = os.environ.get("FASMG_DEVICE_LOOP", "1") != "0"


@dataclass(frozen=True)
class FasParams:
    """tol, cycle cap, smoothing steps per stage, recursion depth
    (PKG/fas.py:37-49)."""

    tol: float
    k_max: int
    s: int
    mesh_level: int

    def __post_init__(self):
        if self.tol <= 0 or self.k_max < 1 or self.s < 1 or self.mesh_level < 1:
            raise ValueError(f"invalid solver parameters {self}")


@dataclass
class SolveReport:
    iterations: int
    residual_history: list
    converged: bool

    @property
    def final_residual(self) -> float:
        return self.residual_history[-1] if self.residual_history else float("nan")


class _Engine:
    """Owner of one native engine handle."""

    def __init__(self, solver: "FasSolver", s: int, device: torch.device):
        g = solver.hierarchy.fine
        kinds, vals = solver.bc.codes()
        masks = solver.plan.class_masks()
        ea = solver.location.edge_axis
        self.device = device
        self.stream = N.engine_stream(device.index)
        args = (g.dim, N.ints(g.shape), -1 if ea is None else ea,
                float(g.domain_min[0]), float(g.domain_max[0]),
                solver.hierarchy.mesh_level, float(solver.coeffs.a), float(solver.coeffs.b),
                N.ints(kinds), N.doubles(vals), len(masks),
                (ctypes.c_uint * len(masks))(*masks), int(s), self.stream)
        self.arena = solver.arena  # keeps the arena alive while the engine lives
        with torch.cuda.device(device):
            if solver.arena is None:
                h = N.lib().fasmg_engine_create(*args)
            else:
                h = N.lib().fasmg_engine_create_in(*args, solver.arena.handle)
        if not h:
            raise NativeError("fasmg_engine_create failed: "
                              + N.lib().fasmg_last_error().decode(errors="replace"))
        self.handle = ctypes.c_void_p(h)

    def close(self):
        if self.handle is not None and N._lib is not None:
            N.lib().fasmg_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _same_device(self, *fields):
        for F in fields:
            if F.device != self.device:
                raise ValueError(f"field on {F.device}, solver engine on {self.device}")

    def load(self, p: Field, f: Field):
        self._same_device(p, f)
        with torch.cuda.device(self.device):
            N.wait(self.stream, N.torch_stream(self.device))
            pc, fc = p.core, f.core
            N.call("fasmg_engine_load", self.handle, N.ptr(pc), N.strides(pc), N.ptr(fc),
                   N.strides(fc))

    def store(self, p: Field):
        self._same_device(p)
        with torch.cuda.device(self.device):
            pc = p.core
            N.call("fasmg_engine_store", self.handle, N.ptr(pc), N.strides(pc))
            N.wait(N.torch_stream(self.device), self.stream)

    def solve_loop(self, k_max: int, tol: float, scale: float) -> list:
        """Up to ``k_max`` V-cycles + norms in ONE graph launch, stopping on
        the device at the first ``scale*sqrt(sumsq) <= tol`` (the host loop's
        test, bitwise): the residual history."""
        hist = (ctypes.c_double * k_max)()
        n = ctypes.c_int(0)
        with torch.cuda.device(self.device):
            N.call("fasmg_engine_solve", self.handle, int(k_max), float(tol), float(scale), hist,
                   ctypes.byref(n))
        return list(hist[: n.value])

    def run(self, count: int, with_norm: bool, use_graph: bool = True) -> float:
        out = ctypes.c_double(0.0)
        with torch.cuda.device(self.device):
            N.call("fasmg_engine_run", self.handle, int(count), 1 if with_norm else 0,
                   ctypes.byref(out), 1 if use_graph else 0)
        return out.value

    def kernels_per_vcycle(self, with_norm: bool = True) -> int:
        """Kernels launched by one captured V-cycle (+ norm) graph."""
        return int(N.lib().fasmg_engine_kernels_per_vcycle(self.handle, 1 if with_norm else 0))

    def time_sweeps(self, level: int = 0, reps: int = 20) -> float:
        """Mean duration (ms) of one smoothing half-sweep launch on `level`,
        CUDA events on the engine stream."""
        ms = ctypes.c_double()
        with torch.cuda.device(self.device):
            N.call("fasmg_engine_time_sweeps", self.handle, int(level), int(reps),
                   ctypes.byref(ms))
        return ms.value


class EngineArena:
    """Level arrays shared by the engines of several solvers that never run
    concurrently (one stream, one solve at a time) -- e.g. the three
    momentum solves and the pressure solve of a projection step, which then
    hold one set of multigrid workspaces instead of four."""

    def __init__(self):
        self.handle = ctypes.c_void_p(N.lib().fasmg_arena_create())

    def __del__(self):
        try:
            if self.handle is not None and N._lib is not None:
                N.lib().fasmg_arena_release(self.handle)
                self.handle = None
        except Exception:
            pass


class FasSolver:
    """Reusable solver owning one workspace set per level (PKG/fas.py:63-89).

    Workspaces live in the native engine (allocated on first use per
    smoothing count ``s``), so time steppers that reuse a solver never
    reallocate.
    """

    def __init__(self, hierarchy: GridHierarchy, location: Location,
                 bc: BoundaryCondition, plan: SweepPlan, coeffs: OperatorCoeffs,
                 arena: EngineArena | None = None):
        self.arena = arena
        self.hierarchy = hierarchy
        self.location = location
        self.bc = bc
        self.bc_homog = bc.homogenized()
        self.plan = plan
        self.coeffs = coeffs
        self.use_graph = True
        self._engines: dict = {}
        self._staging: dict = {}  # solve_host_batch device buffers

    def engine(self, s: int, device: torch.device) -> _Engine:
        key = (int(s), device.index)
        e = self._engines.get(key)
        if e is None:
            e = self._engines[key] = _Engine(self, s, device)
        return e

    def _check(self, p: Field, f: Field):
        if p.location is not self.location or f.location is not self.location:
            raise ValueError("field location does not match the solver")
        if p.grid.shape != self.hierarchy.fine.shape or f.grid.shape != p.grid.shape:
            raise ValueError("field grid does not match the solver hierarchy")

    # -- one V-cycle -------------------------------------------------------
    def vcycle(self, p: Field, f: Field, s: int) -> Field:
        """One V-cycle on ``p`` in place (PKG/fas.py:93-128); leaves ghosts
        stale."""
        self._check(p, f)
        e = self.engine(s, p.device)
        e.load(p, f)
        e.run(1, with_norm=False, use_graph=self.use_graph)
        e.store(p)
        p.ghosts_fresh = False
        return p

    # -- outer loop --------------------------------------------------------
    def _singular(self) -> bool:
        return self.coeffs.a == 0.0 and all(
            rule.kind != "dirichlet" for _, rule in self.bc.faces)

    def solve(self, p: Field, f: Field, params: FasParams) -> SolveReport:
        """Iterate V-cycles on ``p`` until ``res <= tol`` (PKG/fas.py:137-162).
        For a singular problem the rhs is shifted to zero mean in place and
        the returned solution is shifted to zero mean."""
        self._check(p, f)
        with torch.cuda.device(p.device):
            history = self._solve(p, f, params)
        return SolveReport(iterations=len(history), residual_history=history,
                           converged=bool(history and history[-1] <= params.tol))

    def solve_into(self, p0: Field, p: Field, f: Field, params: FasParams) -> SolveReport:
        """``solve`` with the initial guess read from ``p0`` and the solution
        (ghosts filled) written to ``p`` -- bitwise ``p.data.copy_(p0.data);
        solve(p, f, params)`` without the copy: the engine packs ``p0``
        directly, and every element of ``p`` is rewritten (interior by the
        store, the rest by fill_ghosts).  Used by the NS drivers, whose
        momentum solves start from u^n and write u~ into another slot."""
        self._check(p0, f)
        self._check(p, f)
        with torch.cuda.device(p.device):
            history = self._solve(p, f, params, p0=p0)
        return SolveReport(iterations=len(history), residual_history=history,
                           converged=bool(history and history[-1] <= params.tol))

    def _solve(self, p: Field, f: Field, params: FasParams, p0: Field | None = None) -> list:
        singular = self._singular()
        if singular:
            subtract_interior_mean(f)
        e = self.engine(params.s, p.device)
        e.load(p if p0 is None else p0, f)
        g = self.hierarchy.fine
        scale = g.h ** (g.dim / 2.0)
        history: list = []
        if self.use_graph and _DEVICE_LOOP and 1 <= params.k_max <= 4096:
            # the loop below, with the test on the device: one graph launch
            history = e.solve_loop(params.k_max, params.tol, scale)
        else:
            for _ in range(params.k_max):
                sumsq = e.run(1, with_norm=True, use_graph=self.use_graph)
                res = scale * math.sqrt(sumsq)
                history.append(res)
                if res <= params.tol:
                    break
        e.store(p)
        fill_ghosts(p, self.bc)
        if singular:
            subtract_interior_mean(p)
            p.ghosts_fresh = False
        return history

    # -- independent problems held in host memory --------------------------
    def solve_host_batch(self, ps, fs, params: FasParams, out=None, halo: int = 1,
                         device=None) -> list:
        """``solve`` over a sequence of independent problems whose arrays
        live in HOST memory (torch CPU tensors of the full field shape, ghost
        rings included; pinned memory for asynchronous copies).

        Per problem the result equals ``solve(Field(p), Field(f), params)``
        bitwise: the solution (with filled ghosts) is written to ``out[i]``
        (default: ``ps[i]`` in place) and, for a singular problem, the
        mean-shifted rhs back to ``fs[i]`` as the reference mutates the
        caller's f (PKG/fas.py:145).

        The copies are pipelined over two device staging buffers: the
        host->device copy of problem i+1 runs on its own stream while
        problem i is solved, and the device->host copy of problem i runs on a
        third stream in the opposite PCIe direction, so a batch costs about
        max(H2D, solve, D2H) per problem instead of their sum."""
        n = len(ps)
        if len(fs) != n or (out is not None and len(out) != n):
            raise ValueError("ps, fs and out must have the same length")
        if n == 0:
            return []
        out = list(ps) if out is None else list(out)
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        g = self.hierarchy.fine
        singular = self._singular()
        # reject a result that would be copied out while memory it overlaps is
        # still to be read (the input of another problem, or -- singular
        # problems write the shifted rhs back -- a written array of any problem)
        spans = [(_host_span(t), j % n, j < n) for j, t in enumerate((*ps, *fs))]
        written = [(_host_span(t), i) for i, t in enumerate(out)]
        if singular:
            written += [(_host_span(t), i) for i, t in enumerate(fs)]
        for w, i in written:
            for r, j, _ in spans:
                if j != i and _overlap(w, r):
                    raise ValueError(f"a written host array of problem {i} shares memory with "
                                     f"the input of problem {j}")
        if singular:
            for i in range(n):
                if _overlap(_host_span(out[i]), _host_span(fs[i])):
                    raise ValueError(f"problem {i}: out shares memory with f, which a singular "
                                     "solve writes back shifted")
        with torch.cuda.device(dev):
            return self._host_batch(ps, fs, out, params, halo, dev, g, singular)

    def _host_batch(self, ps, fs, out, params, halo, dev, g, singular) -> list:
        n = len(ps)
        # two staging (p, f) pairs per (device, halo), kept on the solver so
        # that repeated batches allocate nothing
        bufs = self._staging.setdefault((dev.index, halo), [])
        while len(bufs) < min(n, 2):
            bufs.append((Field(g, self.location, halo, device=dev),
                         Field(g, self.location, halo, device=dev)))
        bufs = bufs[:max(1, min(n, 2))]
        shape = tuple(bufs[0][0].data.shape)
        for t in (*ps, *fs, *out):
            if t.device.type != "cpu" or tuple(t.shape) != shape or t.dtype != torch.float64:
                raise ValueError(f"host arrays must be float64 CPU tensors of shape {shape}")
        comp = torch.cuda.current_stream(dev)
        h2d = torch.cuda.Stream(dev)
        d2h = torch.cuda.Stream(dev)
        drained = [None] * len(bufs)  # event: buffer's last result copied out
        loaded = [None] * n

        def enqueue_h2d(i):
            b = i % len(bufs)
            with torch.cuda.stream(h2d):
                if drained[b] is not None:
                    h2d.wait_event(drained[b])
                bufs[b][0].data.copy_(ps[i], non_blocking=True)
                bufs[b][1].data.copy_(fs[i], non_blocking=True)
                loaded[i] = torch.cuda.Event()
                loaded[i].record(h2d)

        reports = []
        h2d.wait_stream(comp)  # earlier work on the staging buffers was ordered on comp
        enqueue_h2d(0)
        for i in range(n):
            if i + 1 < n:
                enqueue_h2d(i + 1)
            b = i % len(bufs)
            p, f = bufs[b]
            p.ghosts_fresh = f.ghosts_fresh = False
            comp.wait_event(loaded[i])
            reports.append(self.solve(p, f, params))
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                out[i].copy_(p.data, non_blocking=True)
                if singular:
                    fs[i].copy_(f.data, non_blocking=True)
                drained[b] = torch.cuda.Event()
                drained[b].record(d2h)
        comp.wait_stream(d2h)
        comp.wait_stream(h2d)
        # the results are in host memory when this returns: the last copies
        # out are still in flight on d2h until here
        d2h.synchronize()
        return reports


def _host_span(t: torch.Tensor):
    """(storage address, first byte, end byte) of a host tensor's data."""
    st = t.untyped_storage()
    lo = t.storage_offset() * t.element_size()
    ext = 1 + sum((m - 1) * abs(s) for m, s in zip(t.shape, t.stride())) if t.numel() else 0
    return st.data_ptr(), st.data_ptr() + lo, st.data_ptr() + lo + ext * t.element_size()


def _overlap(a, b) -> bool:
    return a[1] < b[2] and b[1] < a[2]


def vcycle(p: Field, f: Field, coeffs: OperatorCoeffs, params: FasParams,
           plan: SweepPlan, bc: BoundaryCondition, solver: FasSolver | None = None) -> Field:
    """One V-cycle (PKG/fas.py:165-172)."""
    if solver is None:
        hier = make_hierarchy(p.grid, params.mesh_level)
        solver = FasSolver(hier, p.location, bc, plan, coeffs)
    return solver.vcycle(p, f, params.s)


def solve(p0: Field, f: Field, coeffs: OperatorCoeffs, params: FasParams,
          plan: SweepPlan, bc: BoundaryCondition):
    """Solve ``a p - b Lap(p) = f`` from ``p0`` (updated in place)
    (PKG/fas.py:175-181)."""
    hier = make_hierarchy(p0.grid, params.mesh_level)
    solver = FasSolver(hier, p0.location, bc, plan, coeffs)
    report = solver.solve(p0, f, params)
    return p0, report
