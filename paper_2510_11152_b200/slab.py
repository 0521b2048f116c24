"""Axis-0 slab decomposition of the FAS solver across GPUs.

Each rank's native engine owns the slab ``rank`` (a contiguous range of
block planes along array axis 0, the outermost axis of the C-order layout)
of every level whose plane count splits evenly into enough planes per rank;
coarser levels are replicated and solved redundantly on every rank (same
inputs, same results, no scatter).  Inside the V-cycle graph:

* after every smoothing half-sweep the updated classes' boundary planes are
  stored straight into the neighbours' halo planes (CUDA P2P / IPC peer
  memory over NVLink) and published with system-scope release/acquire
  counters -- one exchange per color sweep, as the north star asks;
* after the restriction the coarse slab halos, or -- at the first replicated
  level -- the whole coarse level, are exchanged the same way (all-gather);
* the outer residual's sum of squares is reduced in fixed rank order.

Fields and residual histories equal the single-GPU solve: every per-point
value is computed from identical inputs in identical order (bitwise); only
the norm's summation order differs (~1e-16 relative).

Two front ends share the engine:

* :class:`VirtualSlabSolver` -- P slabs on ONE device in one process, each
  with its own stream; same kernels, same peer-store/counter protocol
  (the "virtual ranks" test of SURVEY.md §4 item 3a);
* :class:`DistSlabSolver` -- one process per GPU (torch.distributed for the
  rendezvous): each rank exports its level arrays as CUDA IPC handles, maps
  its peers', and runs its own graph.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native as N
from .boundary import BoundaryCondition, fill_ghosts
from .errors import NativeError
from .fas import FasParams, SolveReport
from .grid import Field, GridHierarchy, Location, subtract_interior_mean
from .smoothers import SweepPlan
from .stencil import OperatorCoeffs


def slab_cells(n0: int, nranks: int, rank: int):
    """1-based inclusive range of axis-0 cells owned by ``rank`` at the
    finest level (block planes are pairs of cells)."""
    B0 = n0 // 2
    if B0 % nranks:
        raise ValueError(f"{B0} block planes do not split over {nranks} ranks")
    nb = B0 // nranks
    return 2 * rank * nb + 1, 2 * (rank + 1) * nb


def slab_view(data: torch.Tensor, halo: int, n0: int, nranks: int, rank: int) -> torch.Tensor:
    """The rank's cells along axis 0 plus one ghost plane on each side, as a
    view of the global C-order data array (core index 0 at data g-1).  For
    a field whose edge axis is axis 0 the same core range holds the rank's
    nodes (the interface node belongs to the lower rank); the last rank's
    view ends at the wall node n when the array has no ring beyond it."""
    lo, hi = slab_cells(n0, nranks, rank)
    return data[halo - 1 + lo - 1: halo - 1 + hi + 2]


class _SlabEngine:
    def __init__(self, hierarchy: GridHierarchy, location: Location, bc: BoundaryCondition,
                 plan: SweepPlan, coeffs: OperatorCoeffs, s: int, nranks: int, rank: int,
                 device: torch.device, min_planes: int = 4, stream=None):
        g = hierarchy.fine
        kinds, vals = bc.codes()
        masks = plan.class_masks()
        self.device = device
        if stream is None:
            with torch.cuda.device(device):
                stream = ctypes.c_void_p()
                N.check(N.lib().fasmg_stream_create(ctypes.byref(stream)))
            self._own_stream = True
        else:
            self._own_stream = False
        self.stream = stream
        ea = -1 if location is Location.CELL else location.edge_axis
        with torch.cuda.device(device):
            h = N.lib().fasmg_engine_create_slab(
                g.dim, N.ints(g.shape), ea, float(g.domain_min[0]), float(g.domain_max[0]),
                hierarchy.mesh_level, float(coeffs.a), float(coeffs.b), N.ints(kinds),
                N.doubles(vals), len(masks), (ctypes.c_uint * len(masks))(*masks), int(s),
                self.stream, int(nranks), int(rank), int(min_planes))
        if not h:
            raise NativeError("fasmg_engine_create_slab failed: "
                              + N.lib().fasmg_last_error().decode(errors="replace"))
        self.handle = ctypes.c_void_p(h)
        self.nranks, self.rank = nranks, rank
        self.n0 = g.shape[0]
        info = (ctypes.c_int * 3)()
        N.call("fasmg_engine_slab_info", self.handle, info)
        self.kg, self.planes, self.off0 = info[0], info[1], info[2]

    def export(self):
        cnt = N.lib().fasmg_engine_export_count(self.handle)
        arr = (ctypes.c_ulonglong * cnt)()
        N.check(N.lib().fasmg_engine_export(self.handle, arr))
        return list(arr)

    def connect(self, all_exports):
        flat = [x for e in all_exports for x in e]
        arr = (ctypes.c_ulonglong * len(flat))(*flat)
        N.check(N.lib().fasmg_engine_connect(self.handle, arr, len(all_exports)))

    def load(self, pv: torch.Tensor, fv: torch.Tensor, halo_p: int, halo_f: int):
        """Pack slab views (rank cells + 1 ghost plane each side along axis 0)."""
        def core(v, g):
            return v[(slice(None),) + tuple(slice(g - 1, v.shape[a] - (g - 1))
                                            for a in range(1, v.dim()))]
        pc, fc = core(pv, halo_p), core(fv, halo_f)
        N.wait(self.stream, N.torch_stream())
        N.call("fasmg_engine_load", self.handle, N.ptr(pc), N.strides(pc), N.ptr(fc),
               N.strides(fc))

    def store(self, pv: torch.Tensor, halo_p: int):
        pc = pv[(slice(None),) + tuple(slice(halo_p - 1, pv.shape[a] - (halo_p - 1))
                                        for a in range(1, pv.dim()))]
        N.call("fasmg_engine_store", self.handle, N.ptr(pc), N.strides(pc))
        N.wait(N.torch_stream(), self.stream)

    def sync_halos(self):
        N.call("fasmg_engine_sync_halos", self.handle)

    def launch(self, count: int, with_norm: bool):
        N.call("fasmg_engine_launch", self.handle, int(count), 1 if with_norm else 0)

    def prepare(self, with_norm: bool):
        N.call("fasmg_engine_prepare", self.handle, 1 if with_norm else 0)

    def result(self) -> float:
        out = ctypes.c_double()
        N.call("fasmg_engine_result", self.handle, ctypes.byref(out))
        return out.value

    # the device solve loop (fasmg_engine_solve in halves: every rank is
    # prepared, then launched, then waited on)
    def prepare_solve(self):
        N.call("fasmg_engine_prepare_solve", self.handle)

    _kmax = 0  # k_max of the last solve_launch (the history length bound)

    def solve_launch(self, k_max: int, tol: float, scale: float):
        self._kmax = int(k_max)
        N.call("fasmg_engine_solve_launch", self.handle, int(k_max), float(tol), float(scale))

    def solve_wait(self) -> list:
        if self._kmax < 1:
            raise NativeError("solve_wait without a solve_launch")
        hist = (ctypes.c_double * self._kmax)()
        n = ctypes.c_int(0)
        N.call("fasmg_engine_solve_wait", self.handle, hist, ctypes.byref(n))
        return list(hist[: n.value])

    def synchronize(self):
        N.call("fasmg_stream_synchronize", self.stream)

    def time_sweeps(self, level: int = 0, reps: int = 20) -> float:
        ms = ctypes.c_double()
        N.call("fasmg_engine_time_sweeps", self.handle, int(level), int(reps), ctypes.byref(ms))
        return ms.value

    def close(self):
        if getattr(self, "handle", None) is not None and N._lib is not None:
            N.lib().fasmg_engine_destroy(self.handle)
            self.handle = None
            if self._own_stream:
                N.lib().fasmg_stream_destroy(self.stream)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class VirtualSlabSolver:
    """``parts`` slab engines on one device (separate streams), exchanging
    halos through the same peer-store/counter protocol as real ranks."""

    def __init__(self, hierarchy: GridHierarchy, location: Location, bc: BoundaryCondition,
                 plan: SweepPlan, coeffs: OperatorCoeffs, parts: int, min_planes: int = 4):
        self.hierarchy, self.location, self.bc = hierarchy, location, bc
        self.plan, self.coeffs, self.parts, self.min_planes = plan, coeffs, parts, min_planes
        self._engines = {}
        self._pool = None

    def engines(self, s: int, device: torch.device):
        key = (int(s), device.index)
        es = self._engines.get(key)
        if es is None:
            es = [_SlabEngine(self.hierarchy, self.location, self.bc, self.plan, self.coeffs,
                              s, self.parts, r, device, self.min_planes)
                  for r in range(self.parts)]
            exports = [e.export() for e in es]
            for e in es:
                e.connect(exports)
            self._engines[key] = es
        return es

    def launch_all(self, es, count: int, with_norm: bool):
        """Enqueue every virtual rank's graph from its own host thread: a
        graph launch may block the host once its stream's queue is full,
        and a rank's graph stalls on device until its peers' graphs run --
        launching the ranks one after another from one thread can deadlock
        (observed with 8 ranks at 512^3).  ctypes releases the GIL.
        Every rank's graph is captured first (fasmg_engine_prepare): a
        capture that lazily loads a kernel module waits for the running
        kernels, i.e. for peers already spinning on this rank."""
        for e in es:
            e.prepare(with_norm)
        if self._pool is None:
            import concurrent.futures as cf
            self._pool = cf.ThreadPoolExecutor(max_workers=self.parts)
        futs = [self._pool.submit(e.launch, count, with_norm) for e in es]
        for fu in futs:
            fu.result()

    def _singular(self):
        return self.coeffs.a == 0.0 and all(r.kind != "dirichlet" for _, r in self.bc.faces)

    def _load(self, es, p: Field, f: Field):
        n0 = p.grid.shape[0]
        for e in es:
            e.load(slab_view(p.data, p.halo, n0, self.parts, e.rank),
                   slab_view(f.data, f.halo, n0, self.parts, e.rank), p.halo, f.halo)
        for e in es:
            e.synchronize()
        for e in es:
            e.sync_halos()

    def _store(self, es, p: Field):
        n0 = p.grid.shape[0]
        for e in es:
            v = slab_view(p.data, p.halo, n0, self.parts, e.rank)
            e.store(v, p.halo)

    def vcycle(self, p: Field, f: Field, s: int) -> Field:
        es = self.engines(s, p.device)
        self._load(es, p, f)
        self.launch_all(es, 1, False)
        for e in es:
            e.synchronize()
        self._store(es, p)
        p.ghosts_fresh = False
        return p

    def _views_interior(self, v: torch.Tensor, halo: int, rank: int) -> torch.Tensor:
        g = self.hierarchy.fine
        ea = self.location.edge_axis
        m0 = g.shape[0] // self.parts
        if ea == 0 and rank == self.parts - 1:
            m0 -= 1  # the wall node n
        sl = [slice(1, 1 + m0)]
        for a in range(1, g.dim):
            sl.append(slice(halo, halo + (g.shape[a] - 1 if a == ea else g.shape[a])))
        return v[tuple(sl)]

    def _views_subtract_mean(self, vs, halo: int):
        """``interior -= np.mean(interior)`` over a field held as per-rank
        slab views: chunk sums per slab, totalled in rank/chunk order
        (bitwise numpy's order, as dist_subtract_interior_mean)."""
        g = self.hierarchy.fine
        ea = self.location.edge_axis
        gext = tuple(g.shape[a] - 1 if a == ea else g.shape[a] for a in range(g.dim))
        ivs = [self._views_interior(v, halo, r) for r, v in enumerate(vs)]
        total = ordered_total([slab_chunk_sums(v, gext).cpu() for v in ivs])
        tot = torch.tensor([total], dtype=torch.float64, device=vs[0].device)
        for v in ivs:
            N.call("fasmg_sub_mean", N.ptr(v), N.strides(v), v.dim(), N.ints(v.shape),
                   N.ptr(tot), float(math.prod(gext)), N.torch_stream())

    def _outer_loop(self, es, params: FasParams, scale: float) -> list:
        """The outer loop of FasSolver.solve over the virtual ranks: the
        device loop on every rank (all graphs captured, then all launched,
        then waited on: a rank's loop stalls until its peers run), or the
        host loop (FASMG_DEVICE_LOOP=0, kMax above the device loop's cap, or
        more than 4 ranks: 8 ranks' spinning loops on ONE device outrun its
        hardware queues and stall -- a one-device artefact, real ranks each
        have their own GPU)."""
        from . import fas as _fas
        if _fas._DEVICE_LOOP and 1 <= params.k_max <= 4096 and len(es) <= 4:
            for e in es:
                e.prepare_solve()
            for e in es:
                e.solve_launch(params.k_max, params.tol, scale)
            hists = [e.solve_wait() for e in es]
            if any(h != hists[0] for h in hists):
                raise NativeError(f"ranks disagree on the residual history: {hists}")
            return hists[0]
        history = []
        for _ in range(params.k_max):
            self.launch_all(es, 1, True)
            sums = [e.result() for e in es]
            if any(x != sums[0] for x in sums):
                raise NativeError(f"ranks disagree on the residual: {sums}")
            res = scale * math.sqrt(sums[0])
            history.append(res)
            if res <= params.tol:
                break
        return history

    def solve_views(self, pvs, fvs, params: FasParams, halo_p: int = 1,
                    halo_f: int = 1) -> SolveReport:
        """``solve`` on per-rank slab views (rank cells + 1 ghost plane each
        side along axis 0, as DistSlabSolver.solve takes them): the
        virtual-rank form of the distributed solve, singular mean included.
        Ghost values of the views are left to the caller."""
        singular = self._singular()
        if singular:
            self._views_subtract_mean(fvs, halo_f)
        es = self.engines(params.s, pvs[0].device)
        for e, pv, fv in zip(es, pvs, fvs):
            e.load(pv, fv, halo_p, halo_f)
        for e in es:
            e.synchronize()
        for e in es:
            e.sync_halos()
        g = self.hierarchy.fine
        scale = g.h ** (g.dim / 2.0)
        history = self._outer_loop(es, params, scale)
        for e, pv in zip(es, pvs):
            e.store(pv, halo_p)
        if singular:
            self._views_subtract_mean(pvs, halo_p)
        return SolveReport(len(history), history, bool(history and history[-1] <= params.tol))

    def solve(self, p: Field, f: Field, params: FasParams) -> SolveReport:
        singular = self._singular()
        if singular:
            subtract_interior_mean(f)
        es = self.engines(params.s, p.device)
        self._load(es, p, f)
        g = self.hierarchy.fine
        scale = g.h ** (g.dim / 2.0)
        history = self._outer_loop(es, params, scale)
        self._store(es, p)
        fill_ghosts(p, self.bc)
        if singular:
            subtract_interior_mean(p)
            p.ghosts_fresh = False
        return SolveReport(len(history), history, bool(history and history[-1] <= params.tol))


def ordered_total(gathered) -> float:
    """Sequential sum, in chunk order, of every rank's chunk sums gathered in
    rank order (axis-0 slabs are contiguous runs of the C-order chunk list):
    the same adds, in the same order, as numpy's buffered reduction of the
    whole view (SURVEY.md section 8e item v)."""
    acc = 0.0
    for part in gathered:
        for x in part.tolist():
            acc += x
    return acc


def slab_chunk_sums(v: torch.Tensor, global_ext) -> torch.Tensor:
    """Per-chunk sums (numpy's chunk length for the whole view of extent
    ``global_ext``) of this rank's axis-0 slab ``v`` of an interior view."""
    dim = v.dim()
    gext = N.ints(global_ext)
    B = int(N.lib().fasmg_view_chunk_len(dim, gext))
    nch = (v.numel() + B - 1) // B
    scratch = torch.empty(max(v.numel(), 1), dtype=torch.float64, device=v.device)
    sums = torch.empty(max(nch, 1), dtype=torch.float64, device=v.device)
    N.call("fasmg_view_chunk_sums", N.ptr(v), N.strides(v), dim, N.ints(v.shape), gext,
           N.ptr(scratch), N.ptr(sums), N.torch_stream())
    return sums[:nch]


def dist_subtract_interior_mean(v: torch.Tensor, global_ext, group=None) -> float:
    """``interior -= np.mean(interior)`` over a field split into axis-0
    slabs (PKG/fas.py:145,156 on a decomposed field): ``v`` is this rank's
    slab of the interior view of extent ``global_ext``.  The chunk sums are
    all-gathered in rank order (NCCL on device tensors; gloo through host
    copies) and totalled in chunk order, so the result is bitwise the
    single-array ``subtract_interior_mean``.  Returns the mean."""
    import torch.distributed as dist
    sums = slab_chunk_sums(v, global_ext)
    world = dist.get_world_size(group)
    src = sums if dist.get_backend(group) == "nccl" else sums.cpu()
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src, group=group)
    total = ordered_total([o.cpu() for o in out])
    count = float(math.prod(global_ext))
    tot = torch.tensor([total], dtype=torch.float64, device=v.device)
    N.call("fasmg_sub_mean", N.ptr(v), N.strides(v), v.dim(), N.ints(v.shape), N.ptr(tot),
           count, N.torch_stream())
    return total / count


def exchange_ipc(engine_exports, handle_of, open_handle, all_gather_object, rank, world):
    """Turn this rank's exported device pointers into every rank's pointers
    valid in this process: export CUDA-IPC handles, all-gather them,
    open the peers'.  The callables are injected so the host-side protocol
    is testable without GPUs (tests/test_slab_cpu.py)."""
    mine = [handle_of(ptr) for ptr in engine_exports]
    gathered = [None] * world
    all_gather_object(gathered, mine)
    out = []
    for r in range(world):
        if r == rank:
            out.append(list(engine_exports))
        else:
            out.append([open_handle(hd) for hd in gathered[r]])
    return out


class DistSlabSolver:
    """One process per GPU: rank ``rank`` of ``world`` owns its slab; the
    caller passes rank-local slab views (its cells plus one ghost plane on
    each side along axis 0) of the global p and f."""

    def __init__(self, hierarchy: GridHierarchy, location: Location, bc: BoundaryCondition,
                 plan: SweepPlan, coeffs: OperatorCoeffs, s: int, device: torch.device,
                 group=None, min_planes: int = 4):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.hierarchy, self.bc, self.coeffs, self.location = hierarchy, bc, coeffs, location
        self.engine = _SlabEngine(hierarchy, location, bc, plan, coeffs, s, self.world,
                                  self.rank, device, min_planes)
        self._opened = []

        def handle_of(ptr):
            if not ptr:  # arrays a cell-centred engine does not allocate
                return None
            buf = ctypes.create_string_buffer(64)
            N.check(N.lib().fasmg_ipc_get_handle(ctypes.c_void_p(ptr), buf))
            return buf.raw

        def open_handle(hd):
            if hd is None:
                return 0
            out = ctypes.c_void_p()
            N.check(N.lib().fasmg_ipc_open_handle(hd, ctypes.byref(out)))
            self._opened.append(out.value)
            return out.value

        with torch.cuda.device(device):
            ptrs = exchange_ipc(self.engine.export(), handle_of, open_handle,
                                lambda out, obj: dist.all_gather_object(out, obj, group=group),
                                self.rank, self.world)
        self.engine.connect(ptrs)
        dist.barrier(group=group)

    def load(self, pv: torch.Tensor, fv: torch.Tensor, halo_p: int = 1, halo_f: int = 1):
        self.engine.load(pv, fv, halo_p, halo_f)
        self.engine.synchronize()
        self.dist.barrier(group=self.group)
        self.engine.sync_halos()

    def run(self, count: int = 1) -> float:
        """``count`` V-cycles, each followed by the global residual norm."""
        for _ in range(count):
            self.engine.launch(1, True)
        sumsq = self.engine.result()
        g = self.hierarchy.fine
        return g.h ** (g.dim / 2.0) * math.sqrt(sumsq)

    def solve_loop(self, k_max: int, tol: float) -> list:
        """Up to k_max V-cycles + global norms in one device-loop launch per
        rank (every rank captured first, then a barrier: no rank's loop runs
        while a peer still captures); all ranks stop together."""
        g = self.hierarchy.fine
        self.engine.prepare_solve()
        self.dist.barrier(group=self.group)
        self.engine.solve_launch(k_max, tol, g.h ** (g.dim / 2.0))
        return self.engine.solve_wait()

    def solve_loaded(self, params: FasParams) -> SolveReport:
        from . import fas as _fas
        if _fas._DEVICE_LOOP and 1 <= params.k_max <= 4096:
            history = self.solve_loop(params.k_max, params.tol)
        else:
            history = []
            for _ in range(params.k_max):
                res = self.run(1)
                history.append(res)
                if res <= params.tol:
                    break
        return SolveReport(len(history), history, bool(history and history[-1] <= params.tol))

    def store(self, pv: torch.Tensor, halo_p: int = 1):
        self.engine.store(pv, halo_p)

    def _singular(self) -> bool:
        return self.coeffs.a == 0.0 and all(r.kind != "dirichlet" for _, r in self.bc.faces)

    def _interior(self, v: torch.Tensor, halo: int) -> torch.Tensor:
        """This rank's rows of the interior view, from its slab view."""
        g = self.hierarchy.fine
        ea = self.location.edge_axis
        m0 = 2 * self.engine.planes
        if ea == 0 and self.rank == self.world - 1:
            m0 -= 1  # the wall node n
        sl = [slice(1, 1 + m0)]
        for a in range(1, g.dim):
            m = g.shape[a] - 1 if a == ea else g.shape[a]
            sl.append(slice(halo, halo + m))  # core 1 sits at data index halo
        return v[tuple(sl)]

    def solve(self, pv: torch.Tensor, fv: torch.Tensor, params: FasParams, halo_p: int = 1,
              halo_f: int = 1) -> SolveReport:
        """FasSolver.solve on this rank's slab views (PKG/fas.py:137-162): for a
        singular problem f is shifted to zero mean in place first and p after,
        with the distributed ordered mean; the slab's ghost values are left
        to the caller (``ghosts_fresh`` False in the reference)."""
        g = self.hierarchy.fine
        gext = tuple(g.shape[a] - 1 if a == self.location.edge_axis else g.shape[a]
                     for a in range(g.dim))
        singular = self._singular()
        if singular:
            dist_subtract_interior_mean(self._interior(fv, halo_f), gext, self.group)
        self.load(pv, fv, halo_p, halo_f)
        rep = self.solve_loaded(params)
        self.store(pv, halo_p)
        if singular:
            dist_subtract_interior_mean(self._interior(pv, halo_p), gext, self.group)
        return rep

    def close(self):
        for ptr in self._opened:
            N.lib().fasmg_ipc_close_handle(ctypes.c_void_p(ptr))
        self._opened = []
        self.engine.close()
