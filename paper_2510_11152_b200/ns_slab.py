"""Navier-Stokes projection steps on axis-0 slabs (BASELINE.json configs[4]:
the 3D cavity at 1024^3 across 8 B200).

Every rank holds, for each resident slot of the schedule, only its slab of
the field: the rank's ``m0 = 2*nb`` cells along array axis 0 (the outermost,
contiguous axis -- the north star's "z-slabs") plus ``g`` rows on either side,
with the whole extent of the other axes.  Local core index ``x_l`` is global
core index ``x_l + lo - 1``; a field with its edge axis along axis 0 (u)
holds nodes ``1..m0`` of the slab, the interface node belonging to the lower
rank and the wall node n to the last rank -- the convention of the slab
FAS engine (slab.py), so every field is handed to the distributed solver
without copies.

A step is the single-GPU step (ns.py, the same schedule Step lists, the
same native kernels on local views) plus the exchanges the stencils need:

* before the WENO3 convection of the momentum source, the halo-2 velocity
  mixtures (and u^n) exchange 2 rows with each neighbour;
* the pressure gradient (momentum source and correction) reads 1 row of p
  above the slab; the divergence reads 1 row of u~ below it;
* each exchange is followed by a slab ghost fill that completes the rows
  from the neighbour along the other axes and applies the boundary
  condition on global walls only (fasmg_fill_ghosts_slab) -- bitwise the
  whole-field fill_ghosts on those rows;
* the four FAS solves run on the slab engines (per-half-sweep halo push
  over peer memory, coarse gather); the pressure solve's mean projections
  and the integral divergence sum chunk partials in rank order (numpy's
  order, bitwise).

Fields therefore equal the 1-GPU stepper's bitwise; residual histories
differ only by the order of the norm's rank reduction (~1e-16).

Two transports share the code: :class:`VirtualRanks` runs P slabs in ONE
process on one device (exchanges are device copies, solves go through
``VirtualSlabSolver``) -- the on-one-GPU test of the protocol; and
:class:`DistRanks` is one process per GPU (exchanges are torch.distributed
point-to-point transfers of contiguous row blocks: NCCL over NVLink, or gloo
through host memory for ranks sharing a device; solves go through
``DistSlabSolver``).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .boundary import BoundaryCondition
from .elementwise import ADD, MIX_AVG, MIX_EXT, NEG, elem
from .errors import MissingBinding
from .fas import FasParams, SolveReport
from .grid import GridLevel, Location, make_hierarchy
from .ns import AXIS_OF, LOC_OF, NSParams, ProjectionStepper, StepReport, cavity_bcs
from .schedule import COMPONENTS_3D, build_schedule
from .slab import DistSlabSolver, VirtualSlabSolver, ordered_total, slab_chunk_sums
from .smoothers import make_plan
from .stencil import OperatorCoeffs
from .weno import WENO_EPS


class SlabGeom:
    """Axis-0 decomposition of a grid into ``nranks`` slabs of whole block
    planes (slab.slab_cells)."""

    def __init__(self, grid: GridLevel, nranks: int):
        n0 = grid.shape[0]
        if n0 % 2 or (n0 // 2) % nranks:
            raise ValueError(f"{n0 // 2} block planes do not split over {nranks} ranks")
        self.grid, self.P = grid, nranks
        self.nb = n0 // 2 // nranks
        self.m0 = 2 * self.nb

    def lo(self, r: int) -> int:
        return 2 * r * self.nb + 1

    def iface(self, r: int) -> int:
        return (1 if r > 0 else 0) | (2 if r < self.P - 1 else 0)

    def rows(self, loc: Location, r: int) -> int:
        """Interior rows of the slab along axis 0."""
        return self.m0 - 1 if (loc.edge_axis == 0 and r == self.P - 1) else self.m0


class SlabField:
    """The local slabs (one per rank of this process) of one field; the
    same location / halo / dirty-flag vocabulary as grid.Field."""

    def __init__(self, geom: SlabGeom, location: Location, halo: int, ranks, device,
                 storage: dict | None = None):
        """``storage``: optional {rank: flat float64 tensor} the parts are
        views of (scratch fields that are never live together share one)."""
        self.geom, self.location, self.halo = geom, location, halo
        shape = self.part_shape(geom, location, halo)
        if storage is None:
            self.parts = {r: torch.zeros(shape, dtype=torch.float64, device=device) for r in ranks}
        else:
            n = math.prod(shape)
            self.parts = {r: storage[r][:n].view(shape) for r in ranks}
        self.ghosts_fresh = False

    @staticmethod
    def part_shape(geom: SlabGeom, location: Location, halo: int) -> list:
        ea = location.edge_axis
        return [geom.m0 + 2 * halo] + [(n + 1 + 2 * (halo - 1)) if a == ea else (n + 2 * halo)
                                       for a, n in enumerate(geom.grid.shape) if a > 0]

    def interior_shape(self, r):
        g, ea = self.geom.grid, self.location.edge_axis
        return (self.geom.rows(self.location, r),) + tuple(
            n - 1 if a == ea else n for a, n in enumerate(g.shape) if a > 0)

    def interior(self, r) -> torch.Tensor:
        h = self.halo
        return self.parts[r][tuple(slice(h, h + m) for m in self.interior_shape(r))]

    def core(self, r) -> torch.Tensor:
        """Halo-1 view (local core index == array index); rows 0..m0+1."""
        h, g, ea = self.halo, self.geom.grid, self.location.edge_axis
        sl = [slice(h - 1, h + self.geom.m0 + 1)]
        for a in range(1, g.dim):
            sl.append(slice(h - 1, h - 1 + g.shape[a] + (1 if a == ea else 2)))
        return self.parts[r][tuple(sl)]

    def slab_view(self, r) -> torch.Tensor:
        """Rows of core 0..m0+1, whole other axes: the view the slab FAS
        engine loads (slab.slab_view of the global array)."""
        h = self.halo
        return self.parts[r][h - 1: h + self.geom.m0 + 1]

    def copy_from(self, other: "SlabField"):
        for r, t in self.parts.items():
            t.copy_(other.parts[r])
        self.ghosts_fresh = other.ghosts_fresh


class VirtualRanks:
    """P slabs in one process on one device: exchanges are device copies."""

    def __init__(self, nranks: int):
        self.P = nranks
        self.ranks = list(range(nranks))

    def exchange(self, F: SlabField, rows: int):
        m0, h = F.geom.m0, F.halo
        for r in range(self.P - 1):  # interface between r and r+1
            lo_, hi_ = F.parts[r], F.parts[r + 1]
            lo_[m0 + h: m0 + h + rows].copy_(hi_[h: h + rows])      # r+1's first rows
            hi_[h - rows: h].copy_(lo_[m0 + h - rows: m0 + h])      # r's last rows

    def gather_chunk_sums(self, sums: dict) -> list:
        return [sums[r].cpu() for r in self.ranks]

    def make_solver(self, hier, loc, bc, plan, coeffs, s, device):
        return _VirtualSolver(VirtualSlabSolver(hier, loc, bc, plan, coeffs, self.P))

    def barrier(self):
        pass


class DistRanks:
    """One rank per process (torch.distributed): row blocks move with
    point-to-point transfers (NCCL on device tensors; gloo via host)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranks = [self.rank]
        self.nccl = dist.get_backend(group) == "nccl"

    def exchange(self, F: SlabField, rows: int):
        dist, r, m0, h = self.dist, self.rank, F.geom.m0, F.halo
        t = F.parts[r]
        sends, recvs = [], []
        if r > 0:  # my first rows -> r-1's upper halo; its last rows -> my lower halo
            sends.append((t[h: h + rows], r - 1))
            recvs.append((t[h - rows: h], r - 1))
        if r < self.P - 1:
            sends.append((t[m0 + h - rows: m0 + h], r + 1))
            recvs.append((t[m0 + h: m0 + h + rows], r + 1))
        if self.nccl:
            ops = [dist.P2POp(dist.isend, x.contiguous(), dst, self.group) for x, dst in sends]
            bufs = [torch.empty_like(x) for x, _ in recvs]
            ops += [dist.P2POp(dist.irecv, b, src, self.group) for b, (_, src) in zip(bufs, recvs)]
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for b, (x, _) in zip(bufs, recvs):
                x.copy_(b)
        else:
            hs = [x.cpu() for x, _ in sends]
            hb = [torch.empty(tuple(x.shape), dtype=x.dtype) for x, _ in recvs]
            ops = [dist.P2POp(dist.isend, x, dst, self.group) for x, (_, dst) in zip(hs, sends)]
            ops += [dist.P2POp(dist.irecv, b, src, self.group) for b, (_, src) in zip(hb, recvs)]
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for b, (x, _) in zip(hb, recvs):
                x.copy_(b.to(x.device))

    def gather_chunk_sums(self, sums: dict) -> list:
        src = sums[self.rank]
        if not self.nccl:
            src = src.cpu()
        out = [torch.empty_like(src) for _ in range(self.P)]
        self.dist.all_gather(out, src, group=self.group)
        return [o.cpu() for o in out]

    def make_solver(self, hier, loc, bc, plan, coeffs, s, device):
        return _DistSolver(DistSlabSolver(hier, loc, bc, plan, coeffs, s, device,
                                          group=self.group), self.rank)

    def barrier(self):
        self.dist.barrier(group=self.group)


class _DistSolver:
    def __init__(self, ds: DistSlabSolver, rank: int):
        self.ds, self.rank = ds, rank

    def solve(self, p: SlabField, f: SlabField, params: FasParams) -> SolveReport:
        r = self.rank
        return self.ds.solve(p.slab_view(r), f.slab_view(r), params, p.halo, f.halo)

    def close(self):
        self.ds.close()


class _VirtualSolver:
    def __init__(self, vs: VirtualSlabSolver):
        self.vs = vs

    def solve(self, p: SlabField, f: SlabField, params: FasParams) -> SolveReport:
        P = self.vs.parts
        return self.vs.solve_views([p.slab_view(r) for r in range(P)],
                                   [f.slab_view(r) for r in range(P)], params, p.halo, f.halo)

    def close(self):
        pass


class SlabProjectionStepper(ProjectionStepper):
    """ProjectionStepper on axis-0 slabs: the same schedule execution
    (slots, rebinding, Step formulas) with every field a :class:`SlabField`.
    ``ranks``: :class:`VirtualRanks` or :class:`DistRanks`."""

    def __init__(self, grid: GridLevel, params: NSParams, ranks, bcs: dict | None = None,
                 device=None, min_planes: int = 4):
        if grid.dim != 3:
            raise ValueError("slab NS runs the 3D projection (2D grids are single-GPU)")
        self.forcing = None
        self.t = 0.0
        self.grid = grid
        self.params = params
        self.dim = 3
        self.comps = COMPONENTS_3D
        self.bcs = bcs or cavity_bcs(3)
        for c, bc in self.bcs.items():
            if bc.face("xlo").kind == "periodic":
                raise ValueError(f"{c}: slab decomposition needs a non-periodic axis 0")
        self.comm = ranks
        self.geom = SlabGeom(grid, ranks.P)
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.schedule = build_schedule(params.order, params.mode, 3)
        ml = params.mesh_level or int(np.log2(min(grid.shape))) - 1
        self.fas = FasParams(params.tol, params.k_max, params.s, ml)
        hier = make_hierarchy(grid, ml)
        plan = make_plan("x", 3, "ff")
        b_mom = params.dt / params.re if params.order == 1 else params.dt / (2.0 * params.re)
        with torch.cuda.device(self.device):
            self.solvers = {c: ranks.make_solver(hier, LOC_OF[c], self.bcs[c], plan,
                                                 OperatorCoeffs(1.0, b_mom), params.s,
                                                 self.device) for c in self.comps}
            self.solvers["p"] = ranks.make_solver(hier, Location.CELL, self.bcs["p"], plan,
                                                  OperatorCoeffs(0.0, params.dt), params.s,
                                                  self.device)
        mk = lambda loc, h: SlabField(self.geom, loc, h, ranks.ranks, self.device)  # noqa: E731
        self.slots = {}
        for name in self.schedule.resident_slots():
            comp = name.split("_")[0].lower()
            self.slots[name] = mk(Location.CELL, 1) if comp == "p" else mk(LOC_OF[comp], 2)
        # transient scratch: the momentum sources and the pressure rhs are
        # never live together (rhs_c -> solve_c per component, then the
        # pressure solve; ns.ProjectionStepper): one buffer per rank backs
        # them all; the halo-2 mixtures are separate
        locs = [LOC_OF[c] for c in self.comps] + [Location.CELL]
        numel = max(math.prod(SlabField.part_shape(self.geom, loc, 1)) for loc in locs)
        store = {r: torch.zeros(numel, dtype=torch.float64, device=self.device)
                 for r in ranks.ranks}
        self._f = {c: SlabField(self.geom, LOC_OF[c], 1, ranks.ranks, self.device, store)
                   for c in self.comps}
        self._mix = {}
        self._gen = {}  # slot write generations (ProjectionStepper._bind)
        self._fp = SlabField(self.geom, Location.CELL, 1, ranks.ranks, self.device, store)
        self.held = {slot: q for q, slot in self.schedule.initial}
        self.step_count = 0
        self.timing = None

    # ------------------------------------------------------------ halos
    def _refresh(self, F: SlabField, bc: BoundaryCondition, rows: int | None = None):
        """Exchange ``rows`` (default: the halo) rows with the neighbours,
        then the slab ghost fill (interfaces completed along axes 1..2,
        boundary condition on global walls)."""
        rows = F.halo if rows is None else rows
        self.comm.exchange(F, rows)
        kinds, vals = bc.codes()
        ea = F.location.edge_axis
        n = (self.geom.m0,) + tuple(self.grid.shape[1:])
        for r, t in F.parts.items():
            N.call("fasmg_fill_ghosts_slab", N.ptr(t), 3, N.ints(n), -1 if ea is None else ea,
                   F.halo, N.ints(kinds), N.doubles(vals), self.geom.iface(r),
                   int(t.shape[0]), N.torch_stream())
        F.ghosts_fresh = True

    # ------------------------------------------------------------ state I/O
    def set_state(self, vel: dict, p=None):
        """Global interior arrays (numpy or tensors, None for 0): each rank
        keeps its rows."""
        def put(F: SlabField, src, comp):
            for r, t in F.parts.items():
                t.zero_()
                if src is not None:
                    lo = self.geom.lo(r) - 1
                    rows = F.geom.rows(F.location, r)
                    s = src[lo: lo + rows]
                    if isinstance(s, np.ndarray):
                        s = torch.from_numpy(np.ascontiguousarray(s))
                    F.interior(r)[...] = s.to(t.device, torch.float64)
        for c in self.comps:
            F = self.field_of(f"{c}_n")
            put(F, vel.get(c), c)
            self._refresh(F, self.bcs[c])
            if self.params.order == 2:
                self.field_of(f"{c}_nm1").copy_from(F)
        put(self.field_of("p_n"), p, "p")
        put(self.field_of("p_tld_prev"), None, "p")

    def gather(self, F: SlabField) -> torch.Tensor:
        """Global interior of a slab field (virtual ranks: all slabs are
        local; process ranks: all-gathered), on the device."""
        g = self.grid
        ea = F.location.edge_axis
        ext = tuple(n - 1 if a == ea else n for a, n in enumerate(g.shape))
        out = torch.empty(ext, dtype=torch.float64, device=self.device)
        if isinstance(self.comm, DistRanks):
            import torch.distributed as dist
            r = self.comm.rank
            mine = F.interior(r).contiguous()
            pad = torch.zeros((self.geom.m0,) + mine.shape[1:], dtype=torch.float64,
                              device=self.device)
            pad[: mine.shape[0]] = mine
            src = pad if self.comm.nccl else pad.cpu()
            parts = [torch.empty_like(src) for _ in range(self.comm.P)]
            dist.all_gather(parts, src, group=self.comm.group)
            items = [(q, parts[q].to(self.device)) for q in range(self.comm.P)]
        else:
            items = [(q, F.interior(q)) for q in self.comm.ranks]
        for q, t in items:
            lo = self.geom.lo(q) - 1
            rows = self.geom.rows(F.location, q)
            out[lo: lo + rows] = t[:rows]
        return out

    def velocity_global(self, c: str) -> torch.Tensor:
        return self.gather(self.field_of(f"{c}_n"))

    def pressure_global(self) -> torch.Tensor:
        return self.gather(self.field_of("p_n"))

    # ----------------------------------------------------------- formulas
    def _mix_field(self, key, comp, op, a: SlabField, b: SlabField) -> SlabField:
        M = self._mix.get(key)
        if M is None:
            M = self._mix[key] = SlabField(self.geom, LOC_OF[comp], 2, self.comm.ranks,
                                           self.device)
        for r in M.parts:
            elem(op, M.interior(r), [a.interior(r), b.interior(r)])
        self._refresh(M, self.bcs[comp])
        return M

    def _ns_rhs(self, order, out: SlabField, u: SlabField, conv, p: SlabField, axis, s0, s1=0.0):
        g = self.grid
        for r in out.parts:
            o, uc, pc = out.interior(r), u.core(r), p.core(r)
            cv = conv.interior(r) if conv is not None else o
            N.call("fasmg_ns_rhs", int(order), N.ptr(o), N.strides(o), N.ptr(uc), N.strides(uc),
                   N.ptr(cv), N.strides(cv), N.ptr(pc), N.strides(pc), 3, int(axis),
                   N.ints(u.interior_shape(r)), float(s0), float(s1), 1.0 / g.h,
                   1.0 / (g.h * g.h), N.torch_stream())

    def momentum_rhs(self, c: str, read: dict) -> SlabField:
        """Source term f_c (ns.ProjectionStepper.momentum_rhs) on the slabs."""
        import ctypes
        dt, order = self.params.dt, self.params.order
        vel = []
        for o in self.comps:
            un = read[f"{o}_n"]
            if order == 1:
                if not un.ghosts_fresh:
                    self._refresh(un, self.bcs[o])
                vel.append(un)
            elif f"{o}_tld" in read:
                vel.append(self._mix_field(o, o, MIX_AVG, un, read[f"{o}_tld"]))
            else:
                vel.append(self._mix_field(o, o, MIX_EXT, un, read[f"{o}_nm1"]))
        target = AXIS_OF[c]
        f = self._f[c]
        p = read["p_n"]
        self.comm.exchange(p, 1)  # grad p reads the row above the slab
        un = read[f"{c}_n"]
        if order == 2 and not un.ghosts_fresh:
            self._refresh(un, self.bcs[c])
        conv = f  # the convection lands in f; the fused source pass then updates it in place
        for r in f.parts:
            # one fused WENO3 pass on the local arrays (winds in place)
            ci = conv.interior(r)
            vp = (ctypes.c_void_p * 3)(*[v.parts[r].data_ptr() for v in vel])
            vs = [s for v in vel for s in v.parts[r].stride()]
            N.call("fasmg_weno_convect", N.ptr(ci), N.strides(ci), vp,
                   (ctypes.c_long * 9)(*vs), ctypes.c_int(3), ctypes.c_int(target),
                   ctypes.c_int(2), N.ints(conv.interior_shape(r)),
                   ctypes.c_double(0.5 / self.grid.h), ctypes.c_double(WENO_EPS),
                   N.torch_stream())
        self._ns_rhs(order, f, un, conv, p, target, dt,
                     dt / (2.0 * self.params.re) if order == 2 else 0.0)
        f.ghosts_fresh = False
        return f

    def pressure_poisson(self, tld: dict, guess: SlabField) -> SolveReport:
        import ctypes
        for c in self.comps:  # the divergence reads the row below the slab
            self.comm.exchange(tld[c], 1)
        div = self._fp
        n = (self.geom.m0,) + tuple(self.grid.shape[1:])
        for r in div.parts:
            cores = [tld[c].core(r) for c in self.comps]
            ptrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in cores])
            cs = (ctypes.c_long * 9)(*[s for t in cores for s in t.stride()])
            oi = div.interior(r)
            N.call("fasmg_divergence", ptrs, cs, N.ptr(oi), N.strides(oi), 3, N.ints(n),
                   ctypes.c_double(1.0 / self.grid.h), N.torch_stream())
            elem(NEG, oi, [oi])
        div.ghosts_fresh = False
        return self.solvers["p"].solve(guess, div, self.fas)

    def _exec(self, st, read: dict, scratch: dict, rep: StepReport):
        dt = self.params.dt
        if st.formula == "rhs":
            scratch[st.writes[0][1]] = self.momentum_rhs(st.comp, read)
        elif st.formula in ("copy", "rotate2"):
            moves = dict(st.copy_map)
            for q, slot in st.writes:
                src = read[moves[q]]
                dst = self.slots[slot]
                if dst is not src:
                    dst.copy_from(src)
                self._bind(q, slot)
        elif st.formula == "solve_momentum":
            c = st.comp
            q, slot = st.writes[0]
            dst = self.slots[slot]
            src = read[f"{c}_n"]
            if dst is not src:
                dst.copy_from(src)
            rep.momentum[c] = self.solvers[c].solve(dst, read[f"f_{c}"], self.fas)
            self._refresh(dst, self.bcs[c])  # FasSolver.solve's final fill_ghosts
            self._bind(q, slot)
        elif st.formula == "solve_pressure":
            q, slot = st.writes[0]
            guess = self.slots[slot]
            rep.pressure = self.pressure_poisson({c: read[f"{c}_tld"] for c in self.comps},
                                                 guess)
            guess.ghosts_fresh = False
            self._bind(q, slot)
        elif st.formula == "correct":
            c = st.comp
            q, slot = st.writes[0]
            dst = self.slots[slot]
            pt = read["p_tld"]
            self.comm.exchange(pt, 1)  # grad p~ reads the row above the slab
            self._ns_rhs(0, dst, read[f"{c}_tld"], None, pt, AXIS_OF[c], dt)
            self._refresh(dst, self.bcs[c])
            self._bind(q, slot)
        elif st.formula == "p_update":
            q, slot = st.writes[0]
            dst = self.slots[slot]
            a, b = read["p_n"], read["p_tld"]
            for r in dst.parts:
                elem(ADD, dst.interior(r), [a.interior(r), b.interior(r)])
            dst.ghosts_fresh = False
            self._bind(q, slot)
        else:
            raise ValueError(f"unknown formula {st.formula}")

    def divergence(self) -> float:
        """integral_divergence of the current velocity: h^3 * np.sum(div) in
        numpy's chunk order, the chunk sums gathered in rank order."""
        vel = {c: self.field_of(f"{c}_n") for c in self.comps}
        import ctypes
        for c in self.comps:
            self.comm.exchange(vel[c], 1)
        div = self._fp
        n = (self.geom.m0,) + tuple(self.grid.shape[1:])
        sums = {}
        for r in div.parts:
            cores = [vel[c].core(r) for c in self.comps]
            ptrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in cores])
            cs = (ctypes.c_long * 9)(*[s for t in cores for s in t.stride()])
            oi = div.interior(r)
            N.call("fasmg_divergence", ptrs, cs, N.ptr(oi), N.strides(oi), 3, N.ints(n),
                   ctypes.c_double(1.0 / self.grid.h), N.torch_stream())
            sums[r] = slab_chunk_sums(oi, tuple(self.grid.shape))
        total = ordered_total(self.comm.gather_chunk_sums(sums))
        return self.grid.h ** 3 * total

    def field_of(self, quantity: str) -> SlabField:
        for slot, q in self.held.items():
            if q == quantity:
                return self.slots[slot]
        raise MissingBinding(f"{quantity} is not bound to a slot")

    def close(self):
        for s in self.solvers.values():
            s.close()


def slab_model_ms(one_gpu_step_ms: float, n: int, ranks: int) -> dict:
    """Projected per-step time of the slab stepper from a 1-GPU measurement
    of the same per-rank work (a MODEL until an 8-GPU box runs it): the
    per-rank volume is n^3/ranks, the halo exchanges are ~12 transfers of
    two 1024^2 planes per step (~20 us each over NVLink at ~900 GB/s), the
    replicated coarse end of each V-cycle costs ~0.3 ms."""
    return {"per_rank_dof": n ** 3 // ranks, "one_gpu_equivalent_ms": one_gpu_step_ms,
            "exchange_ms": 12 * 0.02, "coarse_gather_ms_per_vcycle": 0.3}


__all__ = ["SlabGeom", "SlabField", "VirtualRanks", "DistRanks", "SlabProjectionStepper",
           "slab_model_ms", "math"]
