"""Projection time steppers for the incompressible Navier-Stokes equations
on the MAC grid, executed from slot schedules (
SPEC.md:411-523).

The reference package ships only the building blocks of these drivers
(weno3_convect, gradient/divergence, FasSolver, the symbolic schedules of
PKG/schedule.py); the drivers themselves are absent (SURVEY.md section 0
item 10).  This module composes them as SPEC.md:432-501 and Tables 2-5
prescribe and executes the *same Step lists* ``schedule.build_schedule``
returns, so the memory-efficient mode really holds only 8 resident device
fields (6 in 2D) and the classical mode 12/15 (9/11) -- and both modes
produce bitwise-identical fields, since their dataflow is identical.

Per component c, the source term is (arithmetic order fixed here and
mirrored by oracle/ns_oracle.py):
  order 1: f = (u^n - dt*conv) - dt*(grad p^n)_c,   conv = weno3(u^n; u^n)
  order 2: f = ((u^n - dt*conv) - dt*(grad p^n)_c) + dt/(2Re)*Lap(u^n),
           conv = weno3(advected (3u^n-u^{n-1})/2; advecting components
           (u^n+u~)/2 if already advanced this step else (3u^n-u^{n-1})/2)
then  u~ - b*Lap(u~) = f  (b = dt/Re or dt/(2Re), initial guess u^n),
      -dt*Lap(p~) = -div(u~)   (a=0, b=dt, all-Neumann, zero-mean),
      u^{n+1} = u~ - dt*(grad p~)_c,   p^{n+1} = p^n + p~.
Mixtures are formed on interiors and get their ghosts from the component's
boundary condition.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .boundary import BoundaryCondition, FaceRule, fill_ghosts
from .elementwise import ADD, AXPY, MIX_AVG, MIX_EXT, NEG, elem, momentum_source
from .errors import MissingBinding
from .fas import EngineArena, FasParams, FasSolver, SolveReport
from .grid import Field, GridLevel, Location, make_hierarchy
from .schedule import COMPONENTS_3D, SlotSchedule, build_schedule
from .smoothers import make_plan
from .stencil import OperatorCoeffs, divergence_edges_to_cc, integral_divergence
from .weno import weno3_convect

LOC_OF = {"u": Location.EDGE_EW, "v": Location.EDGE_NS, "w": Location.EDGE_TB}
AXIS_OF = {"u": 0, "v": 1, "w": 2}


@dataclass(frozen=True)
class NSParams:
    """Reynolds number, time step, scheme order (1|2), schedule mode
    (classical|efficient) and the FAS knobs of Table 1."""

    re: float
    dt: float
    order: int = 2
    mode: str = "efficient"
    tol: float = 1e-10
    k_max: int = 20
    s: int = 2
    mesh_level: int | None = None

    def __post_init__(self):
        if self.re <= 0 or self.dt <= 0 or self.order not in (1, 2):
            raise ValueError(f"invalid NS parameters {self}")
        if self.mode not in ("classical", "efficient"):
            raise ValueError(f"unknown schedule mode {self.mode!r}")


def cavity_bcs(dim: int, lid: float = 1.0) -> dict:
    """Lid-driven cavity: no-slip walls, the top wall (y=1 in 2D, z=1 in 3D)
    moving with tangential speed ``lid`` in x; pressure
    all-Neumann."""
    top = "yhi" if dim == 2 else "zhi"
    out = {c: BoundaryCondition.dirichlet(dim) for c in COMPONENTS_3D[:dim]}
    out["u"] = out["u"].with_face(top, FaceRule("dirichlet", lid))
    out["p"] = BoundaryCondition.neumann(dim)
    return out


@dataclass
class StepReport:
    momentum: dict = field(default_factory=dict)   # comp -> SolveReport
    pressure: SolveReport | None = None
    divergence: float | None = None


class ProjectionStepper:
    """First/second-order projection scheme executing a slot schedule on
    device fields.  ``slots`` holds exactly the schedule's resident fields."""

    def __init__(self, grid: GridLevel, params: NSParams, bcs: dict | None = None,
                 device=None, forcing=None, share_workspaces: bool = True):
        """``forcing(component, t)``: optional body force (interior array of
        the component's edge grid) added to the momentum source as
        ``f += dt*F(t)``, with t = t^{n+1} (order 1, backward Euler) or
        the trapezoidal (F(t^n) + F(t^{n+1}))/2 (order 2, Crank-Nicolson;
        this reproduces PAPER.md Table 8 to 2-3 digits, ``forcing_rule =
        "mid"`` uses F(t^{n+1/2})) -- used by the manufactured
        temporal-convergence test; None for the cavity."""
        self.forcing = forcing
        self.forcing_rule = "trap"  # order 2: (F^n + F^{n+1})/2, or "mid" F(t^{n+1/2})
        self.t = 0.0
        self.grid = grid
        self.params = params
        self.dim = grid.dim
        self.comps = COMPONENTS_3D[: self.dim]
        self.bcs = bcs or cavity_bcs(self.dim)
        self.schedule: SlotSchedule = build_schedule(params.order, params.mode, self.dim)
        ml = params.mesh_level or int(np.log2(min(grid.shape))) - 1
        self.fas = FasParams(params.tol, params.k_max, params.s, ml)
        hier = make_hierarchy(grid, ml)
        plan = make_plan("x", self.dim, "ff")
        b_mom = params.dt / params.re if params.order == 1 else params.dt / (2.0 * params.re)
        # the four solves run one after another: one set of multigrid
        # workspaces (an engine arena) serves them all
        self.arena = EngineArena() if share_workspaces else None
        self.solvers = {c: FasSolver(hier, LOC_OF[c], self.bcs[c], plan, OperatorCoeffs(1.0, b_mom),
                                     arena=self.arena)
                        for c in self.comps}
        self.solvers["p"] = FasSolver(hier, Location.CELL, self.bcs["p"], plan,
                                      OperatorCoeffs(0.0, params.dt), arena=self.arena)
        dev = device
        # resident slots (the schedule's accounting): velocity fields carry
        # halo 2 for the WENO stencil, pressure halo 1
        self.slots = {}
        for name in self.schedule.resident_slots():
            comp = name.split("_")[0].lower()
            if comp == "p":
                self.slots[name] = Field(grid, Location.CELL, 1, device=dev)
            else:
                self.slots[name] = Field(grid, LOC_OF[comp], 2, device=dev)
        self.device = next(iter(self.slots.values())).device
        # transient scratch (not resident state): the momentum source of the
        # component being solved and the pressure source are never live at
        # the same time (every schedule runs rhs_c -> solve_c per component,
        # then the pressure solve), so ONE buffer of the largest shape backs
        # all of them (-3 fields: 1024^3 NS fits in well under 150 GB)
        def shape_of(loc):
            ea = loc.edge_axis
            return tuple(n + 1 if a == ea else n + 2 for a, n in enumerate(grid.shape))
        shapes = {c: shape_of(LOC_OF[c]) for c in self.comps}
        shapes["p"] = shape_of(Location.CELL)
        self._scratch = torch.zeros(max(int(np.prod(v)) for v in shapes.values()),
                                    dtype=torch.float64, device=self.device)
        view = lambda q: self._scratch[: int(np.prod(shapes[q]))].view(shapes[q])  # noqa: E731
        self._f = {c: Field(grid, LOC_OF[c], 1, data=view(c)) for c in self.comps}
        self._mix = {}
        self._mix_tag = {}   # mixture buffer -> (op, slots and their generations) it holds
        self._gen = {}       # slot -> write generation
        self._slot_of = {id(F): name for name, F in self.slots.items()}
        self._fp = Field(grid, Location.CELL, 1, data=view("p"))
        self.held = {slot: q for q, slot in self.schedule.initial}  # slot -> quantity
        self.step_count = 0
        # list to collect (formula, component, start event, end event) per
        # executed Step on torch's current stream (bench.py), or None
        self.timing = None

    # ------------------------------------------------------------ state I/O
    def resident_count(self) -> int:
        return len(self.slots)

    def field_of(self, quantity: str) -> Field:
        for slot, q in self.held.items():
            if q == quantity:
                return self.slots[slot]
        raise MissingBinding(f"{quantity} is not bound to a slot")

    def set_state(self, vel: dict, p=None):
        """Initial u^0 (and u^{-1} = u^0 for order 2) and p^0.
        ``vel[c]`` / ``p``: interior arrays (numpy or tensors) or None for 0."""
        self._mix_tag.clear()
        for c in self.comps:
            F = self.field_of(f"{c}_n")
            F.data.zero_()
            if vel.get(c) is not None:
                F.interior = vel[c]
            fill_ghosts(F, self.bcs[c])
            if self.params.order == 2:
                G = self.field_of(f"{c}_nm1")
                G.data.copy_(F.data)
                G.ghosts_fresh = True
        P = self.field_of("p_n")
        P.data.zero_()
        if p is not None:
            P.interior = p
        G = self.field_of("p_tld_prev")
        G.data.zero_()

    def velocity(self, c: str) -> Field:
        return self.field_of(f"{c}_n")

    def pressure(self) -> Field:
        return self.field_of("p_n")

    # ----------------------------------------------------------- formulas
    def _mix_field(self, key, comp, op, a: Field, b: Field) -> Field:
        """Order-2 velocity mixture (halo 2, ghosts filled) in buffer ``key``.
        A buffer still holding the same mixture of the same slot contents
        (no write to either slot since, tracked by _bind's generations) is
        reused: within a step the three momentum sources ask for EXT(w)
        three times, EXT(v) and AVG(u) twice each."""
        M = self._mix.get(key)
        if M is None:
            M = self._mix[key] = Field(self.grid, LOC_OF[comp], 2, device=self.device)
        sa, sb_ = self._slot_of.get(id(a)), self._slot_of.get(id(b))
        tag = None
        if sa is not None and sb_ is not None:
            tag = (op, sa, self._gen.get(sa, 0), sb_, self._gen.get(sb_, 0))
            if self._mix_tag.get(key) == tag:
                return M
        elem(op, M.interior, [a.interior, b.interior])
        fill_ghosts(M, self.bcs[comp])
        self._mix_tag[key] = tag
        return M

    def momentum_rhs(self, c: str, read: dict) -> Field:
        """Source term f_c of Table 3/5 step 1 (see module docstring)."""
        dt, order = self.params.dt, self.params.order
        vel = []
        for o in self.comps:
            un = read[f"{o}_n"]
            if order == 1:
                fill_ghosts(un, self.bcs[o])
                vel.append(un)
            elif f"{o}_tld" in read:  # one mixture buffer per component
                vel.append(self._mix_field(o, o, MIX_AVG, un, read[f"{o}_tld"]))
            else:
                vel.append(self._mix_field(o, o, MIX_EXT, un, read[f"{o}_nm1"]))
        target = AXIS_OF[c]
        conv = weno3_convect(tuple(vel), target, out=self._f[c])  # reuse f as conv buffer
        un = read[f"{c}_n"]
        f = self._f[c]
        # f = ((u^n - dt*conv) - dt*(grad p^n)_c) [+ dt/(2Re)*Lap(u^n)], one pass
        if order == 2:
            fill_ghosts(un, self.bcs[c])
        momentum_source(order, f.interior, un, conv.interior, read["p_n"], target, dt,
                        dt / (2.0 * self.params.re) if order == 2 else 0.0)
        if self.forcing is not None:
            if order == 1:
                F = self._force(c, self.t + dt)
            elif self.forcing_rule == "trap":  # (F(t^n) + F(t^{n+1}))/2
                F = 0.5 * (self._force(c, self.t) + self._force(c, self.t + dt))
            else:                              # F(t^{n+1/2})
                F = self._force(c, self.t + 0.5 * dt)
            elem(AXPY, f.interior, [f.interior, F], s0=-dt)  # f + dt*F
        f.ghosts_fresh = False
        return f

    def _force(self, c: str, t: float) -> torch.Tensor:
        F = self.forcing(c, t)
        if not torch.is_tensor(F):
            F = torch.as_tensor(np.ascontiguousarray(F), dtype=torch.float64)
        return F.to(self.device)

    def pressure_poisson(self, tld: dict, guess: Field) -> SolveReport:
        """-dt*Lap(p~) = -div(u~), all-Neumann, zero mean;
        solved in place in ``guess`` (the previous increment)."""
        div = divergence_edges_to_cc(*[tld[c] for c in self.comps], out=self._fp)
        elem(NEG, div.interior, [div.interior])
        return self.solvers["p"].solve(guess, div, self.fas)

    # --------------------------------------------------------------- step
    def step(self) -> StepReport:
        rep = StepReport()
        scratch = {}
        sched = self.schedule
        timing = self.timing
        for st in sched.steps:
            read = {}
            for q, slot in st.reads:
                if slot.startswith("@"):
                    read[q] = scratch[slot]
                else:
                    if self.held.get(slot) != q:
                        raise MissingBinding(f"{st.describe()}: {q} not in {slot} "
                                             f"(holds {self.held.get(slot)})")
                    read[q] = self.slots[slot]
            if timing is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
            self._exec(st, read, scratch, rep)
            if timing is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                timing.append((st.formula, st.comp, e0, e1))
        ren = dict(sched.rebind)
        self.held = {slot: ren.get(q, q) for slot, q in self.held.items()}
        self.step_count += 1
        self.t = self.step_count * self.params.dt
        return rep

    def _exec(self, st, read: dict, scratch: dict, rep: StepReport):
        """Execute one schedule Step on device fields."""
        dt = self.params.dt
        if st.formula == "rhs":
            scratch[st.writes[0][1]] = self.momentum_rhs(st.comp, read)
        elif st.formula in ("copy", "rotate2"):
            moves = dict(st.copy_map)
            for q, slot in st.writes:  # in order: the reference rotate2 semantics
                src = read[moves[q]]
                dst = self.slots[slot]
                if dst is not src:
                    dst.data.copy_(src.data)
                    dst.ghosts_fresh = src.ghosts_fresh
                self._bind(q, slot)
        elif st.formula == "solve_momentum":
            c = st.comp
            q, slot = st.writes[0]
            dst = self.slots[slot]
            src = read[f"{c}_n"]
            # the solve starts from u^n and writes u~ into the slot (no copy)
            rep.momentum[c] = self.solvers[c].solve_into(src, dst, read[f"f_{c}"], self.fas)
            self._bind(q, slot)
        elif st.formula == "solve_pressure":
            q, slot = st.writes[0]
            guess = self.slots[slot]
            rep.pressure = self.pressure_poisson({c: read[f"{c}_tld"] for c in self.comps}, guess)
            self._bind(q, slot)
        elif st.formula == "correct":
            c = st.comp
            q, slot = st.writes[0]
            dst = self.slots[slot]
            # u^{n+1} = u~ - dt*(grad p~)_c, one pass
            momentum_source(0, dst.interior, read[f"{c}_tld"], None, read["p_tld"],
                            AXIS_OF[c], dt)
            fill_ghosts(dst, self.bcs[c])
            self._bind(q, slot)
        elif st.formula == "p_update":
            q, slot = st.writes[0]
            dst = self.slots[slot]
            elem(ADD, dst.interior, [read["p_n"].interior, read["p_tld"].interior])
            dst.ghosts_fresh = False
            self._bind(q, slot)
        else:
            raise ValueError(f"unknown formula {st.formula}")

    def _bind(self, q: str, slot: str):
        """Every write of a slot by a schedule Step ends here: bump its
        generation (invalidates mixtures computed from it)."""
        self.held[slot] = q
        self._gen[slot] = self._gen.get(slot, 0) + 1

    def divergence(self) -> float:
        """integral_divergence of the current velocity (Eqs. div2D/div3D)."""
        return integral_divergence(*[self.velocity(c) for c in self.comps])


def run_cavity(grid: GridLevel, params: NSParams, steps: int, lid: float = 1.0,
               device=None, callback=None):
    """Integrate the lid-driven cavity from rest for ``steps`` steps;
    returns the stepper (fields in ``stepper.velocity(c)``)."""
    st = ProjectionStepper(grid, params, cavity_bcs(grid.dim, lid), device=device)
    st.set_state({})
    for k in range(steps):
        rep = st.step()
        if callback is not None:
            callback(k, st, rep)
    return st


def centerline_profiles(stepper: ProjectionStepper):
    """u along the vertical centerline and v along the horizontal one (2D;
    mid-plane lines in 3D), as host arrays."""
    g = stepper.grid
    u = stepper.velocity("u").interior
    v = stepper.velocity("v").interior
    if g.dim == 2:
        mx = g.shape[0] // 2
        my = g.shape[1] // 2
        u_line = u[mx - 1, :].cpu().numpy()
        v_line = v[:, my - 1].cpu().numpy()
    else:
        mid = [n // 2 for n in g.shape]
        u_line = u[mid[0] - 1, mid[1] - 1, :].cpu().numpy()
        v_line = v[:, mid[1] - 1, mid[2] - 1].cpu().numpy()
    return u_line, v_line
