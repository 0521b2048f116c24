"""Slot schedules of the projection schemes (host-side, symbolic).

Same model and API as PKG/schedule.py (Tables 2-5): a
time step is an ordered list of :class:`Step` s, each naming a formula, the
time-level quantities it reads and writes and the resident slot that holds
each one.  ``build_schedule(order, mode, dim)`` gives the four schedules
(classical 12/15 slots, memory-efficient 8 slots in 3D; 9/11 and 6 in 2D),
``validate_schedule`` symbolically executes one against its slot bindings.

The B200 stepper (``ns.py``) executes these same Step lists on device
fields, so a schedule that validates here is exactly the data movement the
GPU performs.

Quantities: ``<c>_n``, ``<c>_nm1``, ``<c>_tld``, ``<c>_np1`` per velocity
component, ``p_n``, ``p_tld``, ``p_tld_prev`` (previous increment, the
pressure solve's initial guess), ``p_np1`` and source terms ``f_<c>``.
Slots whose name starts with ``@`` are per-step scratch (not resident).
"""

from __future__ import annotations

from dataclasses import dataclass

COMPONENTS_3D = ("u", "v", "w")
CARRIED = ("u_n", "v_n", "w_n", "p_n", "p_tld_prev")  # values carried across steps


@dataclass(frozen=True)
class Step:
    formula: str
    comp: str | None
    reads: tuple      # ((quantity, slot), ...)
    writes: tuple     # ((quantity, slot), ...)
    copy_map: tuple = ()  # ((written quantity, read quantity), ...) for data moves

    def describe(self) -> str:
        return self.formula + (f" {self.comp}" if self.comp else "")


@dataclass(frozen=True)
class SlotSchedule:
    name: str
    order: int
    mode: str
    dim: int
    slots: tuple
    initial: tuple    # ((quantity, slot), ...) at the start of a step
    steps: tuple
    rebind: tuple     # end-of-step renames ((old quantity, new quantity), ...)

    @property
    def components(self):
        return COMPONENTS_3D[: self.dim]

    def resident_slots(self):
        return tuple(s for s in self.slots if not s.startswith("@"))


def expected_slot_count(order: int, mode: str, dim: int) -> int:
    """8 (efficient) or 12/15 (classical) in 3D; 6 or 9/11 in 2D."""
    if mode == "efficient":
        return 2 * dim + 2
    return {1: 3, 2: 4}[order] * dim + 3


def _S(comp: str, tag: str) -> str:
    return ("P_" if comp == "p" else comp.upper() + "_") + tag


def _rhs_reads(comps, slot_of, advanced, order):
    """Reads of the source term of one component.  Order 1: u^n of every
    component and p^n.  Order 2 (Table 5): components already advanced this
    step enter through (u^n + u~)/2, the others through (3u^n - u^{n-1})/2."""
    reads = []
    for o in comps:
        reads.append((f"{o}_n", slot_of[f"{o}_n"]))
        if order == 2:
            other = f"{o}_tld" if o in advanced else f"{o}_nm1"
            reads.append((other, slot_of[other]))
    reads.append(("p_n", "P_old"))
    return tuple(reads)


def build_schedule(order: int, mode: str, dim: int) -> SlotSchedule:
    if order not in (1, 2) or mode not in ("classical", "efficient"):
        raise ValueError(f"no schedule for order={order}, mode={mode}")
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    comps = COMPONENTS_3D[:dim]
    eff = mode == "efficient"
    tags = ("new", "old") if eff else (("new", "old", "tld") if order == 1
                                       else ("new", "old", "2old", "tld"))
    slots = tuple(_S(c, t) for c in comps for t in tags) + tuple(
        _S("p", t) for t in (("new", "old") if eff else ("new", "old", "tld")))
    p_guess_slot = "P_new" if eff else "P_tld"

    # where each quantity lives at step start
    if order == 1:
        initial = {f"{c}_n": _S(c, "old") for c in comps}
    elif eff:
        initial = {}
        for c in comps:
            initial[f"{c}_n"] = _S(c, "new")
            initial[f"{c}_nm1"] = _S(c, "old")
    else:
        initial = {}
        for c in comps:
            initial[f"{c}_n"] = _S(c, "old")
            initial[f"{c}_nm1"] = _S(c, "2old")
    initial["p_n"] = "P_old"
    initial["p_tld_prev"] = p_guess_slot

    steps = []
    loc = dict(initial)
    advanced = []
    tld_slot = (lambda c: _S(c, "new")) if eff else (lambda c: _S(c, "tld"))
    for c in comps:
        steps.append(Step("rhs", c, _rhs_reads(comps, loc, advanced, order),
                          ((f"f_{c}", f"@f_{c}"),)))
        if eff and order == 2:
            # lagged rotation: u^{n-1} <- u^n right after its last reader
            steps.append(Step("copy", c, ((f"{c}_n", _S(c, "new")),),
                              ((f"{c}_n", _S(c, "old")),),
                              copy_map=((f"{c}_n", f"{c}_n"),)))
            loc[f"{c}_n"] = _S(c, "old")
            loc.pop(f"{c}_nm1", None)
        # initial guess u^n: order-2 efficient solves in place in U_new, which
        # still holds u^n after the lagged copy
        guess = _S(c, "new") if (eff and order == 2) else loc[f"{c}_n"]
        steps.append(Step("solve_momentum", c,
                          ((f"f_{c}", f"@f_{c}"), (f"{c}_n", guess)),
                          ((f"{c}_tld", tld_slot(c)),)))
        loc[f"{c}_tld"] = tld_slot(c)
        advanced.append(c)
    steps.append(Step("solve_pressure", None,
                      tuple((f"{c}_tld", loc[f"{c}_tld"]) for c in comps)
                      + (("p_tld_prev", p_guess_slot),),
                      (("p_tld", p_guess_slot),)))
    for c in comps:
        dst = _S(c, "old") if (eff and order == 1) else _S(c, "new")
        steps.append(Step("correct", c, ((f"{c}_tld", loc[f"{c}_tld"]), ("p_tld", p_guess_slot)),
                          ((f"{c}_np1", dst),)))
    p_dst = "P_old" if eff else "P_new"
    steps.append(Step("p_update", None, (("p_n", "P_old"), ("p_tld", p_guess_slot)),
                      (("p_np1", p_dst),)))

    if eff:
        rebind = tuple((f"{c}_np1", f"{c}_n") for c in comps)
        if order == 2:
            rebind += tuple((f"{c}_n", f"{c}_nm1") for c in comps)
        rebind += (("p_np1", "p_n"), ("p_tld", "p_tld_prev"))
    else:
        for c in comps:
            if order == 1:
                steps.append(Step("copy", c, ((f"{c}_np1", _S(c, "new")),),
                                  ((f"{c}_n", _S(c, "old")),),
                                  copy_map=((f"{c}_n", f"{c}_np1"),)))
            else:
                steps.append(Step("rotate2", c,
                                  ((f"{c}_n", _S(c, "old")), (f"{c}_np1", _S(c, "new"))),
                                  ((f"{c}_nm1", _S(c, "2old")), (f"{c}_n", _S(c, "old"))),
                                  copy_map=((f"{c}_nm1", f"{c}_n"), (f"{c}_n", f"{c}_np1"))))
        steps.append(Step("copy", "p", (("p_np1", "P_new"),), (("p_n", "P_old"),),
                          copy_map=(("p_n", "p_np1"),)))
        rebind = (("p_tld", "p_tld_prev"),)
    label = ("first" if order == 1 else "second") + f"-order {mode} {dim}D"
    return SlotSchedule(label, order, mode, dim, slots,
                        tuple((q, s) for q, s in initial.items()), tuple(steps), rebind)


def all_schedules(dim: int):
    return tuple(build_schedule(o, m, dim) for o in (1, 2) for m in ("classical", "efficient"))


# ---------------------------------------------------------------------------
# symbolic execution (liveness, layout steadiness, dataflow equality)
# ---------------------------------------------------------------------------

def _run_step(sched: SlotSchedule, bind: dict, problems: list):
    scratch = {}
    for no, st in enumerate(sched.steps, 1):
        vals = {}
        for q, slot in st.reads:
            store = scratch if slot.startswith("@") else bind
            held = store.get(slot)
            if held is None:
                problems.append(f"step {no} ({st.describe()}): reads {q} from empty slot {slot}")
                vals[q] = ("missing", q)
            else:
                if held[0] != q:
                    problems.append(f"step {no} ({st.describe()}): reads {q} from {slot} "
                                    f"but it holds {held[0]}")
                vals[q] = held[1]
        moves = dict(st.copy_map)
        for q, slot in st.writes:
            term = (vals.get(moves[q], ("missing", moves[q])) if q in moves
                    else (st.formula, st.comp, tuple(sorted(vals.items()))))
            (scratch if slot.startswith("@") else bind)[slot] = (q, term)
    ren = dict(sched.rebind)
    for slot, (q, term) in list(bind.items()):
        bind[slot] = (ren.get(q, q), term)


def validate_schedule(schedule: SlotSchedule, reference: SlotSchedule | None = None,
                      steps: int = 2):
    """Violations of a schedule (empty list = sound): clobbered or missing
    reads, wrong slot count, unsteady binding layout, and (with
    ``reference``) any difference in the values carried across steps."""
    problems = []
    want = expected_slot_count(schedule.order, schedule.mode, schedule.dim)
    if len(schedule.slots) != want:
        problems.append(f"slot count {len(schedule.slots)} != expected {want} for "
                        f"{schedule.mode} order {schedule.order} in {schedule.dim}D")
    bind = {slot: (q, ("init", q)) for q, slot in schedule.initial}
    layout0 = {slot: q for slot, (q, _) in bind.items()}
    carried = None
    for _ in range(steps):
        _run_step(schedule, bind, problems)
        carried = {q: t for _, (q, t) in bind.items() if q in CARRIED}
    layout1 = {slot: q for slot, (q, _) in bind.items() if q in layout0.values()}
    for slot, q in layout0.items():
        if layout1.get(slot) != q:
            problems.append(f"binding of {q} moved from {slot}; layout must be steady")
            break
    if reference is not None:
        rb = {slot: (q, ("init", q)) for q, slot in reference.initial}
        for _ in range(steps):
            _run_step(reference, rb, [])
        rc = {q: t for _, (q, t) in rb.items() if q in CARRIED}
        diff = [q for q in rc if carried.get(q) != rc[q]]
        if diff:
            problems.append(f"dataflow differs from {reference.name} for quantities {diff}")
    return problems
