"""Slot schedules (host-only): slot counts, soundness, dataflow equality
(Tables 2-5).  CPU."""
import os

import pytest

from paper_2510_11152_b200 import schedule as S


@pytest.mark.parametrize("dim", [2, 3])
def test_counts_and_validity(dim):
    counts = {(1, "classical"): 3 * dim + 3, (1, "efficient"): 2 * dim + 2,
              (2, "classical"): 4 * dim + 3, (2, "efficient"): 2 * dim + 2}
    for (o, m), n in counts.items():
        sch = S.build_schedule(o, m, dim)
        assert len(sch.slots) == n == S.expected_slot_count(o, m, dim)
        assert S.validate_schedule(sch) == []


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [1, 2])
def test_efficient_equals_classical_dataflow(dim, order):
    eff = S.build_schedule(order, "efficient", dim)
    cls = S.build_schedule(order, "classical", dim)
    assert S.validate_schedule(eff, reference=cls, steps=3) == []


def test_swapped_steps_detected():
    """Table 3 with correct/update steps reordered clobbers."""
    sch = S.build_schedule(1, "efficient", 3)
    steps = list(sch.steps)
    i = next(k for k, s in enumerate(steps) if s.formula == "p_update")
    j = next(k for k, s in enumerate(steps) if s.formula == "solve_pressure")
    steps[i], steps[j] = steps[j], steps[i]
    bad = S.SlotSchedule(sch.name, sch.order, sch.mode, sch.dim, sch.slots, sch.initial,
                         tuple(steps), sch.rebind)
    assert S.validate_schedule(bad)


@pytest.mark.reference
@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg"), reason="reference not mounted")
def test_matches_reference_schedules():
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import import_reference
    fm = import_reference("numpy")
    import fasmg.schedule as R
    for dim in (2, 3):
        for o in (1, 2):
            for m in ("classical", "efficient"):
                a, b = R.build_schedule(o, m, dim), S.build_schedule(o, m, dim)
                assert a.slots == b.slots and dict(a.initial) == dict(b.initial)
                assert a.rebind == b.rebind and a.name == b.name
                assert [(x.formula, x.comp, x.reads, x.writes, x.copy_map) for x in a.steps] == \
                       [(x.formula, x.comp, x.reads, x.writes, x.copy_map) for x in b.steps]
                assert R.validate_schedule(a) == S.validate_schedule(b)
