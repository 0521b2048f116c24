"""Engines sharing their level arrays through an EngineArena (the NS
stepper's four solves): alternating solves of different locations give the
bitwise results of private engines."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


def _solvers(P, g, ml, arena):
    from paper_2510_11152_b200.fas import FasSolver
    plan = P.make_plan("x", 3)
    hier = P.make_hierarchy(g, ml)
    lid = P.BoundaryCondition.dirichlet(3).with_face("zhi", P.FaceRule("dirichlet", 1.0))
    return [
        (P.Location.EDGE_EW, FasSolver(hier, P.Location.EDGE_EW, lid, plan,
                                       P.OperatorCoeffs(1.0, 0.01), arena=arena)),
        (P.Location.CELL, FasSolver(hier, P.Location.CELL, P.BoundaryCondition.neumann(3), plan,
                                    P.OperatorCoeffs(0.0, 0.5), arena=arena)),
        (P.Location.EDGE_TB, FasSolver(hier, P.Location.EDGE_TB, P.BoundaryCondition.dirichlet(3),
                                       plan, P.OperatorCoeffs(1.0, 0.01), arena=arena)),
    ]


def test_arena_solves_bitwise(P):
    import cases as C
    from paper_2510_11152_b200.fas import EngineArena
    n, ml = 64, 5
    g = P.unit_grid((n,) * 3)
    params = P.FasParams(1e-30, 3, 2, ml)
    out = {}
    for shared in (False, True):
        arena = EngineArena() if shared else None
        res = []
        sv = _solvers(P, g, ml, arena)
        for rnd in range(2):  # second round: every engine finds another was last
            for i, (loc, S) in enumerate(sv):
                halo = 1 if loc is P.Location.CELL else 2
                p = P.Field(g, loc, halo, C.rand_field(40 + i, (n,) * 3, loc.value, halo))
                f = P.Field(g, loc, halo, C.rand_field(50 + i, (n,) * 3, loc.value, halo))
                rep = S.solve(p, f, params)
                res.append((p.data.clone(), list(rep.residual_history)))
        out[shared] = res
    for (a, ha), (b, hb) in zip(out[False], out[True]):
        assert torch.equal(a, b)
        assert ha == hb
