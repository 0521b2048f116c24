"""Parity at BASELINE.json's full sizes (configs[1]-[3]): the B200 solve of
the benchmark problems against the CPU oracle (itself pinned bitwise to the
reference, tests/test_oracle_golden.py) on the same inputs.

* 3D heat 512^3 (the bench workload): full solve to tol 1e-9, residual
  history within 1e-10 relative, final field bitwise.
* 2D heat 8192^2: 20 V-cycles (the residual stalls at the roundoff floor
  above tol 1e-9), same bar.
* An edge-centred (MAC face velocity) field at 512^3 with the lid-driven
  cavity BC: two V-cycles, same bar.

The oracle runs with every host thread (its results do not depend on the
thread count); the three cases take about a minute of host time.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cases as C  # noqa: E402

pytestmark = pytest.mark.gpu

HIST_RTOL = 1e-10


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.set_threads(os.cpu_count() or 1)
    yield oracle
    oracle.set_threads(1)


def _bench_inputs(O, n):
    """p0 = default_rng(0).random, f = L_h(exact) -- the
    bench.py / paper timing problem."""
    shape = tuple(m + 2 for m in n)
    p0 = np.zeros(shape)
    p0[(slice(1, -1),) * len(n)] = np.random.default_rng(0).random(n)
    f0 = np.zeros(shape)
    f0[(slice(1, -1),) * len(n)] = O.poisson_rhs_discrete(n)
    return p0, f0


def _check(P, O, n, loc, p0, f0, bc_spec, a, b, tol, k_max):
    dim = len(n)
    ml = int(np.log2(n[0])) - 1
    halo = 1
    g = P.unit_grid(n)
    Lc = getattr(P.Location, loc.upper())
    p = P.Field(g, Lc, halo, p0.copy())
    f = P.Field(g, Lc, halo, f0.copy())
    faces = C.bc_faces(dim, bc_spec)
    bc = P.BoundaryCondition(dim, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))
    _, rep = P.solve(p, f, P.OperatorCoeffs(a, b), P.FasParams(tol, k_max, 2, ml),
                     P.make_plan("x", dim), bc)
    got = p.data.cpu().numpy()
    del p, f
    torch.cuda.empty_cache()
    op = O.OField(n, loc, halo, p0)
    of = O.OField(n, loc, halo, f0)
    it, hist = O.fas_solve(op, of, a, b, faces, O.plan_colors("x", dim), tol, k_max, 2, ml)
    assert rep.iterations == it, (rep.iterations, it)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64)), "field mismatch"
    return rep


def test_heat3d_512_solve_matches_oracle(P, O):
    n = (512, 512, 512)
    p0, f0 = _bench_inputs(O, n)
    rep = _check(P, O, n, "cell", p0, f0, "dirichlet", 1.0, 1.0, 1e-9, 20)
    assert rep.converged


def test_heat2d_8192_solve_matches_oracle(P, O):
    # at h = 1/8192 the scaled residual stalls above 1e-9 (roundoff floor)
    # in the oracle too, so the 20 cycles all run: parity is the check
    n = (8192, 8192)
    p0, f0 = _bench_inputs(O, n)
    rep = _check(P, O, n, "cell", p0, f0, "dirichlet", 1.0, 1.0, 1e-9, 20)
    assert rep.final_residual < 1e-6


def test_edge_512_lid_two_cycles_match_oracle(P, O):
    n = (512, 512, 512)
    p0 = C.rand_field(21, n, "edge_tb", 1)
    f0 = C.rand_field(22, n, "edge_tb", 1)
    _check(P, O, n, "edge_tb", p0, f0, "lid", 1.0, 0.05, 1e-30, 2)
