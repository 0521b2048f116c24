"""Heat driver and paper known answers on the GPU."""
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


def test_heat_steps_match_oracle(P):
    import oracle as O
    from paper_2510_11152_b200.heat import HeatStepper
    n = (32, 32, 32)
    rng = np.random.default_rng(3)
    p0 = np.zeros((34, 34, 34))
    p0[1:-1, 1:-1, 1:-1] = rng.random(n)
    g = P.unit_grid(n)
    p = P.Field(g, P.Location.CELL, 1, p0.copy())
    hs = HeatStepper(g, dt=0.01, tol=1e-10, k_max=20)
    op = O.OField(n, "cell", 1, p0.copy())
    for _ in range(3):
        rep = hs.step(p)
        f = O.OField(n, "cell", 1)
        f.interior[...] = op.interior
        it, hist = O.fas_solve(op, f, 1.0, 0.01, O.uniform_bc(3, "dirichlet"),
                               O.plan_colors("x", 3), 1e-10, 20, 2, 4)
        np.testing.assert_allclose(rep.residual_history, hist, rtol=1e-10)
        assert np.array_equal(p.numpy(), op.data)


@pytest.mark.parametrize("n,err", [(32, 1.74e-3), (64, 4.33e-4), (128, 1.08e-4)])
def test_paper_asymptotic_3d(P, n, err):
    """PAPER.md:442-446 (Table err_3D): second-order error at 32/64/128^3."""
    from paper_2510_11152_b200 import manufactured as M
    g = P.unit_grid((n,) * 3)
    p = P.Field(g, P.Location.CELL)
    f = M.poisson_rhs_continuous(g)
    _, rep = P.solve(p, f, P.OperatorCoeffs(1.0, 1.0), P.FasParams(1e-9, 20, 2, int(np.log2(n)) - 1),
                     P.make_plan("x", 3), P.BoundaryCondition.dirichlet(3))
    e = p.interior.cpu().numpy() - M.poisson_exact_array(g)
    l2 = g.h ** 1.5 * np.sqrt(np.sum(e * e))
    assert abs(l2 - err) / err < 0.01
    assert rep.iterations == 7


def test_paper_asymptotic_2d_1024(P):
    """PAPER.md:423 (Table err_2D): 2.58e-6 at 1024^2."""
    from paper_2510_11152_b200 import manufactured as M
    g = P.unit_grid((1024, 1024))
    p = P.Field(g, P.Location.CELL)
    f = M.poisson_rhs_continuous(g)
    P.solve(p, f, P.OperatorCoeffs(1.0, 1.0), P.FasParams(1e-9, 20, 2, 9),
            P.make_plan("x", 2), P.BoundaryCondition.dirichlet(2))
    e = p.interior.cpu().numpy() - M.poisson_exact_array(g)
    l2 = g.h * np.sqrt(np.sum(e * e))
    assert abs(l2 - 2.58e-6) / 2.58e-6 < 0.01


def test_smoother_ordering_counts(P):
    """PAPER.md:249 / SPEC.md:593: X-ff needs the fewest cycles; measured
    reference counts at 512^2: X-ff 7, X-fb 13, U-ff 19, U-fb 17, Z-ff 24,
    Z-fb 18."""
    from paper_2510_11152_b200 import manufactured as M
    g = P.unit_grid((512, 512))
    want = {("x", "ff"): 7, ("x", "fb"): 13, ("u", "ff"): 19, ("u", "fb"): 17,
            ("z", "ff"): 24, ("z", "fb"): 18, ("rbgs", "ff"): 7}
    p0 = np.zeros((514, 514))
    p0[1:-1, 1:-1] = np.random.default_rng(0).random((512, 512))
    f = M.poisson_rhs_discrete(g)
    for (shape, seq), cnt in want.items():
        p = P.Field(g, P.Location.CELL, 1, p0.copy())
        ff = f.copy()
        _, rep = P.solve(p, ff, P.OperatorCoeffs(1.0, 1.0), P.FasParams(1e-9, 100, 2, 8),
                         P.make_plan(shape, 2, seq), P.BoundaryCondition.dirichlet(2))
        assert rep.iterations == cnt, (shape, seq, rep.iterations)
