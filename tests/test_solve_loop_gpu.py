"""The outer solve loop as one graph launch (fasmg_engine_solve: V-cycle +
norm + the convergence test in a CUDA conditional WHILE node) against the
host loop it replaces (PKG/fas.py:147-154 restated in FasSolver._solve):
same iteration count, bitwise the same residual history and field, for
stops on tol and on k_max, from both speculation states, 2D and 3D,
singular problems, and against the oracle."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cases as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


def make(P, shape, a=1.0, bc=None, ml=3):
    d = len(shape)
    g = P.unit_grid(shape)
    S = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL,
                    bc or P.BoundaryCondition.dirichlet(d), P.make_plan("x", d),
                    P.OperatorCoeffs(a, 0.5))
    return g, S


def host_loop(e, scale, k_max, tol):
    hist = []
    for _ in range(k_max):
        res = scale * math.sqrt(e.run(1, with_norm=True))
        hist.append(res)
        if res <= tol:
            break
    return hist


@pytest.mark.parametrize("shape,env", [
    ((64, 64, 64), {"FASMG_TMA_MIN": 0}),
    ((64, 64, 64), {"FASMG_TMA_MIN": 0, "FASMG_SPEC": 0}),
    ((32, 32, 32), {}),
    ((128, 128), {}),
])
@pytest.mark.parametrize("stop", ["tol", "kmax", "first"])
def test_device_loop_matches_host_loop(P, monkeypatch, shape, env, stop):
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    g, S = make(P, shape)
    p0 = C.rand_field(71, shape, "cell", 1)
    f0 = C.rand_field(72, shape, "cell", 1)
    scale = g.h ** (g.dim / 2.0)
    # a reference history to place tol between two iterations
    p = P.Field(g, P.Location.CELL, 1, p0.copy())
    f = P.Field(g, P.Location.CELL, 1, f0.copy())
    e = S.engine(2, p.device)
    e.load(p, f)
    ref = host_loop(e, scale, 6, -1.0)
    k_max, tol = {"tol": (6, 0.5 * (ref[2] + ref[3])), "kmax": (5, -1.0),
                  "first": (6, 2.0 * ref[0])}[stop]
    e.load(p, f)
    want_h = host_loop(e, scale, k_max, tol)
    want = P.Field(g, P.Location.CELL, 1, p0.copy())
    e.store(want)
    e.load(p, f)
    got_h = e.solve_loop(k_max, tol, scale)
    got = P.Field(g, P.Location.CELL, 1, p0.copy())
    e.store(got)
    torch.cuda.synchronize()
    assert len(got_h) == {"tol": 4, "kmax": 5, "first": 1}[stop]
    assert got_h == want_h
    assert np.array_equal(got.data.cpu().numpy().view(np.uint64),
                          want.data.cpu().numpy().view(np.uint64))


def test_device_loop_from_pending_state_and_repeat(P, monkeypatch):
    """Entered with a speculative half-sweep pending (after a host-loop
    cycle), run twice back to back, then continued by the host loop: the
    host loop's values throughout."""
    monkeypatch.setenv("FASMG_TMA_MIN", "0")
    shape = (64, 64, 64)
    g, S = make(P, shape)
    p0 = C.rand_field(73, shape, "cell", 1)
    f0 = C.rand_field(74, shape, "cell", 1)
    scale = g.h ** 1.5
    p = P.Field(g, P.Location.CELL, 1, p0.copy())
    f = P.Field(g, P.Location.CELL, 1, f0.copy())
    e = S.engine(2, p.device)
    e.load(p, f)
    want = host_loop(e, scale, 8, -1.0)
    e.load(p, f)
    got = host_loop(e, scale, 1, -1.0)
    got += e.solve_loop(3, -1.0, scale)
    got += e.solve_loop(2, -1.0, scale)
    got += host_loop(e, scale, 2, -1.0)
    assert got == want


def test_solver_solve_uses_device_loop_vs_oracle(P):
    """FasSolver.solve (device loop) on a singular Neumann problem: bitwise
    the oracle's field, its iteration count, history within 1e-10 (the
    oracle's numpy norm sums in another order), and bitwise the eager
    host-loop path (use_graph False)."""
    import oracle as O
    shape = (32, 32, 32)
    faces = C.bc_faces(3, "neumann")
    bc = P.BoundaryCondition(3, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))
    g, S = make(P, shape, a=0.0, bc=bc)
    p0 = C.rand_field(75, shape, "cell", 1)
    f0 = C.rand_field(76, shape, "cell", 1)
    op = O.OField(shape, "cell", 1, p0.copy())
    of = O.OField(shape, "cell", 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, 0.0, 0.5, faces, O.plan_colors("x", 3), 1e-9, 40, 2, 3,
                           dmin=0.0, dmax=1.0)
    O.set_threads(1)
    outs = []
    for use_graph in (True, False):
        S.use_graph = use_graph
        p = P.Field(g, P.Location.CELL, 1, p0.copy())
        f = P.Field(g, P.Location.CELL, 1, f0.copy())
        rep = S.solve(p, f, P.FasParams(1e-9, 40, 2, 3))
        torch.cuda.synchronize()
        outs.append((p.data.cpu().numpy(), rep))
    (a, ra), (b, rb) = outs
    assert ra.iterations == it == rb.iterations
    assert ra.residual_history == rb.residual_history
    np.testing.assert_allclose(ra.residual_history, hist, rtol=1e-10, atol=0)
    assert np.array_equal(a.view(np.uint64), op.data.view(np.uint64))
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("k_max,tol", [(3, float("nan")), (5000, 1e-6), (1, 1e-30)])
def test_solver_solve_device_vs_host_loop_edge_cases(P, monkeypatch, k_max, tol):
    """FasSolver.solve with the device loop against FASMG_DEVICE_LOOP=0 (the
    host loop): a NaN tolerance (never met: k_max cycles, as the host's
    `res <= tol` test), a k_max above the device loop's cap (the host loop
    runs; iterations stop on tol), a single cycle."""
    from paper_2510_11152_b200 import fas
    shape = (32, 32, 32)
    g, S = make(P, shape)
    p0 = C.rand_field(77, shape, "cell", 1)
    f0 = C.rand_field(78, shape, "cell", 1)
    outs = []
    for dev in (True, False):
        monkeypatch.setattr(fas, "_DEVICE_LOOP", dev)
        p = P.Field(g, P.Location.CELL, 1, p0.copy())
        f = P.Field(g, P.Location.CELL, 1, f0.copy())
        rep = S.solve(p, f, P.FasParams(tol, k_max, 2, 3))
        torch.cuda.synchronize()
        outs.append((p.data.cpu().numpy(), rep))
    (a, ra), (b, rb) = outs
    assert ra.residual_history == rb.residual_history
    assert ra.iterations == rb.iterations
    if tol != tol:
        assert ra.iterations == k_max
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
