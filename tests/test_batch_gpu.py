"""FasSolver.solve_host_batch: independent problems in host memory, copies
pipelined over streams; every result bitwise equal to a plain solve."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


def _problems(n, k, seed, halo=1, edge=None):
    rng = np.random.default_rng(seed)
    shape = tuple((m + 1 + 2 * (halo - 1)) if a == edge else (m + 2 * halo)
                  for a, m in enumerate(n))
    ps, fs = [], []
    for _ in range(k):
        p = np.zeros(shape)
        f = np.zeros(shape)
        core = tuple(slice(halo, s - halo) for s in shape)
        p[core] = rng.random(p[core].shape)
        f[core] = rng.random(f[core].shape) - 0.5
        ps.append(torch.from_numpy(p).pin_memory())
        fs.append(torch.from_numpy(f).pin_memory())
    return ps, fs


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["dirichlet3d", "neumann_singular3d", "edge_ns3d", "dir2d"])
def test_batch_matches_solve(P, case):
    Loc = P.Location
    halo, edge, loc = 1, None, Loc.CELL
    if case == "dirichlet3d":
        n, bc, co = (32, 32, 32), P.BoundaryCondition.dirichlet(3), P.OperatorCoeffs(1.0, 1.0)
    elif case == "neumann_singular3d":
        n, bc, co = (32, 32, 32), P.BoundaryCondition.neumann(3), P.OperatorCoeffs(0.0, 1.0)
    elif case == "edge_ns3d":
        n, bc, co = (32, 32, 32), P.BoundaryCondition.dirichlet(3), P.OperatorCoeffs(1.0, 0.05)
        halo, edge, loc = 2, 1, Loc.EDGE_NS
    else:
        n, bc, co = (64, 64), P.BoundaryCondition.dirichlet(2), P.OperatorCoeffs(1.0, 1.0)
    dim = len(n)
    g = P.unit_grid(n)
    ml = int(np.log2(n[0])) - 1
    params = P.FasParams(1e-9, 12, 2, ml)
    S = P.FasSolver(P.make_hierarchy(g, ml), loc, bc, P.make_plan("x", dim), co)
    ps, fs = _problems(n, 5, 11, halo, edge)
    ref = []
    for p, f in zip(ps, fs):
        pf = P.Field(g, loc, halo, p.numpy().copy())
        ff = P.Field(g, loc, halo, f.numpy().copy())
        rep = S.solve(pf, ff, params)
        ref.append((rep, pf.data.cpu().numpy(), ff.data.cpu().numpy()))
    out = [torch.empty_like(p).pin_memory() for p in ps]
    reps = S.solve_host_batch(ps, fs, params, out=out, halo=halo)
    torch.cuda.synchronize()
    for (rr, pr, fr), r, o, f in zip(ref, reps, out, fs):
        assert r.iterations == rr.iterations
        assert r.residual_history == rr.residual_history
        assert np.array_equal(o.numpy(), pr)
        assert np.array_equal(f.numpy(), fr)  # singular: the shifted rhs is written back


@pytest.mark.gpu
def test_batch_in_place_ring(P):
    """Default out = ps (in place); the same output tensor may recur."""
    n = (16, 16, 16)
    g = P.unit_grid(n)
    S = P.FasSolver(P.make_hierarchy(g, 3), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                    P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0))
    params = P.FasParams(1e-9, 1, 2, 3)
    ps, fs = _problems(n, 2, 5)
    want = []
    for p, f in zip(ps, fs):
        pf = P.Field(g, P.Location.CELL, 1, p.numpy().copy())
        S.solve(pf, P.Field(g, P.Location.CELL, 1, f.numpy().copy()), params)
        want.append(pf.data.cpu().numpy())
    S.solve_host_batch(ps, fs, params)
    torch.cuda.synchronize()
    for p, w in zip(ps, want):
        assert np.array_equal(p.numpy(), w)


def test_batch_rejects_bad_lengths():
    import paper_2510_11152_b200 as P
    g = P.unit_grid((8, 8))
    S = P.FasSolver(P.make_hierarchy(g, 2), P.Location.CELL, P.BoundaryCondition.dirichlet(2),
                    P.make_plan("x", 2), P.OperatorCoeffs(1.0, 1.0))
    with pytest.raises(ValueError):
        S.solve_host_batch([torch.zeros(10, 10)], [], P.FasParams(1e-9, 1, 2, 2))


@pytest.mark.gpu
def test_batch_rejects_output_aliasing_another_input(P):
    g = P.unit_grid((8, 8, 8))
    S = P.FasSolver(P.make_hierarchy(g, 2), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                    P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0))
    ps, fs = _problems((8, 8, 8), 2, 1)
    with pytest.raises(ValueError):
        S.solve_host_batch(ps, fs, P.FasParams(1e-9, 1, 2, 2), out=[ps[1], ps[0]])
    with pytest.raises(ValueError):  # in place with one tensor for both problems
        S.solve_host_batch([ps[0], ps[0]], fs, P.FasParams(1e-9, 1, 2, 2))
