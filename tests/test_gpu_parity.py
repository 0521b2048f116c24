"""Parity of the B200 CUDA path against the reference golden vectors and the
CPU oracle.  Every test here needs a GPU (``-m gpu``).

Bar (SURVEY.md section 8c / BASELINE.json north_star): per-point results
are bitwise identical to the reference; residual histories within 1e-10
relative (the outer residual norm is summed in a different -- fixed --
order than numpy's pairwise sum, so it may differ in the last few ulps).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cases as C  # noqa: E402
from _golden import cases, digest, expect_array, golden  # noqa: E402

pytestmark = pytest.mark.gpu

HIST_RTOL = 1e-10


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


LOC = {"cell": "CELL", "edge_ew": "EDGE_EW", "edge_ns": "EDGE_NS", "edge_tb": "EDGE_TB"}


def bc_of(P, dim, spec):
    faces = C.bc_faces(dim, spec)
    return P.BoundaryCondition(dim, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))


def loc_of(P, loc):
    return getattr(P.Location, LOC[loc])


@pytest.mark.parametrize("c", cases("kernel"), ids=lambda c: c["key"])
def test_kernel_abi(P, c):
    from paper_2510_11152_b200 import kernels as K
    arrays, sc = C.kernel_inputs(c)
    darr = {k: dev(v) for k, v in arrays.items()}
    C.run_kernel(K.KERNELS, c, darr, sc)
    for nm, a in darr.items():
        expect_array(f"{c['key']}/{nm}", host(a))


@pytest.mark.parametrize("c", cases("fill"), ids=lambda c: c["key"])
def test_fill_ghosts(P, c):
    n = tuple(c["n"])
    g = P.unit_grid(n)
    F = P.Field(g, loc_of(P, c["loc"]), c["halo"], C.rand_field(c["seed"], n, c["loc"], c["halo"]))
    P.fill_ghosts(F, bc_of(P, c["dim"], c["bc"]))
    expect_array(f"{c['key']}/data", host(F.data))


@pytest.mark.parametrize("c", cases("smooth"), ids=lambda c: c["key"])
def test_smooth_api(P, c):
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    g = P.unit_grid(n)
    p = P.Field(g, loc_of(P, loc), halo, C.rand_field(c["seed"], n, loc, halo))
    f = P.Field(g, loc_of(P, loc), halo, C.rand_field(c["seed"] + 1, n, loc, halo))
    plan = P.make_plan(c["plan"][0], c["dim"], c["plan"][1])
    P.smooth(f, p, P.OperatorCoeffs(c["a"], c["b"]), plan, bc_of(P, c["dim"], c["bc"]))
    expect_array(f"{c['key']}/p", host(p.data))


@pytest.mark.parametrize("c", cases("stag"), ids=lambda c: c["key"])
def test_staggered(P, c):
    n = tuple(c["n"])
    g = P.unit_grid(n)
    p = P.Field(g, P.Location.CELL, 1, C.rand_field(c["seed"], n, "cell", 1))
    for ax in range(c["dim"]):
        expect_array(f"{c['key']}/grad{ax}", host(P.gradient_axis(p, ax)))
    locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
    comps = [P.Field(g, loc_of(P, loc), 2, C.rand_field(c["seed"] + 1 + t, n, loc, 2))
             for t, loc in enumerate(locs)]
    div = P.divergence_edges_to_cc(*comps)
    expect_array(f"{c['key']}/div", host(div.interior))
    assert P.integral_divergence(*comps) == float(golden()[f"{c['key']}/intdiv"])


@pytest.mark.parametrize("c", cases("reduce"), ids=lambda c: c["key"])
def test_ordered_mean(P, c):
    from paper_2510_11152_b200.grid import view_sum
    G = golden()
    a = np.random.default_rng(c["seed"]).standard_normal(c["shape"])
    t = dev(a)
    v = t[tuple(slice(1, s - 1) for s in c["shape"])]
    s = float(view_sum(v).item())
    assert s == float(G[f"{c['key']}/sum"])
    assert s / v.numel() == float(G[f"{c['key']}/mean"])


def _manufactured(P):
    import oracle as O
    return O.manufactured


def _solve(P, c):
    import oracle as O
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    p0, f0 = C.solve_inputs(c, O.manufactured)
    if "domain" in c:
        g = P.GridLevel(0, n, (0.0,) * c["dim"], tuple(c["domain"]))
    else:
        g = P.unit_grid(n)
    L = loc_of(P, loc)
    p = P.Field(g, L, halo, p0.copy())
    f = P.Field(g, L, halo, f0.copy())
    params = P.FasParams(c["tol"], c["k_max"], c["s"], c["mesh_level"])
    plan = P.make_plan(c["plan"][0], c["dim"], c["plan"][1])
    _, rep = P.solve(p, f, P.OperatorCoeffs(c["a"], c["b"]), params, plan,
                     bc_of(P, c["dim"], c["bc"]))
    return p, f, rep, p0, f0, g, L, plan


@pytest.mark.parametrize("c", cases("solve"), ids=lambda c: c["key"])
def test_solve_parity(P, c):
    G = golden()
    key = c["key"]
    p, f, rep, p0, f0, g, L, plan = _solve(P, c)
    ref_hist = G[f"{key}/history"]
    assert rep.iterations == int(G[f"{key}/iterations"])
    np.testing.assert_allclose(np.array(rep.residual_history), ref_hist, rtol=HIST_RTOL, atol=0)
    pd = host(p.data)
    interior = pd[tuple(slice(c["halo"], c["halo"] + e)
                        for e in C.interior_extent(tuple(c["n"]), c["loc"]))]
    assert digest(interior) == str(G[f"{key}/pint_sha256"]), "solution interior differs"
    assert digest(pd) == str(G[f"{key}/p_sha256"]), "solution ghosts differ"
    assert digest(host(f.data)) == str(G[f"{key}/f_sha256"]), "rhs (mean shift) differs"
    # one bare V-cycle from the same inputs
    p1 = P.Field(g, L, c["halo"], p0.copy())
    f1 = P.Field(g, L, c["halo"], f0.copy())
    S = P.FasSolver(P.make_hierarchy(g, c["mesh_level"]), L, bc_of(P, c["dim"], c["bc"]), plan,
                    P.OperatorCoeffs(c["a"], c["b"]))
    S.vcycle(p1, f1, c["s"])
    p1d = host(p1.data)
    i1 = p1d[tuple(slice(c["halo"], c["halo"] + e)
                   for e in C.interior_extent(tuple(c["n"]), c["loc"]))]
    assert digest(i1) == str(G[f"{key}/vcycle_pint_sha256"])


def test_graph_and_eager_agree(P):
    c = [x for x in cases("solve") if x["name"] == "heat_3d_16"][0]
    import oracle as O
    p0, f0 = C.solve_inputs(c, O.manufactured)
    g = P.unit_grid(tuple(c["n"]))
    outs = []
    for use_graph in (True, False):
        p = P.Field(g, P.Location.CELL, 1, p0.copy())
        f = P.Field(g, P.Location.CELL, 1, f0.copy())
        S = P.FasSolver(P.make_hierarchy(g, 3), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                        P.make_plan("x", 3), P.OperatorCoeffs(1.0, 1.0))
        S.use_graph = use_graph
        S.solve(p, f, P.FasParams(1e-9, 5, 2, 3))
        outs.append(host(p.data))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n,dim,loc,bc", [
    (64, 3, "cell", "dirichlet"), (64, 3, "edge_tb", "lid"), (128, 3, "cell", "mixed"),
    (512, 2, "cell", "dirichlet"), (256, 2, "edge_ns", "periodic"),
])
def test_solver_vs_oracle_larger(P, n, dim, loc, bc):
    """Bitwise field parity with the CPU oracle at sizes beyond the golden
    set (the oracle is itself pinned to the reference)."""
    import oracle as O
    shape = (n,) * dim
    ml = int(np.log2(n)) - 1
    halo = 1
    p0 = C.rand_field(11, shape, loc, halo)
    f0 = C.rand_field(12, shape, loc, halo)
    faces = C.bc_faces(dim, bc)
    op = O.OField(shape, loc, halo, p0.copy())
    of = O.OField(shape, loc, halo, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, 1.0, 0.5, faces, O.plan_colors("x", dim), 1e-30, 3, 2, ml)
    O.set_threads(1)
    g = P.unit_grid(shape)
    L = loc_of(P, loc)
    p = P.Field(g, L, halo, p0.copy())
    f = P.Field(g, L, halo, f0.copy())
    _, rep = P.solve(p, f, P.OperatorCoeffs(1.0, 0.5), P.FasParams(1e-30, 3, 2, ml),
                     P.make_plan("x", dim), bc_of(P, dim, bc))
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(host(p.data).view(np.uint64), op.data.view(np.uint64))


@pytest.mark.parametrize("shape", [(34, 34, 34), (66, 130, 18), (10, 10, 10), (130, 258), (7, 9, 11),
                                   (1026, 34)])
def test_view_sum_tree_and_serial_paths(P, shape):
    """Ordered (numpy 2.3 buffered-pairwise) interior sum on the device vs the
    oracle restatement, for chunk lengths that take the parallel-tree path
    (128*2^k) and ones that take the serial path."""
    import oracle as O
    from paper_2510_11152_b200.grid import view_sum
    a = np.random.default_rng(sum(shape)).standard_normal(shape)
    inner = tuple(slice(1, s - 1) for s in shape)
    got = float(view_sum(dev(a)[inner]).item())
    assert got == float(O.view_sum(a[inner]))


@pytest.mark.parametrize("c", cases("weno"), ids=lambda c: c["key"])
def test_weno3_convect_api(P, c):
    """The public weno3_convect (fused one-pass kernel) against the
    reference's weno3_convect on the same halo-2 velocities, bitwise."""
    n = tuple(c["n"])
    g = P.unit_grid(n)
    locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
    vel = []
    for t, loc in enumerate(locs):
        F = P.Field(g, loc_of(P, loc), 2, C.rand_field(c["seed"] + 10 * t, n, loc, 2))
        F.ghosts_fresh = True
        vel.append(F)
    res = P.weno3_convect(tuple(vel), c["target"])
    expect_array(f"{c['key']}/conv", host(res.interior))
    assert not res.ghosts_fresh


@pytest.mark.parametrize("c", cases("reduce"), ids=lambda c: c["key"])
def test_norm_l2_scaled_numpy_order(P, c):
    """The public norm_l2_scaled sums squares in numpy's flat pairwise
    order: the sum of squares is the reference's bitwise, on a Field and on
    a bare device array."""
    G = golden()
    a = np.random.default_rng(c["seed"]).standard_normal(c["shape"])
    t = dev(a)
    v = t[tuple(slice(1, s - 1) for s in c["shape"])]
    from paper_2510_11152_b200.grid import view_sumsq
    assert float(view_sumsq(v).item()) == float(G[f"{c['key']}/sumsq"])
    n = tuple(s - 2 for s in c["shape"])
    g = P.GridLevel(0, n, (0.0,) * len(n), tuple(x / n[-1] for x in n))
    F = P.Field(g, P.Location.CELL, 1, a)
    ref = g.h ** (g.dim / 2.0) * np.sqrt(float(G[f"{c['key']}/sumsq"]))
    assert P.norm_l2_scaled(F) == ref
    assert P.norm_l2_scaled(v, g) == ref


@pytest.mark.parametrize("c", C.DENSE_CASES, ids=C.dense_key)
def test_assemble_dense_operator(P, c):
    """stencil.assemble_dense_operator (probed from the device operator)
    against the reference's row-wise assembly (PKG/stencil.py:172-215)."""
    from paper_2510_11152_b200.stencil import assemble_dense_operator
    dim = len(c["n"])
    g = P.unit_grid(tuple(c["n"]))
    mat = assemble_dense_operator(g, loc_of(P, c["loc"]), P.OperatorCoeffs(c["a"], c["b"]),
                                  bc_of(P, dim, c["bc"]))
    ref = golden()[C.dense_key(c)]
    assert mat.shape == ref.shape
    np.testing.assert_allclose(mat, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    assert np.array_equal(mat != 0, ref != 0)
