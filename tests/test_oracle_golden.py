"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference package itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import cases as C
import oracle as O
from _golden import cases, digest, expect_array, golden


@pytest.mark.parametrize("c", cases("kernel"), ids=lambda c: c["key"])
def test_kernel(c):
    arrays, sc = C.kernel_inputs(c)
    C.run_kernel(O.KERNELS, c, arrays, sc)
    for nm, a in arrays.items():
        expect_array(f"{c['key']}/{nm}", a)


@pytest.mark.parametrize("c", cases("fill"), ids=lambda c: c["key"])
def test_fill(c):
    n = tuple(c["n"])
    F = O.OField(n, c["loc"], c["halo"], C.rand_field(c["seed"], n, c["loc"], c["halo"]))
    O.fill_ghosts(F, C.bc_faces(c["dim"], c["bc"]))
    expect_array(f"{c['key']}/data", F.data)


@pytest.mark.parametrize("c", cases("smooth"), ids=lambda c: c["key"])
def test_smooth(c):
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    p = O.OField(n, loc, halo, C.rand_field(c["seed"], n, loc, halo))
    f = O.OField(n, loc, halo, C.rand_field(c["seed"] + 1, n, loc, halo))
    colors = O.plan_colors(c["plan"][0], c["dim"], c["plan"][1])
    O.smooth(f, p, c["a"], c["b"], colors, C.bc_faces(c["dim"], c["bc"]))
    expect_array(f"{c['key']}/p", p.data)


@pytest.mark.parametrize("c", cases("weno"), ids=lambda c: c["key"])
def test_weno(c):
    n = tuple(c["n"])
    locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
    vel = [O.OField(n, loc, 2, C.rand_field(c["seed"] + 10 * t, n, loc, 2))
           for t, loc in enumerate(locs)]
    expect_array(f"{c['key']}/conv", O.weno3_convect(vel, c["target"]))


@pytest.mark.parametrize("c", cases("stag"), ids=lambda c: c["key"])
def test_staggered(c):
    n = tuple(c["n"])
    p = O.OField(n, "cell", 1, C.rand_field(c["seed"], n, "cell", 1))
    for ax in range(c["dim"]):
        expect_array(f"{c['key']}/grad{ax}", O.gradient_axis(p, ax))
    locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
    comps = [O.OField(n, loc, 2, C.rand_field(c["seed"] + 1 + t, n, loc, 2))
             for t, loc in enumerate(locs)]
    expect_array(f"{c['key']}/div", O.divergence_edges_to_cc(comps))


@pytest.mark.parametrize("c", cases("reduce"), ids=lambda c: c["key"])
def test_reductions(c):
    G = golden()
    a = np.random.default_rng(c["seed"]).standard_normal(c["shape"])
    v = a[tuple(slice(1, s - 1) for s in c["shape"])]
    assert O.view_sum(v) == float(G[f"{c['key']}/sum"])
    assert O.view_sum(v) / v.size == float(G[f"{c['key']}/mean"])
    assert O.lib().or_pairwise_sum(
        O._ptr(np.ascontiguousarray(v * v)), (v * v).size) == float(G[f"{c['key']}/sumsq"])


def _solve_case(c):
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    p0, f0 = C.solve_inputs(c, O.manufactured)
    p = O.OField(n, loc, halo, p0.copy())
    f = O.OField(n, loc, halo, f0.copy())
    dmax = c.get("domain", (1.0,))[0]
    colors = O.plan_colors(c["plan"][0], c["dim"], c["plan"][1])
    it, hist = O.fas_solve(p, f, c["a"], c["b"], C.bc_faces(c["dim"], c["bc"]),
                           colors, c["tol"], c["k_max"], c["s"], c["mesh_level"],
                           0.0, dmax)
    return p, f, it, hist, p0, f0, colors, dmax


@pytest.mark.parametrize("c", cases("solve"), ids=lambda c: c["key"])
def test_solve(c):
    G = golden()
    key = c["key"]
    if c["rhs"] in ("discrete", "continuous"):
        assert digest(O.manufactured(c["rhs"], c["n"])) == str(G[f"{key}/rhs_sha256"])
    p, f, it, hist, p0, f0, colors, dmax = _solve_case(c)
    assert it == int(G[f"{key}/iterations"])
    np.testing.assert_array_equal(np.array(hist), G[f"{key}/history"])
    assert digest(p.data) == str(G[f"{key}/p_sha256"])
    assert digest(f.data) == str(G[f"{key}/f_sha256"])
    # bare V-cycle
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    p1 = O.OField(n, loc, halo, p0.copy())
    f1 = O.OField(n, loc, halo, f0.copy())
    O.fas_solve(p1, f1, c["a"], c["b"], C.bc_faces(c["dim"], c["bc"]), colors,
                c["tol"], 1, c["s"], c["mesh_level"], 0.0, dmax, vcycle_only=True)
    assert digest(p1.data) == str(G[f"{key}/vcycle_p_sha256"])


def test_threads_do_not_change_results():
    c = [x for x in cases("solve") if x["name"] == "heat_3d_16"][0]
    O.set_threads(4)
    try:
        p, *_ = _solve_case(c)
    finally:
        O.set_threads(1)
    assert digest(p.data) == str(golden()[f"{c['key']}/p_sha256"])


def test_paper_asymptotic_3d_32():
    """PAPER.md:442 (Table err_3D): 32^3 error 1.74e-3."""
    c = [x for x in cases("solve") if x["name"] == "asym_3d_32"][0]
    p, *_ = _solve_case(c)
    e = p.interior - O.manufactured("exact", c["n"])
    assert float(np.max(np.abs(e))) == float(golden()[f"{c['key']}/err_max"])
    err = (1.0 / 32) ** 1.5 * np.sqrt(np.sum(e * e))  # scaled L2 error
    assert abs(err - 1.74e-3) / 1.74e-3 < 0.01


@pytest.mark.parametrize("c", C.NS_CASES, ids=C.ns_key)
def test_ns_oracle_vs_reference_composition(c):
    """oracle/ns_oracle.py against projection steps composed from the REAL
    reference primitives (tests/golden/make_golden_r2.py): residual
    histories and fields bitwise, step by step."""
    import ns_oracle as NO
    G = golden()
    key = C.ns_key(c)
    orc = NO.NSOracle(tuple(c["n"]), c["re"], c["dt"], c["order"])
    for s in range(c["steps"]):
        hist = orc.step()
        for k in orc.comps + ("p",):
            assert hist[k] == G[f"{key}/s{s}/hist_{k}"].tolist(), (s, k)
        for k in orc.comps:
            expect_array(f"{key}/s{s}/{k}", orc.un[k].data)
        expect_array(f"{key}/s{s}/p", orc.p.interior)
