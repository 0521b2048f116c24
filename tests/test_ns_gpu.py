"""Projection steppers on the GPU vs the composed CPU oracle
(oracle/ns_oracle.py), and classical vs memory-efficient schedules."""
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


def _stepper(P, n, order, mode, dt=1e-2, re=100.0):
    from paper_2510_11152_b200.ns import NSParams, ProjectionStepper, cavity_bcs
    g = P.unit_grid(n)
    st = ProjectionStepper(g, NSParams(re=re, dt=dt, order=order, mode=mode, tol=1e-10, k_max=20))
    st.set_state({})
    return st


@pytest.mark.parametrize("n,order", [((16, 16), 1), ((16, 16), 2), ((8, 8, 8), 1), ((8, 8, 8), 2)])
def test_ns_matches_oracle(P, n, order):
    import ns_oracle as NO
    st = _stepper(P, n, order, "efficient")
    orc = NO.NSOracle(n, 100.0, 1e-2, order)
    for k in range(3):
        rep = st.step()
        hist = orc.step()
        for c in st.comps:
            np.testing.assert_allclose(rep.momentum[c].residual_history, hist[c], rtol=1e-10)
        np.testing.assert_allclose(rep.pressure.residual_history, hist["p"], rtol=1e-10)
        for c in st.comps:
            got = st.velocity(c).numpy()
            assert np.array_equal(got.view(np.uint64), orc.un[c].data.view(np.uint64)), (k, c)
        gp = st.pressure().interior.cpu().numpy()
        assert np.array_equal(gp, orc.p.interior), k


@pytest.mark.parametrize("dim,order", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_classical_equals_efficient(P, dim, order):
    n = (16,) * dim if dim == 2 else (8,) * 3
    a = _stepper(P, n, order, "efficient")
    b = _stepper(P, n, order, "classical")
    assert a.resident_count() == 2 * dim + 2
    assert b.resident_count() == (3 if order == 1 else 4) * dim + 3
    for _ in range(3):
        a.step()
        b.step()
    for c in a.comps:
        assert torch.equal(a.velocity(c).interior, b.velocity(c).interior)
    assert torch.equal(a.pressure().interior, b.pressure().interior)


def test_divergence_free_after_projection(P):
    st = _stepper(P, (32, 32), 2, "efficient")
    for _ in range(5):
        st.step()
        assert abs(st.divergence()) <= 1e-12


@pytest.mark.parametrize("order", [1, 2])
def test_ns_3d_32_matches_oracle(P, order):
    """Medium-size 3D cavity (32^3, mesh level 4): momentum and pressure
    residual histories within 1e-10 and bitwise fields after 2 steps."""
    import ns_oracle as NO
    import oracle as O
    st = _stepper(P, (32, 32, 32), order, "efficient", dt=1e-3)
    O.set_threads(8)
    orc = NO.NSOracle((32, 32, 32), 100.0, 1e-3, order)
    try:
        for k in range(2):
            rep = st.step()
            hist = orc.step()
            for c in st.comps:
                np.testing.assert_allclose(rep.momentum[c].residual_history, hist[c], rtol=1e-10)
            np.testing.assert_allclose(rep.pressure.residual_history, hist["p"], rtol=1e-10)
            for c in st.comps:
                got = st.velocity(c).numpy()
                assert np.array_equal(got.view(np.uint64), orc.un[c].data.view(np.uint64)), (k, c)
    finally:
        O.set_threads(1)


@pytest.mark.parametrize("dim,n", [(2, (24, 16)), (3, (8, 12, 16))])
def test_weno_fused_equals_per_axis(P, dim, n):
    """fasmg_weno_convect (one pass, winds in place) is bitwise the
    reference's per-axis kernel sequence, for every target component."""
    from paper_2510_11152_b200.weno import weno3_convect
    g = P.GridLevel(0, n, (0.0,) * dim, tuple(x / n[-1] for x in n))
    locs = [P.Location.EDGE_EW, P.Location.EDGE_NS, P.Location.EDGE_TB][:dim]
    rng = np.random.default_rng(dim)
    vel = []
    for L in locs:
        F = P.Field(g, L, 2)
        F.data.copy_(torch.from_numpy(rng.standard_normal(tuple(F.data.shape))))
        F.ghosts_fresh = True
        vel.append(F)
    for t in range(dim):
        a = weno3_convect(tuple(vel), t, fused=True).interior.cpu().numpy()
        b = weno3_convect(tuple(vel), t, fused=False).interior.cpu().numpy()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), t


@pytest.mark.parametrize("c", __import__("cases").NS_CASES, ids=__import__("cases").ns_key)
def test_ns_matches_reference_composition(P, c):
    """GPU stepper against projection steps composed from the REAL reference
    primitives (tests/golden/make_golden_r2.py): histories within 1e-10,
    velocity (with ghosts) and pressure fields bitwise, every step."""
    from _golden import expect_array, golden
    import cases as C
    G = golden()
    key = C.ns_key(c)
    st = _stepper(P, tuple(c["n"]), c["order"], "efficient", dt=c["dt"], re=c["re"])
    for s in range(c["steps"]):
        rep = st.step()
        for k in st.comps:
            np.testing.assert_allclose(rep.momentum[k].residual_history,
                                       G[f"{key}/s{s}/hist_{k}"], rtol=1e-10, atol=0)
        np.testing.assert_allclose(rep.pressure.residual_history, G[f"{key}/s{s}/hist_p"],
                                   rtol=1e-10, atol=0)
        for k in st.comps:
            expect_array(f"{key}/s{s}/{k}", st.velocity(k).numpy())
        expect_array(f"{key}/s{s}/p", st.pressure().interior.cpu().numpy())


def _host_mem_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 0.0


@pytest.mark.slow
def test_ns_512_config4_matches_oracle(P):
    """BASELINE.json configs[3] at full size: 3D lid-driven cavity 512^3,
    second-order projection, memory-efficient 8-slot schedule, Re 100,
    dt 1e-3, tol 1e-10, kMax 20, s 2, meshLevel 8.  Two steps on the GPU
    against the pinned NS oracle (oracle/ns_oracle.py, C kernels on all host
    threads): every momentum/pressure residual history within 1e-10 and
    the velocity and pressure fields bitwise after each step."""
    import os
    import ns_oracle as NO
    import oracle as O
    if _host_mem_gb() < 40:
        pytest.skip(f"the 512^3 CPU oracle needs ~30 GB of host RAM ({_host_mem_gb():.0f} GB free)")
    n = (512, 512, 512)
    from paper_2510_11152_b200.ns import NSParams, ProjectionStepper
    st = ProjectionStepper(P.unit_grid(n), NSParams(re=100.0, dt=1e-3, order=2, mode="efficient",
                                                    tol=1e-10, k_max=20, s=2, mesh_level=8))
    st.set_state({})
    O.set_threads(len(os.sched_getaffinity(0)))
    orc = NO.NSOracle(n, 100.0, 1e-3, 2, tol=1e-10, k_max=20, s=2, mesh_level=8)
    try:
        for k in range(2):
            rep = st.step()
            hist = orc.step()
            for c in st.comps:
                np.testing.assert_allclose(rep.momentum[c].residual_history, hist[c],
                                           rtol=1e-10, atol=0)
            np.testing.assert_allclose(rep.pressure.residual_history, hist["p"], rtol=1e-10,
                                       atol=0)
            for c in st.comps:
                got = st.velocity(c).data
                ref = torch.from_numpy(orc.un[c].data).to(got.device)
                assert torch.equal(got.view(torch.int64), ref.view(torch.int64)), (k, c)
                del ref
            gp = st.pressure().interior
            ref = torch.from_numpy(np.ascontiguousarray(orc.p.interior)).to(gp.device)
            assert torch.equal(gp.contiguous().view(torch.int64), ref.view(torch.int64)), k
            del ref
    finally:
        O.set_threads(1)
