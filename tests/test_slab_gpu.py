"""Axis-0 slab decomposition with virtual ranks on one GPU: bitwise field
parity with the single-engine solve."""
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


@pytest.mark.parametrize("n,dim,parts,bc,a", [
    (64, 3, 2, "dirichlet", 1.0), (64, 3, 4, "dirichlet", 1.0), (128, 3, 4, "mixed", 1.0),
    (64, 3, 2, "neumann", 0.0), (256, 2, 4, "dirichlet", 1.0), (128, 3, 8, "dirichlet", 1.0),
])
def test_virtual_slabs_match_single(P, n, dim, parts, bc, a):
    import cases as C
    from paper_2510_11152_b200.slab import VirtualSlabSolver
    shape = (n,) * dim
    faces = C.bc_faces(dim, bc)
    if bc == "mixed":  # x periodic is not slab-able: make x dirichlet
        faces["xlo"] = ("dirichlet", 0.25)
        faces["xhi"] = ("neumann", 0.0)
    bcond = P.BoundaryCondition(dim, tuple((k, P.FaceRule(*v)) for k, v in faces.items()))
    ml = int(np.log2(n)) - 1
    p0 = C.rand_field(21, shape, "cell", 1)
    f0 = C.rand_field(22, shape, "cell", 1)
    g = P.unit_grid(shape)
    coeffs = P.OperatorCoeffs(a, 0.5)
    plan = P.make_plan("x", dim)
    params = P.FasParams(1e-30, 4, 2, ml)
    p1 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f1 = P.Field(g, P.Location.CELL, 1, f0.copy())
    rep1 = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bcond, plan, coeffs).solve(p1, f1, params)
    p2 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f2 = P.Field(g, P.Location.CELL, 1, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bcond, plan, coeffs, parts)
    rep2 = vs.solve(p2, f2, params)
    np.testing.assert_allclose(rep2.residual_history, rep1.residual_history, rtol=1e-12)
    assert torch.equal(p1.data, p2.data)
    assert torch.equal(f1.data, f2.data)


@pytest.mark.parametrize("n,parts", [(128, 2), (128, 4), (128, 8), (256, 8)])
def test_virtual_slabs_tma_levels(P, monkeypatch, n, parts):
    """Sharded levels on the TMA march (FASMG_TMA_MIN=0 forces it onto small
    slabs): bitwise equal to the single-engine solve."""
    from paper_2510_11152_b200.slab import VirtualSlabSolver
    import cases as C
    monkeypatch.setenv("FASMG_TMA_MIN", "0")
    shape = (n,) * 3
    ml = int(np.log2(n)) - 1
    p0 = C.rand_field(61, shape, "cell", 1)
    f0 = C.rand_field(62, shape, "cell", 1)
    g = P.unit_grid(shape)
    bc = P.BoundaryCondition.dirichlet(3)
    coeffs = P.OperatorCoeffs(1.0, 0.5)
    plan = P.make_plan("x", 3)
    params = P.FasParams(1e-30, 2, 2, ml)
    p1 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f1 = P.Field(g, P.Location.CELL, 1, f0.copy())
    rep1 = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs).solve(p1, f1, params)
    p2 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f2 = P.Field(g, P.Location.CELL, 1, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs, parts)
    rep2 = vs.solve(p2, f2, params)
    np.testing.assert_allclose(rep2.residual_history, rep1.residual_history, rtol=1e-12)
    assert torch.equal(p1.data, p2.data)


@pytest.mark.parametrize("fuse", ["0", "1"])
def test_virtual_slabs_push_modes(P, monkeypatch, fuse):
    """Halo push as a separate kernel (FASMG_FUSE_PUSH=0) and fused into the
    sweep kernels (default): both bitwise equal to the single-engine solve."""
    from paper_2510_11152_b200.slab import VirtualSlabSolver
    import cases as C
    monkeypatch.setenv("FASMG_FUSE_PUSH", fuse)
    monkeypatch.setenv("FASMG_TMA_MIN", "0")
    n, parts = 128, 4
    shape = (n,) * 3
    ml = int(np.log2(n)) - 1
    p0 = C.rand_field(71, shape, "cell", 1)
    f0 = C.rand_field(72, shape, "cell", 1)
    g = P.unit_grid(shape)
    bc = P.BoundaryCondition.dirichlet(3)
    coeffs = P.OperatorCoeffs(1.0, 0.5)
    plan = P.make_plan("x", 3)
    params = P.FasParams(1e-30, 2, 2, ml)
    p1 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f1 = P.Field(g, P.Location.CELL, 1, f0.copy())
    rep1 = P.FasSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs).solve(p1, f1, params)
    p2 = P.Field(g, P.Location.CELL, 1, p0.copy())
    f2 = P.Field(g, P.Location.CELL, 1, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), P.Location.CELL, bc, plan, coeffs, parts)
    rep2 = vs.solve(p2, f2, params)
    np.testing.assert_allclose(rep2.residual_history, rep1.residual_history, rtol=1e-12)
    assert torch.equal(p1.data, p2.data)


@pytest.mark.parametrize("tma_min", ["0", "2097152"])
def test_two_process_slabs_ipc(tma_min):
    """Two processes (one slab each, sharing the device through CUDA IPC
    peer pointers) run scripts/dist_selftest.py: each rank's slab bitwise
    equal to the single-engine solve."""
    import os, subprocess, sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SELFTEST_N="128", FASMG_TMA_MIN=tma_min)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + int(tma_min != "0")),
           os.path.join(root, "scripts", "dist_selftest.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("field bitwise True, history True") == 2, r.stdout
