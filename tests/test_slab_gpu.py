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


@pytest.mark.parametrize("tma_min,loc,bc", [("0", "cell", "dirichlet"), ("2097152", "cell", "dirichlet"),
                                            ("0", "edge_ew", "dirichlet"),
                                            ("2097152", "edge_ns", "dirichlet"),
                                            ("2097152", "cell", "neumann")])
def test_two_process_slabs_ipc(tma_min, loc, bc):
    """Two processes (one slab each, sharing the device through CUDA IPC
    peer pointers) run scripts/dist_selftest.py: each rank's slab bitwise
    equal to the single-engine solve."""
    import os, subprocess, sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SELFTEST_N="128", FASMG_TMA_MIN=tma_min, SELFTEST_LOC=loc,
               SELFTEST_BC=bc)
    port = 29600 + int(tma_min != "0") + 2 * ["cell", "edge_ew", "edge_ns"].index(loc) + \
        10 * (bc == "neumann")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "scripts", "dist_selftest.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("field bitwise True, history True") == 2, r.stdout


@pytest.mark.parametrize("loc,n,dim,parts,bc,halo,tma_min", [
    ("edge_ew", 64, 3, 2, "dirichlet", 1, None), ("edge_ew", 64, 3, 4, "lid", 2, None),
    ("edge_ns", 64, 3, 2, "dirichlet", 1, None), ("edge_tb", 64, 3, 4, "lid", 2, None),
    ("edge_ew", 128, 3, 4, "neumann_a1", 1, "0"), ("edge_ns", 128, 3, 8, "lid", 2, "0"),
    ("edge_tb", 128, 3, 2, "dirichlet_val", 1, "0"),
    ("edge_ew", 256, 2, 4, "dirichlet", 1, None), ("edge_ns", 256, 2, 4, "lid", 2, None),
])
def test_virtual_slabs_edge_fields(P, monkeypatch, loc, n, dim, parts, bc, halo, tma_min):
    """Edge-centred (MAC face-velocity) fields on axis-0 slabs -- the edge
    axis along the slab axis (edge_ew: the interface node belongs to the
    lower rank) or tangential to it (the residual's halo plane is exchanged
    for the tangential restriction): bitwise equal to the single engine."""
    import cases as C
    from paper_2510_11152_b200.slab import VirtualSlabSolver
    if tma_min is not None:
        monkeypatch.setenv("FASMG_TMA_MIN", tma_min)
    shape = (n,) * dim
    spec = "neumann" if bc == "neumann_a1" else bc
    faces = C.bc_faces(dim, spec)
    bcond = P.BoundaryCondition(dim, tuple((k, P.FaceRule(*v)) for k, v in faces.items()))
    L = getattr(P.Location, loc.upper())
    ml = int(np.log2(n)) - 1
    p0 = C.rand_field(31, shape, loc, halo)
    f0 = C.rand_field(32, shape, loc, halo)
    g = P.unit_grid(shape)
    coeffs = P.OperatorCoeffs(1.0, 0.05 if bc == "lid" else 0.5)
    plan = P.make_plan("x", dim)
    params = P.FasParams(1e-30, 3, 2, ml)
    p1 = P.Field(g, L, halo, p0.copy())
    f1 = P.Field(g, L, halo, f0.copy())
    rep1 = P.FasSolver(P.make_hierarchy(g, ml), L, bcond, plan, coeffs).solve(p1, f1, params)
    p2 = P.Field(g, L, halo, p0.copy())
    f2 = P.Field(g, L, halo, f0.copy())
    vs = VirtualSlabSolver(P.make_hierarchy(g, ml), L, bcond, plan, coeffs, parts)
    rep2 = vs.solve(p2, f2, params)
    assert all(e.kg >= 1 for e in vs.engines(params.s, p2.device))  # levels really split
    np.testing.assert_allclose(rep2.residual_history, rep1.residual_history, rtol=1e-12)
    assert torch.equal(p1.interior, p2.interior)
    assert torch.equal(p1.data, p2.data)


@pytest.mark.parametrize("loc,bc", [("cell", "dirichlet"), ("cell", "neumann"),
                                    ("edge_ew", "dirichlet"), ("edge_tb", "dirichlet")])
def test_four_process_slabs_ipc(loc, bc):
    """Four processes at 64^3 (16 cells per slab): the two interior ranks
    have a neighbour on both sides across processes, so every send/receive
    ordering of the counter protocol is exercised; each rank's slab is
    bitwise equal to the single-engine solve."""
    import os, subprocess, sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SELFTEST_N="64", SELFTEST_LOC=loc, SELFTEST_BC=bc)
    port = 29640 + ["cell", "edge_ew", "edge_tb"].index(loc) + 5 * (bc == "neumann")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "scripts", "dist_selftest.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("field bitwise True, history True") == 4, r.stdout
