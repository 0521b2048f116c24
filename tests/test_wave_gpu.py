"""TMA-fed marching kernels (csrc/fasmg_wave.cuh): the 3D and 2D half-sweeps
and the coarse correction fused into the first post-smoothing half-sweep,
forced onto small levels (FASMG_TMA_MIN=0) so that the oracle finishes in
seconds: bitwise parity with the CPU oracle for every cell/edge location,
boundary kinds on every axis, partial tiles and ragged march chunks.
"""
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


LOC = {"cell": "CELL", "edge_ew": "EDGE_EW", "edge_ns": "EDGE_NS", "edge_tb": "EDGE_TB"}

FACES = {
    "dirichlet": None,
    "mixed_dn": {"xlo": ("dirichlet", 0.25), "xhi": ("neumann", 0.0),
                 "ylo": ("neumann", 0.0), "yhi": ("dirichlet", 0.5),
                 "zlo": ("dirichlet", -1.0), "zhi": ("neumann", 0.0)},
    "lid": None,
    # y periodic (in-plane wrap), x / z mixed Dirichlet values and Neumann
    "mixed_yz": {"xlo": ("dirichlet", 0.25), "xhi": ("neumann", 0.0),
                 "ylo": ("periodic", 0.0), "yhi": ("periodic", 0.0),
                 "zlo": ("neumann", 0.0), "zhi": ("dirichlet", -1.0)},
    "neumann_x": {"xlo": ("neumann", 0.0), "xhi": ("neumann", 0.0),
                  "ylo": ("dirichlet", 0.0), "yhi": ("dirichlet", 1.0),
                  "zlo": ("periodic", 0.0), "zhi": ("periodic", 0.0)},
}


def faces_of(spec):
    f = FACES[spec]
    return C.bc_faces(3, spec) if f is None else dict(f)


def bc_of(P, faces):
    return P.BoundaryCondition(3, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))


def run_gpu(P, monkeypatch, env, shape, loc, faces, p0, f0, ml, k_max):
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    if len(set(shape)) == 1:
        g = P.unit_grid(shape)
    else:  # uniform h on a box domain
        g = P.GridLevel(0, shape, (0.0,) * 3, tuple(s / shape[-1] for s in shape))
    L = getattr(P.Location, LOC[loc])
    p = P.Field(g, L, 1, p0.copy())
    f = P.Field(g, L, 1, f0.copy())
    _, rep = P.solve(p, f, P.OperatorCoeffs(1.0, 0.5), P.FasParams(1e-30, k_max, 2, ml),
                     P.make_plan("x", 3), bc_of(P, faces))
    torch.cuda.synchronize()
    return p.data.cpu().numpy(), rep


@pytest.mark.parametrize("shape,loc,spec", [
    ((64, 64, 64), "cell", "dirichlet"),
    ((48, 112, 80), "cell", "mixed_yz"),      # partial tile along b2
    ((64, 64, 96), "edge_ew", "lid"),
    ((64, 48, 64), "edge_ns", "neumann_x"),
    ((32, 64, 128), "edge_tb", "lid"),
])
def test_tma_sweep_vs_oracle(P, monkeypatch, shape, loc, spec):
    """k_sweep_tma (TMA-fed marching half-sweep) forced onto small levels:
    bitwise equal to the oracle, including partial edge tiles."""
    import oracle as O
    faces = faces_of(spec)
    ml = 3
    p0 = C.rand_field(41, shape, loc, 1)
    f0 = C.rand_field(42, shape, loc, 1)
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, 1.0, 0.5, faces, O.plan_colors("x", 3), 1e-30, 2, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    got, rep = run_gpu(P, monkeypatch, {"FASMG_TMA_MIN": 0, "FASMG_MARCH_CHUNK": 3}, shape, loc,
                       faces, p0, f0, ml, 2)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64))


@pytest.mark.parametrize("shape,loc,spec", [
    ((256, 256), "cell", "dirichlet"),
    ((128, 320), "cell", "mixed"),        # x periodic, partial tile along b1
    ((256, 128), "edge_ew", "lid"),
    ((128, 256), "edge_ns", "periodic"),
])
def test_tma_sweep_2d_vs_oracle(P, monkeypatch, shape, loc, spec):
    """k_sweep_tma2d forced onto small 2D levels: bitwise vs the oracle."""
    import oracle as O
    faces = C.bc_faces(2, spec)
    ml = 4
    p0 = C.rand_field(71, shape, loc, 1)
    f0 = C.rand_field(72, shape, loc, 1)
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, 1.0, 0.5, faces, O.plan_colors("x", 2), 1e-30, 2, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    for k, v in {"FASMG_TMA_MIN": 0, "FASMG_MARCH_CHUNK": 3}.items():
        monkeypatch.setenv(k, str(v))
    g = P.unit_grid(shape) if shape[0] == shape[1] else \
        P.GridLevel(0, shape, (0.0, 0.0), tuple(s / shape[-1] for s in shape))
    L = getattr(P.Location, LOC[loc])
    p = P.Field(g, L, 1, p0.copy())
    f = P.Field(g, L, 1, f0.copy())
    bc = P.BoundaryCondition(2, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))
    _, rep = P.solve(p, f, P.OperatorCoeffs(1.0, 0.5), P.FasParams(1e-30, 2, 2, ml),
                     P.make_plan("x", 2), bc)
    torch.cuda.synchronize()
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(p.data.cpu().numpy().view(np.uint64), op.data.view(np.uint64))


@pytest.mark.parametrize("shape,spec,env", [
    ((64, 64, 64), "dirichlet", {}),
    ((48, 112, 80), "mixed_dn", {}),
    ((96, 64, 128), "mixed_dn", {"FASMG_MARCH_CHUNK": 5}),
    ((64, 64, 64), "lid", {"FASMG_MARCH_CHUNK": 1}),
    ((64, 64, 64), "neumann", {}),
])
def test_fused_correction_vs_oracle(P, monkeypatch, shape, spec, env):
    """Coarse correction fused into the first post-smoothing half-sweep
    (k_sweep_tma<.., CORR>, pinit stored by the tau pass), forced onto small
    levels: fields bitwise equal to the oracle and to the unfused path."""
    import oracle as O
    faces = faces_of(spec) if spec in FACES else C.bc_faces(3, spec)
    a = 0.0 if spec == "neumann" else 1.0
    ml = 3
    p0 = C.rand_field(81, shape, "cell", 1)
    f0 = C.rand_field(82, shape, "cell", 1)
    op = O.OField(shape, "cell", 1, p0.copy())
    of = O.OField(shape, "cell", 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, a, 0.5, faces, O.plan_colors("x", 3), 1e-30, 3, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    e = {"FASMG_TMA_MIN": 0, **env}
    got, rep = run_gpu_a(P, monkeypatch, e, shape, faces, p0, f0, ml, 3, a)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64))
    off, _ = run_gpu_a(P, monkeypatch, {**e, "FASMG_CORR_FUSE": 0}, shape, faces, p0, f0, ml, 3, a)
    assert np.array_equal(got.view(np.uint64), off.view(np.uint64))


def run_gpu_a(P, monkeypatch, env, shape, faces, p0, f0, ml, k_max, a):
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    g = P.unit_grid(shape) if len(set(shape)) == 1 else \
        P.GridLevel(0, shape, (0.0,) * 3, tuple(s / shape[-1] for s in shape))
    p = P.Field(g, P.Location.CELL, 1, p0.copy())
    f = P.Field(g, P.Location.CELL, 1, f0.copy())
    _, rep = P.solve(p, f, P.OperatorCoeffs(a, 0.5), P.FasParams(1e-30, k_max, 2, ml),
                     P.make_plan("x", 3), bc_of(P, faces))
    torch.cuda.synchronize()
    return p.data.cpu().numpy(), rep


@pytest.mark.parametrize("shape,loc,spec,env", [
    ((64, 64, 64), "edge_ew", "lid", {}),
    ((64, 64, 64), "edge_ns", "lid", {}),
    ((64, 64, 64), "edge_tb", "lid", {}),
    ((48, 112, 80), "edge_ew", "mixed_dn", {}),                      # partial tiles, Neumann faces
    ((48, 112, 80), "edge_ns", "mixed_dn", {"FASMG_ETAU_CHUNK": 5}),  # ragged chunks
    ((96, 48, 80), "edge_tb", "mixed_dn", {"FASMG_ETAU_CHUNK": 3}),
    ((64, 64, 96), "edge_ns", "dirichlet", {"FASMG_ETAU_CHUNK": 1}),
    ((64, 64, 64), "edge_tb", "lid", {"FASMG_ETAU_CHUNK": 32}),       # one chunk: the axis-0 ghost
])
def test_edge_tau_march_vs_oracle(P, monkeypatch, shape, loc, spec, env):
    """Edge-field tau pass in one TMA march (k_tau_edge_tma: residual, both
    edge restrictions, pinit), forced onto small levels: fields bitwise equal
    to the oracle and to the unfused residual + pads + restriction kernels."""
    import oracle as O
    faces = faces_of(spec) if spec in FACES else C.bc_faces(3, spec)
    ml = 3
    p0 = C.rand_field(61, shape, loc, 1)
    f0 = C.rand_field(62, shape, loc, 1)
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, 1.0, 0.5, faces, O.plan_colors("x", 3), 1e-30, 2, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    e = {"FASMG_TMA_MIN": 0, **env}
    got, rep = run_gpu(P, monkeypatch, e, shape, loc, faces, p0, f0, ml, 2)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64))
    off, _ = run_gpu(P, monkeypatch, {**e, "FASMG_EDGE_TAU": 0}, shape, loc, faces, p0, f0, ml, 2)
    assert np.array_equal(got.view(np.uint64), off.view(np.uint64))


@pytest.mark.parametrize("shape,spec,env,a", [
    ((64, 64, 64), "dirichlet", {}, 1.0),
    ((48, 112, 80), "mixed_dn", {}, 1.0),                       # partial tiles, Neumann faces
    ((96, 64, 128), "mixed_dn", {"FASMG_MARCH_CHUNK": 5}, 1.0),  # ragged chunks
    ((64, 64, 64), "neumann", {}, 0.0),                          # singular (pressure-like)
    ((64, 64, 64), "lid", {"FASMG_CORR_FUSE": 0}, 1.0),
])
def test_speculative_first_sweep_vs_oracle(P, monkeypatch, shape, spec, env, a):
    """The outer norm also running the next V-cycle's first pre-smoothing
    half-sweep into a second buffer (k_resid_tma<2>, FASMG_SPEC), forced onto
    small levels over 4 V-cycles: fields bitwise equal to the oracle and to
    FASMG_SPEC=0, residual histories within 1e-10 / identical."""
    import oracle as O
    faces = faces_of(spec) if spec in FACES else C.bc_faces(3, spec)
    ml = 3
    p0 = C.rand_field(93, shape, "cell", 1)
    f0 = C.rand_field(94, shape, "cell", 1)
    op = O.OField(shape, "cell", 1, p0.copy())
    of = O.OField(shape, "cell", 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, a, 0.5, faces, O.plan_colors("x", 3), 1e-30, 4, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    e = {"FASMG_TMA_MIN": 0, **env}
    got, rep = run_gpu_a(P, monkeypatch, e, shape, faces, p0, f0, ml, 4, a)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64))
    off, rep2 = run_gpu_a(P, monkeypatch, {**e, "FASMG_SPEC": 0}, shape, faces, p0, f0, ml, 4, a)
    assert np.array_equal(got.view(np.uint64), off.view(np.uint64))
    assert rep.residual_history == rep2.residual_history


def test_speculation_state_transitions(P, monkeypatch):
    """Engine calls that read or replace the state while a speculative
    half-sweep is pending (store, the bare V-cycle, level copies, the
    residual, a new load) see exactly the non-speculative engine's values."""
    import ctypes
    from paper_2510_11152_b200 import _native as N
    monkeypatch.setenv("FASMG_TMA_MIN", "0")
    shape = (64, 64, 64)
    g = P.unit_grid(shape)
    p0 = C.rand_field(95, shape, "cell", 1)
    f0 = C.rand_field(96, shape, "cell", 1)
    outs = []
    for spec in ("1", "0"):
        monkeypatch.setenv("FASMG_SPEC", spec)
        S = P.FasSolver(P.make_hierarchy(g, 3), P.Location.CELL, P.BoundaryCondition.dirichlet(3),
                        P.make_plan("x", 3), P.OperatorCoeffs(1.0, 0.5))
        p = P.Field(g, P.Location.CELL, 1, p0.copy())
        f = P.Field(g, P.Location.CELL, 1, f0.copy())
        e = S.engine(2, p.device)
        e.load(p, f)
        r = [e.run(1, True), e.run(1, True)]
        e.store(p)                       # pending: the stored state is the real one
        rs = ctypes.c_double()
        N.call("fasmg_engine_residual_sumsq", e.handle, ctypes.byref(rs))  # cancels
        r.append(rs.value)
        r.append(e.run(2, True))
        e.run(1, False)                  # bare V-cycle after a pending norm
        r.append(e.run(1, True))
        q = P.Field(g, P.Location.CELL, 1, p0.copy())
        e.store(q)
        e.load(q, f)                     # a new load drops the speculation
        r.append(e.run(1, True))
        e.store(q)
        torch.cuda.synchronize()
        outs.append((p.data.cpu().numpy(), q.data.cpu().numpy(), r))
    assert np.array_equal(outs[0][0].view(np.uint64), outs[1][0].view(np.uint64))
    assert np.array_equal(outs[0][1].view(np.uint64), outs[1][1].view(np.uint64))
    np.testing.assert_allclose(outs[0][2], outs[1][2], rtol=1e-13, atol=0)


def run_gpu_loc(P, monkeypatch, env, shape, loc, faces, p0, f0, ml, k_max, a):
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    g = P.unit_grid(shape) if len(set(shape)) == 1 else \
        P.GridLevel(0, shape, (0.0,) * 3, tuple(s / shape[-1] for s in shape))
    L = getattr(P.Location, LOC[loc])
    p = P.Field(g, L, 1, p0.copy())
    f = P.Field(g, L, 1, f0.copy())
    _, rep = P.solve(p, f, P.OperatorCoeffs(a, 0.5), P.FasParams(1e-30, k_max, 2, ml),
                     P.make_plan("x", 3), bc_of(P, faces))
    torch.cuda.synchronize()
    return p.data.cpu().numpy(), rep


@pytest.mark.parametrize("shape,loc,spec,env,a", [
    ((64, 64, 64), "edge_ew", "lid", {}, 1.0),
    ((64, 64, 64), "edge_ns", "lid", {}, 1.0),
    ((64, 64, 64), "edge_tb", "lid", {}, 1.0),
    ((48, 112, 80), "edge_ew", "mixed_dn", {}, 1.0),                       # Neumann edge-axis wall
    ((48, 112, 80), "edge_ns", "mixed_dn", {"FASMG_MARCH_CHUNK": 5}, 1.0),  # ragged chunks
    ((96, 48, 80), "edge_tb", "mixed_dn", {"FASMG_MARCH_CHUNK": 3}, 1.0),
    ((64, 64, 96), "edge_ns", "dirichlet", {"FASMG_MARCH_CHUNK": 1}, 1.0),
    ((64, 64, 64), "edge_ew", "neumann", {}, 0.0),                         # singular
    ((64, 64, 64), "edge_tb", "lid", {"FASMG_CORR_CHUNK": 32}, 1.0),        # one chunk
])
def test_edge_fused_correction_vs_oracle(P, monkeypatch, shape, loc, spec, env, a):
    """Edge-field coarse correction fused into the first post-smoothing
    half-sweep (k_sweep_tma<EA, M, true>: the opposite-class boxes corrected
    in shared memory by the edge prolongation of Corr), forced onto small
    levels over 3 V-cycles: fields bitwise equal to the oracle and to the
    unfused k_correct_edge_fast + pad fill path, histories within 1e-10 /
    identical."""
    import oracle as O
    faces = faces_of(spec) if spec in FACES else C.bc_faces(3, spec)
    ml = 3
    p0 = C.rand_field(63, shape, loc, 1)
    f0 = C.rand_field(64, shape, loc, 1)
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, a, 0.5, faces, O.plan_colors("x", 3), 1e-30, 3, 2, ml,
                           dmin=0.0, dmax=shape[0] / shape[-1])
    O.set_threads(1)
    e = {"FASMG_TMA_MIN": 0, **env}
    got, rep = run_gpu_loc(P, monkeypatch, e, shape, loc, faces, p0, f0, ml, 3, a)
    np.testing.assert_allclose(rep.residual_history, hist, rtol=HIST_RTOL, atol=0)
    assert np.array_equal(got.view(np.uint64), op.data.view(np.uint64))
    off, rep2 = run_gpu_loc(P, monkeypatch, {**e, "FASMG_CORR_FUSE": 0}, shape, loc, faces, p0,
                            f0, ml, 3, a)
    assert np.array_equal(got.view(np.uint64), off.view(np.uint64))
    assert rep.residual_history == rep2.residual_history
