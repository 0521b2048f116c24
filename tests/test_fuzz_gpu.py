"""Randomised configurations through the public solve() API with every
B200 fast path forced on small levels (TMA march, TMA residuals, fused
correction, coarse cluster kernel, pad-materialised edge transfers):
fields bitwise equal to the CPU oracle, residual histories within 1e-10."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cases as C  # noqa: E402

pytestmark = pytest.mark.gpu

LOCS3 = ("cell", "cell", "edge_ew", "edge_ns", "edge_tb")
FACE = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")
LOCNAME = {"cell": "CELL", "edge_ew": "EDGE_EW", "edge_ns": "EDGE_NS", "edge_tb": "EDGE_TB"}


def config(seed):
    rng = np.random.default_rng(1000 + seed)
    ml = int(rng.integers(2, 4))
    unit = 2 ** (ml + 1)
    # the last axis >= 64 cells so the TMA kernels (32-block tiles) engage
    shape = (int(unit * rng.integers(2, 7)), int(unit * rng.integers(2, 7)),
             int(max(64, unit * rng.integers(4, 9))))
    shape = tuple(((n + unit - 1) // unit) * unit for n in shape)
    loc = LOCS3[int(rng.integers(len(LOCS3)))]
    faces = {}
    for a in range(3):
        kind = ("dirichlet", "neumann", "periodic")[int(rng.integers(3))]
        if kind == "periodic":
            faces[FACE[2 * a]] = faces[FACE[2 * a + 1]] = ("periodic", 0.0)
        else:
            for sd in range(2):
                k2 = ("dirichlet", "neumann")[int(rng.integers(2))]
                faces[FACE[2 * a + sd]] = (k2, float(np.round(rng.normal(), 3)) if k2 == "dirichlet" else 0.0)
    a = 1.0 if rng.random() < 0.8 else 0.0
    if a == 0.0 and any(k == "dirichlet" for k, _ in faces.values()):
        a = 1.0
    b = float(np.round(rng.uniform(0.1, 2.0), 3))
    env = {"FASMG_TMA_MIN": 0, "FASMG_COARSE_MAX": int(rng.choice([0, 64, 4096])),
           "FASMG_MARCH_CHUNK": int(rng.choice([1, 3, 4])),
           "FASMG_CORR_FUSE": int(rng.integers(2))}
    return shape, ml, loc, faces, a, b, env


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_solve_vs_oracle(monkeypatch, seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O
    import paper_2510_11152_b200 as P
    shape, ml, loc, faces, a, b, env = config(seed)
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    p0 = C.rand_field(2000 + seed, shape, loc, 1)
    f0 = C.rand_field(3000 + seed, shape, loc, 1)
    dmax = shape[0] / shape[-1]
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    it, hist = O.fas_solve(op, of, a, b, faces, O.plan_colors("x", 3), 1e-30, 2, 2, ml,
                           dmin=0.0, dmax=dmax)
    O.set_threads(1)
    g = P.GridLevel(0, shape, (0.0,) * 3, tuple(s / shape[-1] for s in shape))
    L = getattr(P.Location, LOCNAME[loc])
    p = P.Field(g, L, 1, p0.copy())
    f = P.Field(g, L, 1, f0.copy())
    bc = P.BoundaryCondition(3, tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))
    _, rep = P.solve(p, f, P.OperatorCoeffs(a, b), P.FasParams(1e-30, 2, 2, ml),
                     P.make_plan("x", 3), bc)
    torch.cuda.synchronize()
    np.testing.assert_allclose(rep.residual_history, hist, rtol=1e-10, atol=0)
    assert np.array_equal(p.data.cpu().numpy().view(np.uint64), op.data.view(np.uint64)), \
        (shape, ml, loc, faces, a, b, env)
    assert np.array_equal(f.data.cpu().numpy().view(np.uint64), of.data.view(np.uint64))
