"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over the kernels the V-cycle depends on:
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py CASE
CASE: tma (TMA march + CORR sweep + k_resid_tma, 3D cell, forced onto a
64^3 level), edge (edge-field V-cycle with the edge transfers), d2 (2D TMA
march), ns (two 16^3 projection steps).  Each solve case checks its field
against the oracle, so a sanitizer run also proves the result.  (Slab
ranks need concurrent kernels, which the sanitizer serialises inside a
process: scripts/gpu_r02c.sh runs them as 2 processes, each under its own
sanitizer.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases as C  # noqa: E402
import oracle as O  # noqa: E402
import paper_2510_11152_b200 as P  # noqa: E402


def solve_gpu(shape, loc, faces, p0, f0, ml, k_max, a=1.0, b=0.5):
    g = P.unit_grid(shape) if len(set(shape)) == 1 else \
        P.GridLevel(0, shape, (0.0,) * len(shape), tuple(s / shape[-1] for s in shape))
    L = getattr(P.Location, loc.upper())
    p = P.Field(g, L, 1, p0.copy())
    f = P.Field(g, L, 1, f0.copy())
    bc = P.BoundaryCondition(len(shape), tuple((nm, P.FaceRule(k, v)) for nm, (k, v) in faces.items()))
    _, rep = P.solve(p, f, P.OperatorCoeffs(a, b), P.FasParams(1e-30, k_max, 2, ml),
                     P.make_plan("x", len(shape)), bc)
    torch.cuda.synchronize()
    return p.data.cpu().numpy(), rep


def solve_oracle(shape, loc, faces, p0, f0, ml, k_max, a=1.0, b=0.5):
    op = O.OField(shape, loc, 1, p0.copy())
    of = O.OField(shape, loc, 1, f0.copy())
    O.set_threads(8)
    O.fas_solve(op, of, a, b, faces, O.plan_colors("x", len(shape)), 1e-30, k_max, 2, ml,
                dmin=0.0, dmax=shape[0] / shape[-1])
    return op.data


def check(shape, loc, spec, ml=3, k_max=2):
    faces = C.bc_faces(len(shape), spec)
    p0 = C.rand_field(11, shape, loc, 1)
    f0 = C.rand_field(12, shape, loc, 1)
    got, _ = solve_gpu(shape, loc, faces, p0, f0, ml, k_max)
    want = solve_oracle(shape, loc, faces, p0, f0, ml, k_max)
    ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
    print(f"{loc} {shape} {spec}: bitwise {ok}", flush=True)
    return ok


def main(case):
    os.environ.setdefault("FASMG_TMA_MIN", "0")
    os.environ.setdefault("FASMG_MARCH_CHUNK", "3")
    ok = True
    if case == "tma":
        ok &= check((64, 64, 64), "cell", "dirichlet")
        ok &= check((48, 64, 80), "cell", "mixed")
    elif case == "edge":
        ok &= check((32, 32, 32), "edge_ew", "lid")
        ok &= check((32, 32, 32), "edge_tb", "lid")
    elif case == "d2":
        ok &= check((128, 128), "cell", "dirichlet", ml=4)
        ok &= check((128, 128), "edge_ns", "periodic", ml=4)
    elif case == "ns":
        from paper_2510_11152_b200.ns import NSParams, ProjectionStepper
        st = ProjectionStepper(P.unit_grid((16, 16, 16)),
                               NSParams(re=100.0, dt=1e-3, order=2, tol=1e-10, k_max=20))
        st.set_state({})
        for _ in range(2):
            st.step()
        torch.cuda.synchronize()
        print("ns 16^3: 2 steps, divergence", st.divergence(), flush=True)
    else:
        raise SystemExit(f"unknown case {case}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main(sys.argv[1])
