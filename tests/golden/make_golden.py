"""Generate golden vectors by running the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference (``/root/reference/pkg``) is copied to a scratch directory
(its numba cache writes into the package dir) and imported from there with
``NUMBA_NUM_THREADS=1`` (the reference's parallel Gauss-Seidel ``prange``
with step 2 is rejected by numba 0.65).  Inputs
come from ``cases.py`` (numpy only); outputs are written to ``golden.npz``.
Large fields are stored as SHA-256 digests of their bytes; small ones in
full.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import cases as C  # noqa: E402

REF = "/root/reference/pkg"
FULL_LIMIT = 40_000  # elements stored in full; larger arrays as digests


def import_reference(backend="numba"):
    dst = os.path.join(tempfile.gettempdir(), "fasmg_ref_copy")
    if not os.path.exists(dst):
        shutil.copytree(REF, dst)
    os.environ.setdefault("NUMBA_NUM_THREADS", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(dst, "_nbcache"))
    os.environ["FASMG_BACKEND"] = backend
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.path.insert(0, os.path.join(dst, "src"))
    import fasmg  # noqa: F401
    return sys.modules["fasmg"]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_bc(fm, dim, spec):
    faces = C.bc_faces(dim, spec)
    return fm.BoundaryCondition(dim, tuple(
        (nm, fm.FaceRule(k, v)) for nm, (k, v) in faces.items()))


def ref_loc(fm, loc):
    return {"cell": fm.Location.CELL, "edge_ew": fm.Location.EDGE_EW,
            "edge_ns": fm.Location.EDGE_NS, "edge_tb": fm.Location.EDGE_TB}[loc]


def manufactured_ref(fm):
    from fasmg import manufactured as M

    def mk(kind, n):
        g = fm.unit_grid(tuple(n))
        if kind == "discrete":
            return M.poisson_rhs_discrete(g).interior.copy()
        if kind == "continuous":
            return M.poisson_rhs_continuous(g).interior.copy()
        if kind == "exact":
            return M.poisson_exact(g).interior.copy()
        raise ValueError(kind)
    return mk


def store(out, key, arr):
    arr = np.asarray(arr)
    if arr.size <= FULL_LIMIT:
        out[key] = arr
    else:
        out[key + "#sha256"] = np.array(digest(arr))
        out[key + "#shape"] = np.array(arr.shape)


def main():
    fm = import_reference("numba")
    from fasmg import kernels as RK
    from fasmg import stencil as RS
    K = {name: getattr(RK, name) for name in RK._KERNEL_NAMES}
    out = {}
    meta = []
    mk = manufactured_ref(fm)
    for c in C.all_cases():
        key = C.case_key(c)
        meta.append(dict(key=key, **{k: v for k, v in c.items()}))
        kind = c["kind"]
        if kind == "kernel":
            arrays, sc = C.kernel_inputs(c)
            C.run_kernel(K, c, arrays, sc)
            for nm, a in arrays.items():
                store(out, f"{key}/{nm}", a)
        elif kind == "fill":
            n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
            data = C.rand_field(c["seed"], n, loc, halo)
            F = fm.Field(fm.unit_grid(n), ref_loc(fm, loc), halo, data)
            fm.fill_ghosts(F, ref_bc(fm, c["dim"], c["bc"]))
            store(out, f"{key}/data", F.data)
        elif kind == "smooth":
            n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
            g = fm.unit_grid(n)
            p = fm.Field(g, ref_loc(fm, loc), halo,
                         C.rand_field(c["seed"], n, loc, halo))
            f = fm.Field(g, ref_loc(fm, loc), halo,
                         C.rand_field(c["seed"] + 1, n, loc, halo))
            plan = fm.make_plan(c["plan"][0], c["dim"], c["plan"][1])
            fm.smooth(f, p, fm.OperatorCoeffs(c["a"], c["b"]), plan,
                      ref_bc(fm, c["dim"], c["bc"]))
            store(out, f"{key}/p", p.data)
        elif kind == "weno":
            n = tuple(c["n"])
            g = fm.unit_grid(n)
            locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
            vel = []
            for t, loc in enumerate(locs):
                F = fm.Field(g, ref_loc(fm, loc), 2,
                             C.rand_field(c["seed"] + 10 * t, n, loc, 2))
                F.ghosts_fresh = True
                vel.append(F)
            res = fm.weno3_convect(tuple(vel), c["target"])
            store(out, f"{key}/conv", res.interior)
        elif kind == "stag":
            n = tuple(c["n"])
            g = fm.unit_grid(n)
            p = fm.Field(g, fm.Location.CELL, 1,
                         C.rand_field(c["seed"], n, "cell", 1))
            for ax in range(c["dim"]):
                store(out, f"{key}/grad{ax}", RS.gradient_axis(p, ax))
            locs = ("edge_ew", "edge_ns", "edge_tb")[: c["dim"]]
            comps = [fm.Field(g, ref_loc(fm, loc), 2,
                              C.rand_field(c["seed"] + 1 + t, n, loc, 2))
                     for t, loc in enumerate(locs)]
            div = fm.divergence_edges_to_cc(*comps)
            store(out, f"{key}/div", div.interior)
            out[f"{key}/intdiv"] = np.array(fm.integral_divergence(*comps))
        elif kind == "reduce":
            a = np.random.default_rng(c["seed"]).standard_normal(c["shape"])
            v = a[tuple(slice(1, s - 1) for s in c["shape"])]
            out[f"{key}/sum"] = np.array(np.sum(v))
            out[f"{key}/mean"] = np.array(np.mean(v))
            out[f"{key}/sumsq"] = np.array(np.sum(v * v))
        elif kind == "solve":
            n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
            p0, f0 = C.solve_inputs(c, mk)
            if "domain" in c:
                g = fm.GridLevel(0, n, (0.0,) * c["dim"], tuple(c["domain"]))
            else:
                g = fm.unit_grid(n)
            L = ref_loc(fm, loc)
            p = fm.Field(g, L, halo, p0.copy())
            f = fm.Field(g, L, halo, f0.copy())
            params = fm.FasParams(c["tol"], c["k_max"], c["s"],
                                  c["mesh_level"])
            plan = fm.make_plan(c["plan"][0], c["dim"], c["plan"][1])
            _, rep = fm.solve(p, f, fm.OperatorCoeffs(c["a"], c["b"]), params,
                              plan, ref_bc(fm, c["dim"], c["bc"]))
            out[f"{key}/history"] = np.array(rep.residual_history)
            out[f"{key}/iterations"] = np.array(rep.iterations)
            out[f"{key}/p_sha256"] = np.array(digest(p.data))
            out[f"{key}/pint_sha256"] = np.array(digest(p.interior))
            out[f"{key}/f_sha256"] = np.array(digest(f.data))
            if c.get("store_field"):
                out[f"{key}/p_interior"] = p.interior.copy()
            if c["rhs"] in ("discrete", "continuous"):
                out[f"{key}/rhs_sha256"] = np.array(digest(mk(c["rhs"], n)))
                if c["rhs"] == "continuous":
                    ex = mk("exact", n)
                    out[f"{key}/err_max"] = np.array(
                        float(np.max(np.abs(p.interior - ex))))
            # one bare V-cycle from the same inputs (PKG/fas.py:93-94)
            p1 = fm.Field(g, L, halo, p0.copy())
            f1 = fm.Field(g, L, halo, f0.copy())
            hier = fm.make_hierarchy(g, c["mesh_level"])
            S = fm.FasSolver(hier, L, ref_bc(fm, c["dim"], c["bc"]), plan,
                             fm.OperatorCoeffs(c["a"], c["b"]))
            S.vcycle(p1, f1, c["s"])
            out[f"{key}/vcycle_p_sha256"] = np.array(digest(p1.data))
            out[f"{key}/vcycle_pint_sha256"] = np.array(digest(p1.interior))
        print(key, flush=True)
    out["__meta__"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
