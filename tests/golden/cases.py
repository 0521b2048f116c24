"""Golden-vector case registry shared by the generator and the tests.

Each case is a plain dict (JSON-able) plus a deterministic input builder
that needs only numpy, so the tests can rebuild inputs without importing the
reference.  ``make_golden.py`` runs the *reference* package on the same
inputs and stores the outputs in ``golden.npz``.
"""

from __future__ import annotations

import itertools

import numpy as np

EDGE_AXIS = {"cell": -1, "edge_ew": 0, "edge_ns": 1, "edge_tb": 2}
FACE_NAMES = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")


def full_shape(n, loc, halo):
    ea = EDGE_AXIS[loc]
    return tuple((m + 1 + 2 * (halo - 1)) if a == ea else (m + 2 * halo)
                 for a, m in enumerate(n))


def interior_extent(n, loc):
    ea = EDGE_AXIS[loc]
    return tuple(m - 1 if a == ea else m for a, m in enumerate(n))


def rand_field(seed, n, loc, halo):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(full_shape(n, loc, halo))


def bc_faces(dim, spec):
    """spec: 'dirichlet' | 'neumann' | 'periodic' | 'lid' | 'mixed' |
    'dirichlet_val' -> dict face -> (kind, value)."""
    names = FACE_NAMES[: 2 * dim]
    if spec in ("dirichlet", "neumann", "periodic"):
        return {nm: (spec, 0.0) for nm in names}
    if spec == "dirichlet_val":
        return {nm: ("dirichlet", 0.25 + 0.5 * t) for t, nm in enumerate(names)}
    if spec == "lid":
        f = {nm: ("dirichlet", 0.0) for nm in names}
        f[names[-1]] = ("dirichlet", 1.0)
        return f
    if spec == "mixed":
        # x periodic, y dirichlet(0.5)/neumann, z neumann/dirichlet(-1)
        f = {"xlo": ("periodic", 0.0), "xhi": ("periodic", 0.0),
             "ylo": ("dirichlet", 0.5), "yhi": ("neumann", 0.0)}
        if dim == 3:
            f["zlo"] = ("neumann", 0.0)
            f["zhi"] = ("dirichlet", -1.0)
        return f
    raise ValueError(spec)


LOCS = {2: ("cell", "edge_ew", "edge_ns"), 3: ("cell", "edge_ew", "edge_ns", "edge_tb")}
BCS = ("dirichlet", "dirichlet_val", "neumann", "periodic", "lid", "mixed")


def fill_cases():
    out = []
    seed = 100
    for dim, n in ((2, (6, 6)), (3, (6, 6, 6))):
        for loc in LOCS[dim]:
            for halo in (1, 2):
                for bc in BCS:
                    seed += 1
                    out.append(dict(kind="fill", dim=dim, n=n, loc=loc,
                                    halo=halo, bc=bc, seed=seed))
    return out


def smooth_cases():
    out = []
    seed = 1000
    for dim, n in ((2, (8, 8)), (3, (8, 8, 8))):
        for loc in LOCS[dim]:
            for bc in BCS:
                seed += 1
                out.append(dict(kind="smooth", dim=dim, n=n, loc=loc, halo=1,
                                bc=bc, plan=("x", "ff"), a=1.0, b=0.7,
                                seed=seed))
        for plan in (("rbgs", "ff"), ("x", "fb"), ("x", "single")) + (
                (("u", "ff"), ("z", "fb")) if dim == 2 else ()):
            seed += 1
            out.append(dict(kind="smooth", dim=dim, n=n, loc="cell", halo=1,
                            bc="dirichlet", plan=plan, a=1.0, b=1.0, seed=seed))
        seed += 1
        out.append(dict(kind="smooth", dim=dim, n=n, loc="cell", halo=2,
                        bc="mixed", plan=("x", "ff"), a=0.0, b=0.3, seed=seed))
    return out


def solve_cases():
    """FAS solves; 'init' = 'random01' (default_rng(seed).random interior) or
    'zero'; 'rhs' = 'random' | 'discrete' (L_h of the manufactured exact
    solution, PKG/manufactured.py:76-84) | 'continuous'."""
    out = []
    # C1 of BASELINE.json: 2D 256^2 heat (a=b=1), Dirichlet 0, X ff, s=2
    out.append(dict(kind="solve", name="C1_2d_256", dim=2, n=(256, 256),
                    loc="cell", halo=1, bc="dirichlet", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-9, k_max=100, s=2, mesh_level=7,
                    init="random01", rhs="discrete", seed=0, store_field=True))
    out.append(dict(kind="solve", name="heat_3d_16", dim=3, n=(16, 16, 16),
                    loc="cell", halo=1, bc="dirichlet", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-9, k_max=20, s=2, mesh_level=3,
                    init="random01", rhs="discrete", seed=0, store_field=True))
    out.append(dict(kind="solve", name="heat_3d_32", dim=3, n=(32, 32, 32),
                    loc="cell", halo=1, bc="dirichlet", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-9, k_max=20, s=2, mesh_level=4,
                    init="random01", rhs="discrete", seed=0, store_field=False))
    out.append(dict(kind="solve", name="asym_3d_32", dim=3, n=(32, 32, 32),
                    loc="cell", halo=1, bc="dirichlet", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-9, k_max=20, s=2, mesh_level=4,
                    init="zero", rhs="continuous", seed=0, store_field=False))
    # singular all-Neumann pressure solves (a=0): mean projection path
    out.append(dict(kind="solve", name="pressure_2d_64", dim=2, n=(64, 64),
                    loc="cell", halo=1, bc="neumann", plan=("x", "ff"),
                    a=0.0, b=1e-3, tol=1e-10, k_max=20, s=2, mesh_level=5,
                    init="zero", rhs="random", seed=7, store_field=True))
    out.append(dict(kind="solve", name="pressure_3d_16", dim=3,
                    n=(16, 16, 16), loc="cell", halo=1, bc="neumann",
                    plan=("x", "ff"), a=0.0, b=1e-3, tol=1e-10, k_max=20, s=2,
                    mesh_level=3, init="zero", rhs="random", seed=8,
                    store_field=True))
    # edge-centered momentum-type solves (a=1, b=dt/Re) with a moving lid
    for loc in ("edge_ew", "edge_ns"):
        out.append(dict(kind="solve", name=f"mom_2d_32_{loc}", dim=2,
                        n=(32, 32), loc=loc, halo=2, bc="lid", plan=("x", "ff"),
                        a=1.0, b=0.05, tol=1e-10, k_max=20, s=2, mesh_level=4,
                        init="random01", rhs="random", seed=11,
                        store_field=True))
    for loc in ("edge_ew", "edge_ns", "edge_tb"):
        out.append(dict(kind="solve", name=f"mom_3d_16_{loc}", dim=3,
                        n=(16, 16, 16), loc=loc, halo=2, bc="lid",
                        plan=("x", "ff"), a=1.0, b=0.05, tol=1e-10, k_max=20,
                        s=2, mesh_level=3, init="random01", rhs="random",
                        seed=12, store_field=True))
    # periodic / mixed BCs, halo 2 caller fields
    out.append(dict(kind="solve", name="mixed_3d_16", dim=3, n=(16, 16, 16),
                    loc="cell", halo=2, bc="mixed", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-10, k_max=20, s=2, mesh_level=3,
                    init="random01", rhs="random", seed=13, store_field=True))
    out.append(dict(kind="solve", name="periodic_2d_32_ew", dim=2, n=(32, 32),
                    loc="edge_ew", halo=1, bc="periodic", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-10, k_max=20, s=2, mesh_level=4,
                    init="random01", rhs="random", seed=14, store_field=True))
    # rectangular grid, shallow hierarchy
    out.append(dict(kind="solve", name="rect_3d", dim=3, n=(8, 16, 32),
                    domain=(1.0, 2.0, 4.0),
                    loc="cell", halo=1, bc="dirichlet_val", plan=("x", "ff"),
                    a=1.0, b=1.0, tol=1e-10, k_max=15, s=2, mesh_level=2,
                    init="random01", rhs="random", seed=15, store_field=True))
    # ordering variants (the ordering study, PKG/smoothers.py:96-109)
    for shape, seq in (("u", "ff"), ("z", "fb"), ("rbgs", "ff")):
        out.append(dict(kind="solve", name=f"order_{shape}{seq}", dim=2,
                        n=(64, 64), loc="cell", halo=1, bc="dirichlet",
                        plan=(shape, seq), a=1.0, b=1.0, tol=1e-9, k_max=60,
                        s=2, mesh_level=5, init="random01", rhs="discrete",
                        seed=0, store_field=False))
    return out


def kernel_cases():
    out = []
    seed = 5000
    for dim in (2, 3):
        for name in ("gs_sweep", "apply_op", "residual", "restrict_cc",
                     "prolong_cc", "restrict_edge0", "prolong_edge0",
                     "weno_deriv0"):
            for rep in range(2):
                seed += 1
                out.append(dict(kind="kernel", name=f"{name}_{dim}d", dim=dim,
                                seed=seed, rep=rep))
    return out


def weno_cases():
    out = []
    seed = 7000
    for dim, n in ((2, (12, 12)), (3, (8, 8, 8))):
        for target in range(dim):
            seed += 1
            out.append(dict(kind="weno", dim=dim, n=n, target=target,
                            seed=seed))
    return out


def stag_cases():
    out = []
    seed = 8000
    for dim, n in ((2, (12, 12)), (3, (8, 8, 8))):
        seed += 1
        out.append(dict(kind="stag", dim=dim, n=n, seed=seed))
    return out


def reduce_cases():
    out = []
    seed = 9000
    for shp in ((10, 10), (258, 258), (34, 33, 34), (34, 34, 33), (66, 66, 66),
                (20, 36, 50), (130, 130, 130), (1026, 1026)):
        seed += 1
        out.append(dict(kind="reduce", shape=shp, seed=seed))
    return out


def all_cases():
    return (kernel_cases() + fill_cases() + smooth_cases() + weno_cases()
            + stag_cases() + reduce_cases() + solve_cases())


def case_key(c):
    if c["kind"] == "solve":
        return f"solve/{c['name']}"
    parts = [c["kind"]] + [f"{k}={c[k]}" for k in sorted(c) if k != "kind"]
    return "/".join(str(p) for p in parts).replace(" ", "")


# ---------------------------------------------------------------------------
# deterministic kernel-case inputs
# ---------------------------------------------------------------------------

def kernel_inputs(c):
    """Arrays and scalar args for one kernel case (reference ABI order).
    Arrays are core-view-shaped (index = grid index) fresh C arrays."""
    rng = np.random.default_rng(c["seed"])
    dim, name = c["dim"], c["name"]
    base = name.rsplit("_", 1)[0]
    if dim == 2:
        m = (6 + 2 * c["rep"], 8)
    else:
        m = (4 + 2 * c["rep"], 6, 8)
    arrays = {}
    if base in ("gs_sweep", "apply_op", "residual"):
        shp = tuple(x + 2 for x in m)
        arrays["p"] = rng.standard_normal(shp)
        arrays["f"] = rng.standard_normal(shp)
        arrays["out"] = rng.standard_normal(shp)
        # inclusive interior bounds, possibly a sub-box
        lo = [1 + c["rep"] for _ in m]
        hi = [x - c["rep"] for x in m]
        pars = [int(v) for v in rng.integers(0, 2, size=dim)]
        scal = dict(a=float(rng.uniform(0, 2)), b=float(rng.uniform(0.1, 2)),
                    h=float(1.0 / m[0]))
        return arrays, dict(lo=lo, hi=hi, pars=pars, **scal)
    if base in ("restrict_cc", "prolong_cc"):
        mc = tuple(x // 2 for x in m)
        arrays["fine"] = rng.standard_normal(tuple(x + 2 for x in m))
        arrays["coarse"] = rng.standard_normal(tuple(x + 2 for x in mc))
        return arrays, dict(mc=mc)
    if base in ("restrict_edge0", "prolong_edge0"):
        # edge axis 0: core extents fine (M+1, N+2[, L+2]); coarse likewise
        mc = tuple(x // 2 for x in m)
        fshape = (m[0] + 1,) + tuple(x + 2 for x in m[1:])
        cshape = (mc[0] + 1,) + tuple(x + 2 for x in mc[1:])
        arrays["fine"] = rng.standard_normal(fshape)
        arrays["coarse"] = rng.standard_normal(cshape)
        return arrays, dict(mc=mc)
    if base == "weno_deriv0":
        ni = m
        arrays["out"] = rng.standard_normal(ni)
        arrays["q"] = rng.standard_normal(tuple(x + 4 for x in ni))
        w = rng.standard_normal(ni)
        w.flat[::5] = 0.0  # exercise the wind >= 0 branch at exactly zero
        arrays["wind"] = w
        return arrays, dict(h=1.0 / m[0], eps=1e-6)
    raise ValueError(name)


def run_kernel(K, c, arrays, sc):
    """Run one kernel case through a kernel module ``K`` exposing the
    reference kernel ABI (the reference's ``fasmg.kernels``, the oracle or
    the product).  Mutates ``arrays`` in place."""
    dim, name = c["dim"], c["name"]
    base = name.rsplit("_", 1)[0]
    if base == "gs_sweep":
        h2 = sc["h"] * sc["h"]
        denom = sc["a"] * h2 + (2 * dim) * sc["b"]
        bounds = list(itertools.chain(*zip(sc["lo"], sc["hi"])))
        K[name](arrays["p"], arrays["f"], sc["b"], h2, denom, *bounds,
                *sc["pars"])
    elif base == "apply_op":
        inv_h2 = 1.0 / (sc["h"] * sc["h"])
        bounds = list(itertools.chain(*zip(sc["lo"], sc["hi"])))
        K[name](arrays["out"], arrays["p"], sc["a"], sc["b"], inv_h2, *bounds)
    elif base == "residual":
        inv_h2 = 1.0 / (sc["h"] * sc["h"])
        bounds = list(itertools.chain(*zip(sc["lo"], sc["hi"])))
        K[name](arrays["out"], arrays["p"], arrays["f"], sc["a"], sc["b"],
                inv_h2, *bounds)
    elif base in ("restrict_cc", "restrict_edge0"):
        K[name](arrays["fine"], arrays["coarse"], *sc["mc"])
    elif base in ("prolong_cc", "prolong_edge0"):
        K[name](arrays["coarse"], arrays["fine"], *sc["mc"])
    elif base == "weno_deriv0":
        inv_2h = 0.5 / sc["h"]
        if dim == 2:
            K[name](arrays["out"], arrays["q"], arrays["wind"], 2, 2, inv_2h,
                    sc["eps"])
        else:
            K[name](arrays["out"], arrays["q"], arrays["wind"], 2, 2, 2,
                    inv_2h, sc["eps"])
    else:
        raise ValueError(name)


def solve_inputs(c, manufactured=None):
    """(p0_data, f_data) for a solve case.  ``manufactured`` supplies the
    discrete/continuous manufactured RHS interiors when needed (a callable
    ``(kind, n) -> interior array``)."""
    n, loc, halo = tuple(c["n"]), c["loc"], c["halo"]
    shp = full_shape(n, loc, halo)
    ext = interior_extent(n, loc)
    g = halo
    isl = tuple(slice(g, g + e) for e in ext)
    p = np.zeros(shp)
    f = np.zeros(shp)
    if c["init"] == "random01":
        p[isl] = np.random.default_rng(c["seed"]).random(ext)
    if c["rhs"] == "random":
        f[isl] = np.random.default_rng(c["seed"] + 1).standard_normal(ext)
    else:
        f[isl] = manufactured(c["rhs"], n)
    return p, f


# ---- round-2 golden set (make_golden_r2.py -> golden_r2.npz) ----
NS_CASES = [
    dict(n=(16, 16), order=1, re=100.0, dt=1e-2, steps=3),
    dict(n=(16, 16), order=2, re=100.0, dt=1e-2, steps=3),
    dict(n=(8, 8, 8), order=1, re=100.0, dt=1e-2, steps=3),
    dict(n=(8, 8, 8), order=2, re=100.0, dt=1e-2, steps=3),
    dict(n=(16, 16, 16), order=2, re=100.0, dt=1e-3, steps=2),
]

DENSE_CASES = [
    dict(n=(4, 4), loc="cell", bc=bc, a=1.0, b=0.5) for bc in BCS
] + [
    dict(n=(4, 4), loc="edge_ew", bc="lid", a=1.0, b=0.25),
    dict(n=(4, 4), loc="edge_ns", bc="mixed", a=1.0, b=0.25),
    dict(n=(4, 4, 4), loc="cell", bc="neumann", a=0.0, b=1.0),
    dict(n=(4, 4, 4), loc="edge_tb", bc="lid", a=1.0, b=0.1),
    dict(n=(4, 4, 4), loc="edge_ew", bc="periodic", a=1.0, b=0.1),
]


def ns_key(c):
    return "ns/{}_o{}_dt{:g}".format("x".join(map(str, c["n"])), c["order"], c["dt"])


def dense_key(c):
    return "dense/{}_{}_{}_a{:g}_b{:g}".format("x".join(map(str, c["n"])), c["loc"], c["bc"],
                                               c["a"], c["b"])
