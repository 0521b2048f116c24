"""CPU oracle for the FAS multigrid hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 product path.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import it; the product package never does.

It restates the reference package ``fasmg`` (``/root/reference/pkg/src/
fasmg``; cited below as ``PKG/`` and ``KER/`` = ``PKG/kernels/``) in two
layers:

* ``fasmg_oracle.c`` (built into ``oracle/build/libfasmg_oracle.so`` by
  ``oracle/Makefile``): the 16 kernels, ghost fill, smoother, V-cycle and
  outer solve loop, and numpy-ordered reductions, in the reference's exact
  association order;
* this file: numpy-side restatements of the elementwise glue the reference
  writes in numpy (staggered gradient/divergence, WENO wind averaging) and
  thin ctypes wrappers.

Pinned against golden vectors generated from the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libfasmg_oracle.so")
_lib = None

KIND_CODES = {"dirichlet": 0, "neumann": 1, "periodic": 2}
EDGE_AXIS = {"cell": -1, "edge_ew": 0, "edge_ns": 1, "edge_tb": 2}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)


def build(force: bool = False) -> str:
    """Compile the C oracle (``make -C oracle``)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH)
        < os.path.getmtime(os.path.join(_HERE, "fasmg_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE, "CC=gcc"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.or_pairwise_sum.restype = ctypes.c_double
        _lib.or_view_sum.restype = ctypes.c_double
        _lib.or_sumsq.restype = ctypes.c_double
        _lib.or_interior_mean.restype = ctypes.c_double
        _lib.or_norm_l2_scaled.restype = ctypes.c_double
        _lib.or_reduce_chunk.restype = ctypes.c_long
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64
    return ctypes.cast(a.ctypes.data, _dp)


def _st(a: np.ndarray):
    return [ctypes.c_long(s // 8) for s in a.strides]


def _d(x):
    return ctypes.c_double(float(x))


# ---------------------------------------------------------------------------
# Kernel ABI (KER/__init__.py:37-46): numpy views of any stride, in place.
# ---------------------------------------------------------------------------

def gs_sweep_2d(p, f, b, h2, denom, ilo, ihi, jlo, jhi, ipar, jpar):
    lib().or_gs_sweep_2d(_ptr(p), *_st(p), _ptr(f), *_st(f), _d(b), _d(h2),
                         _d(denom), ilo, ihi, jlo, jhi, ipar, jpar)


def gs_sweep_3d(p, f, b, h2, denom, ilo, ihi, jlo, jhi, klo, khi, ipar, jpar,
                kpar):
    lib().or_gs_sweep_3d(_ptr(p), *_st(p), _ptr(f), *_st(f), _d(b), _d(h2),
                         _d(denom), ilo, ihi, jlo, jhi, klo, khi, ipar, jpar,
                         kpar)


def apply_op_2d(out, p, a, b, inv_h2, ilo, ihi, jlo, jhi):
    lib().or_apply_op_2d(_ptr(out), *_st(out), _ptr(p), *_st(p), _d(a), _d(b),
                         _d(inv_h2), ilo, ihi, jlo, jhi)


def apply_op_3d(out, p, a, b, inv_h2, ilo, ihi, jlo, jhi, klo, khi):
    lib().or_apply_op_3d(_ptr(out), *_st(out), _ptr(p), *_st(p), _d(a), _d(b),
                         _d(inv_h2), ilo, ihi, jlo, jhi, klo, khi)


def residual_2d(out, p, fsrc, a, b, inv_h2, ilo, ihi, jlo, jhi):
    lib().or_residual_2d(_ptr(out), *_st(out), _ptr(p), *_st(p), _ptr(fsrc),
                         *_st(fsrc), _d(a), _d(b), _d(inv_h2), ilo, ihi, jlo,
                         jhi)


def residual_3d(out, p, fsrc, a, b, inv_h2, ilo, ihi, jlo, jhi, klo, khi):
    lib().or_residual_3d(_ptr(out), *_st(out), _ptr(p), *_st(p), _ptr(fsrc),
                         *_st(fsrc), _d(a), _d(b), _d(inv_h2), ilo, ihi, jlo,
                         jhi, klo, khi)


def restrict_cc_2d(fine, coarse, m0, n0):
    lib().or_restrict_cc_2d(_ptr(fine), *_st(fine), _ptr(coarse), *_st(coarse),
                            m0, n0)


def restrict_cc_3d(fine, coarse, m0, n0, l0):
    lib().or_restrict_cc_3d(_ptr(fine), *_st(fine), _ptr(coarse), *_st(coarse),
                            m0, n0, l0)


def prolong_cc_2d(coarse, fine, m0, n0):
    lib().or_prolong_cc_2d(_ptr(coarse), *_st(coarse), _ptr(fine), *_st(fine),
                           m0, n0)


def prolong_cc_3d(coarse, fine, m0, n0, l0):
    lib().or_prolong_cc_3d(_ptr(coarse), *_st(coarse), _ptr(fine), *_st(fine),
                           m0, n0, l0)


def restrict_edge0_2d(fine, coarse, m0, n0):
    lib().or_restrict_edge0_2d(_ptr(fine), *_st(fine), _ptr(coarse),
                               *_st(coarse), m0, n0)


def restrict_edge0_3d(fine, coarse, m0, n0, l0):
    lib().or_restrict_edge0_3d(_ptr(fine), *_st(fine), _ptr(coarse),
                               *_st(coarse), m0, n0, l0)


def prolong_edge0_2d(coarse, fine, m0, n0):
    lib().or_prolong_edge0_2d(_ptr(coarse), *_st(coarse), _ptr(fine),
                              *_st(fine), m0, n0)


def prolong_edge0_3d(coarse, fine, m0, n0, l0):
    lib().or_prolong_edge0_3d(_ptr(coarse), *_st(coarse), _ptr(fine),
                              *_st(fine), m0, n0, l0)


def weno_deriv0_2d(out, q, wind, oi, oj, inv_2h, eps):
    ni, nj = out.shape
    lib().or_weno_deriv0_2d(_ptr(out), *_st(out), _ptr(q), *_st(q),
                            _ptr(wind), *_st(wind), ni, nj, oi, oj,
                            _d(inv_2h), _d(eps))


def weno_deriv0_3d(out, q, wind, oi, oj, ok, inv_2h, eps):
    ni, nj, nk = out.shape
    lib().or_weno_deriv0_3d(_ptr(out), *_st(out), _ptr(q), *_st(q),
                            _ptr(wind), *_st(wind), ni, nj, nk, oi, oj, ok,
                            _d(inv_2h), _d(eps))


KERNELS = {
    name: globals()[name] for name in (
        "gs_sweep_2d", "gs_sweep_3d", "apply_op_2d", "apply_op_3d",
        "residual_2d", "residual_3d", "restrict_cc_2d", "restrict_cc_3d",
        "prolong_cc_2d", "prolong_cc_3d", "restrict_edge0_2d",
        "restrict_edge0_3d", "prolong_edge0_2d", "prolong_edge0_3d",
        "weno_deriv0_2d", "weno_deriv0_3d",
    )
}


# ---------------------------------------------------------------------------
# Fields (PKG/grid.py:145-232), BCs (PKG/boundary.py), plans
# (PKG/smoothers.py:41-110)
# ---------------------------------------------------------------------------

def full_shape(n, loc, halo):
    """PKG/grid.py:178-184"""
    ea = EDGE_AXIS[loc]
    return tuple((m + 1 + 2 * (halo - 1)) if a == ea else (m + 2 * halo)
                 for a, m in enumerate(n))


def interior_extent(n, loc):
    ea = EDGE_AXIS[loc]
    return tuple(m - 1 if a == ea else m for a, m in enumerate(n))


class OField:
    """numpy field in the reference layout (PKG/grid.py:145-232)."""

    def __init__(self, n, loc="cell", halo=1, data=None):
        self.n = tuple(int(x) for x in n)
        self.loc = loc
        self.halo = halo
        shp = full_shape(self.n, loc, halo)
        self.data = np.zeros(shp) if data is None else data
        assert self.data.shape == shp and self.data.flags.c_contiguous

    @property
    def dim(self):
        return len(self.n)

    @property
    def ea(self):
        return EDGE_AXIS[self.loc]

    @property
    def core(self):
        g = self.halo
        return self.data[tuple(
            slice(g - 1, g - 1 + m + (1 if a == self.ea else 2))
            for a, m in enumerate(self.n))]

    @property
    def interior(self):
        g = self.halo
        ext = interior_extent(self.n, self.loc)
        return self.data[tuple(slice(g, g + e) for e in ext)]

    def copy(self):
        return OField(self.n, self.loc, self.halo, self.data.copy())


def bc_codes(faces):
    """``faces``: dict face-name -> (kind, value) for xlo..zhi."""
    kinds = np.zeros(6, dtype=np.int32)
    vals = np.zeros(6)
    for t, name in enumerate(("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")):
        if name in faces:
            k, v = faces[name]
            kinds[t] = KIND_CODES[k]
            vals[t] = v
    return kinds, vals


def uniform_bc(dim, kind, value=0.0):
    names = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")[: 2 * dim]
    return {nm: (kind, value) for nm in names}


_X_2D = ((1, 0), (0, 1), (0, 0), (1, 1))
_U_2D = ((1, 1), (0, 1), (0, 0), (1, 0))
_Z_2D = ((1, 1), (0, 1), (1, 0), (0, 0))
_X_3D = ((1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1),
         (1, 0, 1), (0, 1, 1), (0, 0, 0), (1, 1, 0))


def plan_colors(shape, dim, sequence="ff"):
    """Color list of make_plan (PKG/smoothers.py:87-110): each color is a
    tuple of parity sub-tuples swept after one ghost refresh."""
    base_x = _X_2D if dim == 2 else _X_3D
    if shape == "rbgs":
        base = [tuple(t for t in base_x if sum(t) % 2 == 1),
                tuple(t for t in base_x if sum(t) % 2 == 0)]
    elif shape == "x":
        base = [(t,) for t in base_x]
    elif shape in ("u", "z"):
        assert dim == 2
        base = [(t,) for t in (_U_2D if shape == "u" else _Z_2D)]
    else:
        raise ValueError(shape)
    if sequence == "ff":
        seq = base + base
    elif sequence == "fb":
        seq = base + base[::-1]
    elif sequence == "single":
        seq = base
    else:
        raise ValueError(sequence)
    return seq


def _plan_arrays(colors):
    nsub = np.array([len(c) for c in colors], dtype=np.int32)
    subs = np.array([list(t) + [0] * (3 - len(t)) for c in colors for t in c],
                    dtype=np.int32).reshape(-1)
    return nsub, subs


def _ip_of(a):
    return ctypes.cast(a.ctypes.data, _ip)


def fill_ghosts(F: OField, faces):
    kinds, vals = bc_codes(faces)
    n = np.array(list(F.n) + [1] * (3 - F.dim), dtype=np.int32)
    lib().or_fill_ghosts(_ptr(F.data), F.dim, _ip_of(n), F.ea, F.halo,
                         _ip_of(kinds), _ptr(vals))
    return F


def smooth(f: OField, p: OField, a, b, colors, faces, h=None):
    kinds, vals = bc_codes(faces)
    n = np.array(list(p.n) + [1] * (3 - p.dim), dtype=np.int32)
    nsub, subs = _plan_arrays(colors)
    h = 1.0 / p.n[0] if h is None else h
    lib().or_smooth(_ptr(p.data), p.halo, _ptr(f.data), f.halo, p.dim,
                    _ip_of(n), p.ea, _d(h), _d(a), _d(b), _ip_of(kinds),
                    _ptr(vals), len(colors), _ip_of(nsub), _ip_of(subs))
    return p


def fas_solve(p: OField, f: OField, a, b, faces, colors, tol, k_max, s,
              mesh_level, dmin=0.0, dmax=1.0, vcycle_only=False):
    """FasSolver(...).solve(p, f, FasParams(tol, k_max, s, mesh_level))
    (PKG/fas.py:137-162); returns (iterations, residual_history).  With
    ``vcycle_only`` runs ``k_max`` bare V-cycles (PKG/fas.py:93-94)."""
    kinds, vals = bc_codes(faces)
    n = np.array(list(p.n) + [1] * (3 - p.dim), dtype=np.int32)
    nsub, subs = _plan_arrays(colors)
    hist = np.zeros(max(k_max, 1))
    it = lib().or_fas_solve(
        _ptr(p.data), p.halo, _ptr(f.data), f.halo, p.dim, _ip_of(n), p.ea,
        _d(dmin), _d(dmax), mesh_level, _d(a), _d(b), _ip_of(kinds),
        _ptr(vals), len(colors), _ip_of(nsub), _ip_of(subs), _d(tol), k_max,
        s, _ptr(hist), 1 if vcycle_only else 0)
    return it, [float(x) for x in hist[:it]] if not vcycle_only else []


# ---------------------------------------------------------------------------
# Reductions (PKG/grid.py:235-254)
# ---------------------------------------------------------------------------

def norm_l2_scaled(F: OField, h=None):
    n = np.array(list(F.n) + [1] * (3 - F.dim), dtype=np.int32)
    h = 1.0 / F.n[0] if h is None else h
    return lib().or_norm_l2_scaled(_ptr(F.data), F.dim, _ip_of(n), F.ea,
                                   F.halo, _d(h))


def interior_mean(F: OField):
    n = np.array(list(F.n) + [1] * (3 - F.dim), dtype=np.int32)
    return lib().or_interior_mean(_ptr(F.data), F.dim, _ip_of(n), F.ea,
                                  F.halo)


def view_sum(v: np.ndarray):
    """np.sum over a (non-contiguous) C-order view."""
    ext = np.array(v.shape, dtype=np.int32)
    st = np.array([s // 8 for s in v.strides], dtype=np.int64)
    return lib().or_view_sum(_ptr(v), v.ndim, _ip_of(ext),
                             ctypes.cast(st.ctypes.data, _lp))


def reduce_chunk(shape):
    ext = np.array(shape, dtype=np.int32)
    return lib().or_reduce_chunk(len(shape), _ip_of(ext))


# ---------------------------------------------------------------------------
# Staggered operators (PKG/stencil.py:93-169) -- numpy restatement
# ---------------------------------------------------------------------------

_EDGE_OF_AXIS = ("edge_ew", "edge_ns", "edge_tb")


def gradient_axis(p: OField, axis: int) -> np.ndarray:
    """PKG/stencil.py:114-125"""
    pc = p.core
    hi = [slice(1, m + 1) for m in p.n]
    lo = [slice(1, m + 1) for m in p.n]
    hi[axis] = slice(2, p.n[axis] + 1)
    lo[axis] = slice(1, p.n[axis])
    return (pc[tuple(hi)] - pc[tuple(lo)]) * (1.0 / (1.0 / p.n[0]))


def divergence_edges_to_cc(comps) -> np.ndarray:
    """PKG/stencil.py:128-156 (returns the interior array)."""
    n = comps[0].n
    inv_h = 1.0 / (1.0 / n[0])
    acc = None
    for axis, c in enumerate(comps):
        cc = c.core
        hi = [slice(1, m + 1) for m in n]
        lo = [slice(1, m + 1) for m in n]
        hi[axis] = slice(1, n[axis] + 1)
        lo[axis] = slice(0, n[axis])
        term = (cc[tuple(hi)] - cc[tuple(lo)]) * inv_h
        acc = term if acc is None else acc + term
    return acc


def avg_to_target(adv: OField, target_axis: int) -> np.ndarray:
    """PKG/weno.py:26-51"""
    adv_axis = adv.ea
    core = adv.core
    dim = adv.dim

    def pick(d_target, d_adv):
        sl = []
        for axis in range(dim):
            n_int = adv.n[axis] - (1 if axis == adv_axis else 0)
            if axis == target_axis:
                lo = 1 + d_target
                sl.append(slice(lo, lo + adv.n[axis] - 1))
            elif axis == adv_axis:
                lo = 0 + d_adv
                sl.append(slice(lo, lo + adv.n[axis]))
            else:
                sl.append(slice(1, 1 + n_int))
        return core[tuple(sl)]

    return 0.25 * ((pick(0, 0) + pick(0, 1)) + (pick(1, 0) + pick(1, 1)))


def weno3_convect(vel, target, eps=1e-6) -> np.ndarray:
    """PKG/weno.py:54-91 (returns the interior array)."""
    q = vel[target]
    dim = q.dim
    conv = np.zeros(interior_extent(q.n, q.loc))
    inv_2h = 0.5 / (1.0 / q.n[0])
    g = q.halo
    for axis in range(dim):
        if axis == target:
            wind = np.ascontiguousarray(q.interior)
        else:
            wind = np.ascontiguousarray(avg_to_target(vel[axis], target))
        conv_v = np.moveaxis(conv, axis, 0)
        q_v = np.moveaxis(q.data, axis, 0)
        wind_v = np.moveaxis(wind, axis, 0)
        if dim == 2:
            weno_deriv0_2d(conv_v, q_v, wind_v, g, g, inv_2h, eps)
        else:
            weno_deriv0_3d(conv_v, q_v, wind_v, g, g, g, inv_2h, eps)
    return conv


# ---------------------------------------------------------------------------
# Manufactured problems (PKG/manufactured.py:47-84) -- numpy restatement
# ---------------------------------------------------------------------------

def _g(s):
    return np.sin(np.pi * np.sin(np.pi * s))


def _g2(s):
    pi = np.pi
    inner = pi * np.sin(pi * s)
    return (-np.sin(inner) * (pi * pi * np.cos(pi * s)) ** 2
            - np.cos(inner) * pi ** 3 * np.sin(pi * s))


def cell_coords(n, axis, dmin=0.0, dmax=1.0):
    """GridLevel.cell_coords (PKG/grid.py:88-91) on a unit-h grid."""
    h = (dmax - dmin) / n[0]
    return dmin + (np.arange(1, n[axis] + 1) - 0.5) * h


def poisson_exact(n) -> np.ndarray:
    axes = [_g(cell_coords(n, a)) for a in range(len(n))]
    if len(n) == 2:
        return axes[0][:, None] * axes[1][None, :]
    return axes[0][:, None, None] * axes[1][None, :, None] * axes[2][None, None, :]


def poisson_rhs_continuous(n) -> np.ndarray:
    g = [_g(cell_coords(n, a)) for a in range(len(n))]
    g2 = [_g2(cell_coords(n, a)) for a in range(len(n))]
    if len(n) == 2:
        p = g[0][:, None] * g[1][None, :]
        lap = g2[0][:, None] * g[1][None, :] + g[0][:, None] * g2[1][None, :]
    else:
        p = g[0][:, None, None] * g[1][None, :, None] * g[2][None, None, :]
        lap = (g2[0][:, None, None] * g[1][None, :, None] * g[2][None, None, :]
               + g[0][:, None, None] * g2[1][None, :, None] * g[2][None, None, :]
               + g[0][:, None, None] * g[1][None, :, None] * g2[2][None, None, :])
    return p - lap


def poisson_rhs_discrete(n, a=1.0, b=1.0) -> np.ndarray:
    F = OField(n, "cell", 1)
    F.interior[...] = poisson_exact(n)
    fill_ghosts(F, uniform_bc(len(n), "dirichlet"))
    out = OField(n, "cell", 1)
    h = 1.0 / n[0]
    inv_h2 = 1.0 / (h * h)
    bounds = [x for m in n for x in (1, m)]
    if len(n) == 2:
        apply_op_2d(out.core, F.core, a, b, inv_h2, *bounds)
    else:
        apply_op_3d(out.core, F.core, a, b, inv_h2, *bounds)
    return out.interior.copy()


def manufactured(kind, n):
    if kind == "discrete":
        return poisson_rhs_discrete(tuple(n))
    if kind == "continuous":
        return poisson_rhs_continuous(tuple(n))
    if kind == "exact":
        return poisson_exact(tuple(n))
    raise ValueError(kind)
