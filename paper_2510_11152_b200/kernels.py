"""The reference kernel ABI on the B200 (drop-in for ``fasmg.kernels``).

Same 16 names and argument order as KER/__init__.py:37-46 /
KER/numpy_backend.py, taking CUDA float64 tensor views of any stride
(``Field.core`` views and ``movedim`` permutations) instead of numpy views.
Each call launches one sm_100a kernel of libfasmg_b200.so on torch's
current stream.  There is no backend switch and no CPU path.
"""

from __future__ import annotations

from . import _native as N

_KERNEL_NAMES = (
    "gs_sweep_2d", "gs_sweep_3d",
    "apply_op_2d", "apply_op_3d",
    "residual_2d", "residual_3d",
    "restrict_cc_2d", "restrict_cc_3d",
    "prolong_cc_2d", "prolong_cc_3d",
    "restrict_edge0_2d", "restrict_edge0_3d",
    "prolong_edge0_2d", "prolong_edge0_3d",
    "weno_deriv0_2d", "weno_deriv0_3d",
)


def _v(t):
    return N.ptr(t), N.strides(t)


def gs_sweep_2d(p, f, b, h2, denom, ilo, ihi, jlo, jhi, ipar, jpar):
    N.call("fasmg_gs_sweep_2d", *_v(p), *_v(f), b, h2, denom, ilo, ihi, jlo, jhi,
           ipar, jpar, N.torch_stream())


def gs_sweep_3d(p, f, b, h2, denom, ilo, ihi, jlo, jhi, klo, khi, ipar, jpar, kpar):
    N.call("fasmg_gs_sweep_3d", *_v(p), *_v(f), b, h2, denom, ilo, ihi, jlo, jhi,
           klo, khi, ipar, jpar, kpar, N.torch_stream())


def apply_op_2d(out, p, a, b, inv_h2, ilo, ihi, jlo, jhi):
    N.call("fasmg_apply_op_2d", *_v(out), *_v(p), a, b, inv_h2, ilo, ihi, jlo, jhi,
           N.torch_stream())


def apply_op_3d(out, p, a, b, inv_h2, ilo, ihi, jlo, jhi, klo, khi):
    N.call("fasmg_apply_op_3d", *_v(out), *_v(p), a, b, inv_h2, ilo, ihi, jlo, jhi,
           klo, khi, N.torch_stream())


def residual_2d(out, p, fsrc, a, b, inv_h2, ilo, ihi, jlo, jhi):
    N.call("fasmg_residual_2d", *_v(out), *_v(p), *_v(fsrc), a, b, inv_h2, ilo, ihi,
           jlo, jhi, N.torch_stream())


def residual_3d(out, p, fsrc, a, b, inv_h2, ilo, ihi, jlo, jhi, klo, khi):
    N.call("fasmg_residual_3d", *_v(out), *_v(p), *_v(fsrc), a, b, inv_h2, ilo, ihi,
           jlo, jhi, klo, khi, N.torch_stream())


def restrict_cc_2d(fine, coarse, m0, n0):
    N.call("fasmg_restrict_cc_2d", *_v(fine), *_v(coarse), m0, n0, N.torch_stream())


def restrict_cc_3d(fine, coarse, m0, n0, l0):
    N.call("fasmg_restrict_cc_3d", *_v(fine), *_v(coarse), m0, n0, l0, N.torch_stream())


def prolong_cc_2d(coarse, fine, m0, n0):
    N.call("fasmg_prolong_cc_2d", *_v(coarse), *_v(fine), m0, n0, N.torch_stream())


def prolong_cc_3d(coarse, fine, m0, n0, l0):
    N.call("fasmg_prolong_cc_3d", *_v(coarse), *_v(fine), m0, n0, l0, N.torch_stream())


def restrict_edge0_2d(fine, coarse, m0, n0):
    N.call("fasmg_restrict_edge0_2d", *_v(fine), *_v(coarse), m0, n0, N.torch_stream())


def restrict_edge0_3d(fine, coarse, m0, n0, l0):
    N.call("fasmg_restrict_edge0_3d", *_v(fine), *_v(coarse), m0, n0, l0,
           N.torch_stream())


def prolong_edge0_2d(coarse, fine, m0, n0):
    N.call("fasmg_prolong_edge0_2d", *_v(coarse), *_v(fine), m0, n0, N.torch_stream())


def prolong_edge0_3d(coarse, fine, m0, n0, l0):
    N.call("fasmg_prolong_edge0_3d", *_v(coarse), *_v(fine), m0, n0, l0,
           N.torch_stream())


def weno_deriv0_2d(out, q, wind, oi, oj, inv_2h, eps):
    ni, nj = out.shape
    N.call("fasmg_weno_deriv0_2d", *_v(out), *_v(q), *_v(wind), ni, nj, oi, oj, inv_2h,
           eps, N.torch_stream())


def weno_deriv0_3d(out, q, wind, oi, oj, ok, inv_2h, eps):
    ni, nj, nk = out.shape
    N.call("fasmg_weno_deriv0_3d", *_v(out), *_v(q), *_v(wind), ni, nj, nk, oi, oj, ok,
           inv_2h, eps, N.torch_stream())


def active_backend() -> str:
    return "b200"


def available_backends():
    return ("b200",)


KERNELS = {name: globals()[name] for name in _KERNEL_NAMES}

__all__ = list(_KERNEL_NAMES) + ["active_backend", "available_backends"]
