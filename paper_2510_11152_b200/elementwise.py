"""Interior elementwise kernels of the projection drivers (fasmg_ns_elem,
fasmg_laplacian in csrc/fasmg_natural.cu).  Each call is one native launch
on torch's current stream; views may have any strides."""

from __future__ import annotations

import ctypes

import torch

from . import _native as N

MIX_EXT, MIX_AVG, AVG4, AXPY, ADD, COPY, RHS1, RHS2, NEG = range(9)


def elem(op: int, out: torch.Tensor, inputs, s0: float = 0.0, s1: float = 0.0) -> torch.Tensor:
    ins = list(inputs) + [None] * (4 - len(inputs))
    for t in ins:
        if t is not None and tuple(t.shape) != tuple(out.shape):
            raise ValueError(f"shape mismatch {tuple(t.shape)} vs {tuple(out.shape)}")
    ptrs = (ctypes.c_void_p * 4)(*[(t.data_ptr() if t is not None else None) for t in ins])
    st = []
    for t in ins:
        s = list(t.stride()) if t is not None else []
        st += s + [0] * (3 - len(s))
    N.require_cuda(out)
    N.call("fasmg_ns_elem", ctypes.c_int(op), N.ptr(out), N.strides(out), ptrs,
           (ctypes.c_long * 12)(*st), ctypes.c_double(s0), ctypes.c_double(s1),
           ctypes.c_int(out.dim()), N.ints(out.shape), N.torch_stream())
    return out


def laplacian(field, out: torch.Tensor | None = None) -> torch.Tensor:
    """(nsum - 2d*c) / h^2 at the interior points of a field with fresh ghosts
    (the _lap helper of KER/numpy_backend.py:66-88)."""
    shape = field.interior_shape
    if out is None:
        out = torch.empty(shape, dtype=torch.float64, device=field.device)
    pc = field.core
    N.call("fasmg_laplacian", N.ptr(out), N.strides(out), N.ptr(pc), N.strides(pc),
           ctypes.c_int(field.grid.dim), N.ints(shape),
           ctypes.c_double(1.0 / (field.grid.h * field.grid.h)), N.torch_stream())
    return out


def momentum_source(order: int, out: torch.Tensor, u, conv: torch.Tensor, p, axis: int,
                    s0: float, s1: float = 0.0) -> torch.Tensor:
    """``out = ((u - s0*conv) - s0*grad_axis(p)) [+ s1*Lap(u)]`` on the
    interior of velocity component ``u`` (Field, fresh ghosts for order 2)
    in one native pass -- bitwise the RHS1/RHS2 elem of gradient_axis and
    laplacian temporaries.  order 0: ``out = u - s0*grad_axis(p)`` (the
    projection correction, bitwise AXPY; ``conv`` unused)."""
    g = u.grid
    N.require_cuda(out)
    uc, pc = u.core, p.core
    N.call("fasmg_ns_rhs", int(order), N.ptr(out), N.strides(out), N.ptr(uc), N.strides(uc),
           N.ptr(conv if conv is not None else out), N.strides(conv if conv is not None else out),
           N.ptr(pc), N.strides(pc), g.dim, int(axis),
           N.ints(u.interior_shape), float(s0), float(s1), 1.0 / g.h, 1.0 / (g.h * g.h),
           N.torch_stream())
    return out
