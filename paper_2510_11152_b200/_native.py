"""ctypes binding of libfasmg_b200.so (declared in include/fasmg_b200.h).

The product path has no CPU fallback: importing this module on a machine
without the built library, or calling into it without a CUDA device, raises
:class:`NativeError`.  PyTorch owns device memory and streams; every call
passes raw device pointers, int64 element strides and a cudaStream_t.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfasmg_b200.so")

_c_long_p = ctypes.POINTER(ctypes.c_long)
_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_double_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

_lib = None
_lock = threading.Lock()

# name -> argtypes ("p" device pointer, "s" stride array, "i" int, "d" double,
# "l" long, "S" stream, "I" int array, "D" double array, "U" uint array)
_SIGS = {
    "fasmg_gs_sweep_2d": "psps" + "ddd" + "iiii" + "ii" + "S",
    "fasmg_gs_sweep_3d": "psps" + "ddd" + "iiiiii" + "iii" + "S",
    "fasmg_apply_op_2d": "psps" + "ddd" + "iiii" + "S",
    "fasmg_apply_op_3d": "psps" + "ddd" + "iiiiii" + "S",
    "fasmg_residual_2d": "pspsps" + "ddd" + "iiii" + "S",
    "fasmg_residual_3d": "pspsps" + "ddd" + "iiiiii" + "S",
    "fasmg_restrict_cc_2d": "pspsiiS",
    "fasmg_restrict_cc_3d": "pspsiiiS",
    "fasmg_prolong_cc_2d": "pspsiiS",
    "fasmg_prolong_cc_3d": "pspsiiiS",
    "fasmg_restrict_edge0_2d": "pspsiiS",
    "fasmg_restrict_edge0_3d": "pspsiiiS",
    "fasmg_prolong_edge0_2d": "pspsiiS",
    "fasmg_prolong_edge0_3d": "pspsiiiS",
    "fasmg_weno_deriv0_2d": "pspsps" + "iiii" + "dd" + "S",
    "fasmg_weno_deriv0_3d": "pspsps" + "iiiiii" + "dd" + "S",
    "fasmg_fill_ghosts": "piIiiIDS",
    "fasmg_fill_ghosts_slab": "piIiiIDiiS",
    "fasmg_view_sum": "psiIpppS",
    "fasmg_view_sumsq": "psiIppS",
    "fasmg_sub_mean": "psiIpdS",
    "fasmg_view_chunk_sums": "psiIIppS",
    "fasmg_chunk_total": "plpS",
    "fasmg_ns_rhs": "ipspspspsiiIddddS",
    "fasmg_engine_load": "vpsps",
    "fasmg_engine_store": "vps",
    "fasmg_engine_run": "viiDi",
    "fasmg_engine_residual_sumsq": "vD",
    "fasmg_engine_level_info": "viL",
    "fasmg_engine_time_sweeps": "viiD",
    "fasmg_engine_launch": "vii",
    "fasmg_engine_prepare": "vi",
    "fasmg_engine_solve": "viddDI",
    "fasmg_engine_prepare_solve": "v",
    "fasmg_engine_solve_launch": "vidd",
    "fasmg_engine_solve_wait": "vDI",
    "fasmg_selftest_div": "llDiiL",
    "fasmg_engine_level_geom": "viL",
    "fasmg_engine_level_copy": "viip",
    "fasmg_engine_result": "vD",
    "fasmg_engine_sync_halos": "v",
    "fasmg_engine_slab_info": "vI",
    "fasmg_ipc_close_handle": "v",
    "fasmg_stream_create": "V",
    "fasmg_stream_destroy": "v",
    "fasmg_stream_synchronize": "v",
    "fasmg_stream_wait": "vv",
    "fasmg_device_count": "I",
    "fasmg_gradient_axis": "psp" + "iIi" + "dS",
    "fasmg_weno_convect": "psVLiiiIddS",
}

_CT = {
    "p": _vp, "s": _c_long_p, "i": ctypes.c_int, "d": ctypes.c_double,
    "l": ctypes.c_long, "S": _vp, "I": _c_int_p, "D": _c_double_p,
    "U": ctypes.POINTER(ctypes.c_uint), "v": _vp, "V": ctypes.POINTER(_vp),
    "L": _c_long_p,
}


def lib():
    """Load the native library (raises NativeError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} not found: build it with "
                "paper_2510_11152_b200/csrc/build.sh (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, sig in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = [_CT[c] for c in sig]
            fn.restype = ctypes.c_int
        L.fasmg_last_error.restype = ctypes.c_char_p
        L.fasmg_version.restype = ctypes.c_int
        L.fasmg_view_sum_chunks.argtypes = [ctypes.c_int, _c_int_p]
        L.fasmg_view_sum_chunks.restype = ctypes.c_long
        L.fasmg_view_sumsq_scratch.argtypes = [ctypes.c_int, _c_int_p]
        L.fasmg_view_sumsq_scratch.restype = ctypes.c_long
        L.fasmg_view_chunk_len.argtypes = [ctypes.c_int, _c_int_p]
        L.fasmg_view_chunk_len.restype = ctypes.c_long
        L.fasmg_engine_create.argtypes = [
            ctypes.c_int, _c_int_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            ctypes.c_int, ctypes.c_double, ctypes.c_double, _c_int_p, _c_double_p,
            ctypes.c_int, ctypes.POINTER(ctypes.c_uint), ctypes.c_int, _vp]
        L.fasmg_engine_create.restype = _vp
        L.fasmg_engine_create_slab.argtypes = L.fasmg_engine_create.argtypes + [
            ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.fasmg_engine_create_slab.restype = _vp
        L.fasmg_engine_create_in.argtypes = L.fasmg_engine_create.argtypes + [_vp]
        L.fasmg_engine_create_in.restype = _vp
        L.fasmg_arena_create.argtypes = []
        L.fasmg_arena_create.restype = _vp
        L.fasmg_arena_release.argtypes = [_vp]
        L.fasmg_arena_release.restype = None
        L.fasmg_engine_export_count.argtypes = [_vp]
        L.fasmg_engine_export_count.restype = ctypes.c_int
        L.fasmg_engine_export.argtypes = [_vp, ctypes.POINTER(ctypes.c_ulonglong)]
        L.fasmg_engine_export.restype = ctypes.c_int
        L.fasmg_engine_connect.argtypes = [_vp, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
        L.fasmg_engine_connect.restype = ctypes.c_int
        L.fasmg_ipc_get_handle.argtypes = [_vp, ctypes.c_char_p]
        L.fasmg_ipc_get_handle.restype = ctypes.c_int
        L.fasmg_ipc_open_handle.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
        L.fasmg_ipc_open_handle.restype = ctypes.c_int
        L.fasmg_engine_destroy.argtypes = [_vp]
        L.fasmg_engine_destroy.restype = None
        L.fasmg_engine_kernels_per_vcycle.argtypes = [_vp, ctypes.c_int]
        L.fasmg_engine_kernels_per_vcycle.restype = ctypes.c_long
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().fasmg_last_error().decode(errors="replace")
        raise NativeError(f"libfasmg_b200 error {status}: {msg}")


_ctx = threading.local()  # device of the tensors of the call being assembled


def call(name: str, *args) -> None:
    """Call one C-ABI entry point with the CUDA device of its tensor
    arguments current (a stream or kernel of another device would be
    rejected by the runtime)."""
    dev = getattr(_ctx, "dev", None)
    _ctx.dev = None
    if dev is not None and dev.index != torch.cuda.current_device():
        with torch.cuda.device(dev):
            check(getattr(lib(), name)(*args))
    else:
        check(getattr(lib(), name)(*args))


def require_cuda(t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise NativeError("fasmg_b200 operates on CUDA tensors only (no CPU path)")
    if t.dtype != torch.float64:
        raise NativeError(f"fasmg_b200 needs float64 tensors, got {t.dtype}")


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    """Device pointer of ``t``; also records t's device for the enclosing
    :func:`call` and :func:`torch_stream`."""
    require_cuda(t)
    _ctx.dev = t.device
    return ctypes.c_void_p(t.data_ptr())


def strides(t: torch.Tensor):
    st = list(t.stride()) + [0] * (3 - t.dim())
    return (ctypes.c_long * 3)(*st)


def ints(seq):
    seq = list(seq)
    return (ctypes.c_int * max(len(seq), 1))(*seq)


def doubles(seq):
    seq = list(seq)
    return (ctypes.c_double * max(len(seq), 1))(*seq)


def torch_stream(device=None) -> ctypes.c_void_p:
    """cudaStream_t of torch's current stream on ``device`` (default: the
    device of the tensors passed to :func:`ptr` for the call being
    assembled, else the current device)."""
    if device is None:
        device = getattr(_ctx, "dev", None)
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_streams: dict = {}


def engine_stream(device: int) -> ctypes.c_void_p:
    """A non-blocking library stream per device (graph capture cannot use
    the legacy default stream)."""
    s = _streams.get(device)
    if s is None:
        with torch.cuda.device(device):
            h = ctypes.c_void_p()
            check(lib().fasmg_stream_create(ctypes.byref(h)))
        s = _streams[device] = h
    return s


def wait(waiter, signaler) -> None:
    call("fasmg_stream_wait", waiter, signaler)
