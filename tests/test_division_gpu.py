"""The sweep kernels divide by the level's denom through a host-computed
reciprocal (dvr in csrc/fasmg_common.cuh: one fma-Newton step, then
Markstein's correction).  IEEE division is what the reference computes
(KER/numpy_backend.py:44,62: ``(h2*f + b*nsum) / denom``), so dvr must be
bitwise __ddiv_rn: checked on 2^25 random normal numerators per divisor for
the denominators of every level of the bench and NS configurations, and for
random divisors."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def denoms():
    out = []
    for n0 in (8192, 1024, 512, 256, 16):
        for k in range(12):
            n = n0 >> k
            if n < 2:
                break
            h = 1.0 / n
            for a, b, d in ((1.0, 1.0, 3), (1.0, 1.0, 2), (1.0, 1e-3 / 100, 3),
                            (1.0, 1e-3 / 200, 3), (0.0, 1e-3, 3), (1.0, 0.5, 3), (0.0, 1.0, 2)):
                out.append(a * (h * h) + (2 * d) * b)
    rng = np.random.default_rng(5)
    out += list(np.ldexp(1.0 + rng.random(64), rng.integers(-40, 40, 64)))
    out += [1.0, 2.0, 3.0, 6.0, 1.0 - 2.0 ** -52, 1.0 + 2.0 ** -52, 2.0 - 2.0 ** -52]
    return np.array(out, dtype=np.float64)


def test_reciprocal_division_is_ieee():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_11152_b200 import _native as N
    d = denoms()
    bad = ctypes.c_long(0)
    N.call("fasmg_selftest_div", 1 << 25, 12345, d.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
           len(d), 60, ctypes.byref(bad))
    assert bad.value == 0, f"{bad.value} quotients differ from IEEE division"
