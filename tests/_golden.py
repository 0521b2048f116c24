"""Helpers to read tests/golden/golden.npz (generated from the reference by
tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

import cases as C

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
PATH_R2 = os.path.join(os.path.dirname(PATH), "golden_r2.npz")  # make_golden_r2.py
_G = None


def golden():
    global _G
    if _G is None:
        _G = dict(np.load(PATH, allow_pickle=False))
        _G.update(np.load(PATH_R2, allow_pickle=False))
    return _G


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def expect_array(key, arr):
    """Bitwise comparison of ``arr`` against the stored golden array (full
    array or sha256 digest)."""
    G = golden()
    arr = np.asarray(arr)
    if key in G:
        ref = G[key]
        assert ref.shape == arr.shape, (key, ref.shape, arr.shape)
        if not np.array_equal(ref.view(np.uint64), np.ascontiguousarray(arr).view(np.uint64)):
            bad = np.argwhere(ref.view(np.uint64) != np.ascontiguousarray(arr).view(np.uint64))
            raise AssertionError(f"{key}: {len(bad)} elements differ, first at {bad[:3].tolist()}; "
                                 f"max |diff| {np.max(np.abs(ref - arr))}")
    else:
        d = str(G[key + "#sha256"])
        assert tuple(G[key + "#shape"]) == arr.shape, key
        assert digest(arr) == d, f"{key}: digest mismatch"


def cases(kind=None):
    out = [c for c in C.all_cases() if kind is None or c["kind"] == kind]
    for c in out:
        c["key"] = C.case_key(c)
    return out
