"""CPU-side checks of the product package: the C-ABI library loads and
exports every symbol include/fasmg_b200.h declares; host logic (plans,
masks, BC codes, hierarchy validation); no CPU fallback."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_11152_b200", "libfasmg_b200.so")
HDR = os.path.join(ROOT, "include", "fasmg_b200.h")


def _ensure_lib():
    if not os.path.exists(LIB):
        subprocess.run(["bash", os.path.join(ROOT, "paper_2510_11152_b200", "csrc", "build.sh")],
                       check=True)


def test_library_exports_header_symbols():
    _ensure_lib()
    names = re.findall(r"^[\w\s\*]*?\b(fasmg_\w+)\s*\(", open(HDR).read(), re.M)
    assert len(names) >= 40
    lib = ctypes.CDLL(LIB)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    _ensure_lib()
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_kernel_abi_names_match_reference():
    from paper_2510_11152_b200 import kernels as K
    assert K._KERNEL_NAMES == (
        "gs_sweep_2d", "gs_sweep_3d", "apply_op_2d", "apply_op_3d", "residual_2d",
        "residual_3d", "restrict_cc_2d", "restrict_cc_3d", "prolong_cc_2d", "prolong_cc_3d",
        "restrict_edge0_2d", "restrict_edge0_3d", "prolong_edge0_2d", "prolong_edge0_3d",
        "weno_deriv0_2d", "weno_deriv0_3d")


def test_class_masks():
    from paper_2510_11152_b200 import make_plan
    assert make_plan("x", 3, "ff").class_masks() == [0x96, 0x69, 0x96, 0x69]
    assert make_plan("x", 2, "ff").class_masks() == [0x6, 0x9, 0x6, 0x9]
    assert make_plan("rbgs", 3, "ff").class_masks() == [0x96, 0x69, 0x96, 0x69]
    # fb: the repeated classes at the turn must not merge with themselves
    assert make_plan("x", 2, "fb").class_masks() == [0x6, 0x9, 0x9, 0x6]
    assert make_plan("u", 2, "ff").class_masks() == [1 << 3, 1 << 1, 1 << 0, 1 << 2] * 2


def test_bc_codes_and_hierarchy():
    import paper_2510_11152_b200 as P
    bc = P.BoundaryCondition.dirichlet(3).with_face("zhi", P.FaceRule("dirichlet", 1.0))
    kinds, vals = bc.codes()
    assert kinds == [0] * 6 and vals[5] == 1.0
    assert P.BoundaryCondition.periodic(2).codes()[0][:4] == [2, 2, 2, 2]
    with pytest.raises(P.NonDivisibleGrid):
        P.make_hierarchy(P.unit_grid((12, 12)), 2)
    assert P.make_hierarchy(P.unit_grid((2048, 2048)), 10).mesh_level == 10
    with pytest.raises(ValueError):
        P.BoundaryCondition(2, (("xlo", P.FaceRule("periodic")), ("xhi", P.FaceRule("dirichlet")),
                                ("ylo", P.FaceRule("dirichlet")), ("yhi", P.FaceRule("dirichlet"))))


def test_no_cpu_fallback():
    import torch
    import paper_2510_11152_b200 as P
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(P.NativeError):
        P.Field(P.unit_grid((8, 8)), P.Location.CELL)
