"""The drop-in surface: every public name of the reference package
(PKG/__init__.py:13-25) is importable from this package under the same
name.  CPU only (importing the package does not load the CUDA library)."""
import ast
import os

import pytest

# PKG/__init__.py's imports, frozen here because /root/reference does not
# exist on the GPU box
REFERENCE_PUBLIC = (
    "BoundaryCondition", "FaceRule", "fill_ghosts",
    "ConfigError", "FasmgError", "IncompatibleRHS", "LocationMismatch", "MissingBinding",
    "NonDivisibleGrid", "PlanDimMismatch", "UnfilledGhosts",
    "FasParams", "FasSolver", "SolveReport", "solve", "vcycle",
    "Field", "GridHierarchy", "GridLevel", "Location", "make_hierarchy", "norm_l2_scaled",
    "unit_grid",
    "ColorSet", "SweepPlan", "gs_update", "make_plan", "smooth",
    "OperatorCoeffs", "apply_operator", "divergence_edges_to_cc", "gradient_cc_to_edges",
    "integral_divergence", "residual",
    "prolong", "prolong_cc", "prolong_edge", "restrict", "restrict_cc", "restrict_edge",
    "weno3_convect",
    "__version__",
)
REF_INIT = "/root/reference/pkg/src/fasmg/__init__.py"


def test_reference_public_names_importable():
    import paper_2510_11152_b200 as P
    missing = [nm for nm in REFERENCE_PUBLIC if not hasattr(P, nm)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(REF_INIT), reason="reference tree not present")
def test_frozen_list_matches_reference():
    tree = ast.parse(open(REF_INIT).read())
    names = {a.asname or a.name for node in tree.body if isinstance(node, ast.ImportFrom)
             for a in node.names}
    names |= {t.id for node in tree.body if isinstance(node, ast.Assign)
              for t in node.targets if isinstance(t, ast.Name)}
    assert names == set(REFERENCE_PUBLIC)


def test_submodules_mirror_reference():
    """The reference's modules exist under the same names (kernels is the
    16-name kernel ABI)."""
    import importlib
    for mod in ("boundary", "errors", "fas", "grid", "kernels", "manufactured", "schedule",
                "smoothers", "stencil", "transfer", "weno"):
        importlib.import_module(f"paper_2510_11152_b200.{mod}")
    from paper_2510_11152_b200 import kernels
    assert len(kernels._KERNEL_NAMES) == 16
    for nm in kernels._KERNEL_NAMES:
        assert callable(getattr(kernels, nm))
    from paper_2510_11152_b200.stencil import assemble_dense_operator, gradient_axis  # noqa
