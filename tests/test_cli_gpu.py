"""Experiment CLI on the GPU: paper known answers through the command line
(SPEC.md acceptance criteria 1-3, 4, 5, 7 at reduced sizes)."""
import io

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def csv_rows(argv, capsys):
    from paper_2510_11152_b200 import cli
    rc = cli.main(argv)
    out = capsys.readouterr().out
    assert rc == 0, out
    lines = [l for l in out.splitlines() if not l.startswith("#")]
    head = lines[0].split(",")
    return [dict(zip(head, l.split(","))) for l in lines[1:]]


def test_poisson_asymptotic_3d(capsys):
    rows = csv_rows(["poisson", "--mode", "asymptotic", "--dim", "3", "--size", "32,64"], capsys)
    err = [float(r["error"]) for r in rows]
    assert abs(err[0] - 1.74e-3) / 1.74e-3 < 0.02 and abs(err[1] - 4.33e-4) / 4.33e-4 < 0.02
    assert 1.95 <= float(rows[1]["order"]) <= 2.05


def test_poisson_algebraic_h_independent(capsys):
    rows = csv_rows(["poisson", "--mode", "algebraic", "--size", "64,128,256"], capsys)
    last = {}
    for r in rows:
        last[int(r["size"])] = int(r["cycle"])
    assert max(last.values()) - min(last.values()) <= 2
    assert all(float(r["residual"]) < 1e-9 for r in rows if int(r["cycle"]) == last[int(r["size"])])


def test_smoother_compare_x_fewest(capsys):
    rows = csv_rows(["smoother-compare", "--size", "256"], capsys)
    it = {(r["shape"], r["sequence"]): int(r["iterations"]) for r in rows}
    assert it[("x", "ff")] == min(it.values())
    assert it[("x", "ff")] <= 0.7 * max(it[("u", "ff")], it[("u", "fb")])


def test_ns_temporal_first_order(capsys):
    rows = csv_rows(["ns", "--mode", "temporal", "--order", "1", "--size", "64",
                     "--dt", "1/10,1/20,1/40"], capsys)
    assert len(rows) == 3
    for key in ("order_u", "order_v"):
        assert 0.7 < float(rows[-1][key]) < 1.4


def test_ns_divergence_machine_precision(capsys):
    rows = csv_rows(["ns", "--mode", "divergence", "--size", "32", "--steps", "20"], capsys)
    assert len(rows) == 20
    assert max(abs(float(r["integral_divergence"])) for r in rows) <= 1e-12


def test_timing_rows(capsys):
    rows = csv_rows(["timing", "--dim", "2", "--size", "256", "--cycles", "3"], capsys)
    assert len(rows) == 1 and float(rows[0]["mean_ms"]) > 0 and int(rows[0]["cycles"]) == 3
