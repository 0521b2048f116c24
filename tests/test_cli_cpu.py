"""Experiment CLI (paper_2510_11152_b200/cli.py): config
schema, CSV format and the GPU-free subcommands, on CPU."""
import io
import json

import pytest

from paper_2510_11152_b200 import cli


def run(argv, capsys):
    rc = cli.main(argv)
    cap = capsys.readouterr()
    return rc, cap.out, cap.err


def test_schedule_audit_rows(capsys):
    rc, out, _ = run(["ns", "--mode", "schedule-audit"], capsys)
    assert rc == 0
    lines = out.strip().splitlines()
    assert lines[0].startswith("# fasmg-b200 ns; config_sha256=")
    assert lines[1] == "dim,order,mode,slots,status"
    rows = [l.split(",") for l in lines[2:]]
    assert [int(r[3]) for r in rows] == [9, 6, 11, 6, 12, 8, 15, 8]   # Tables 2-5 (+2D)
    assert all(r[4] == "ok" for r in rows)


@pytest.mark.parametrize("argv,msg", [
    (["poisson", "--mode", "asymptotic", "--size", ""], "empty size list"),
    (["poisson"], "--mode is required"),
    (["poisson", "--mode", "spectral"], "unknown mode"),
    (["poisson", "--mode", "algebraic", "--size", "100"], "powers of two"),
    (["ns", "--mode", "temporal", "--order", "3"], "order must be 1 or 2"),
    (["timing", "--smoother", "jacobi"], "unknown smoother"),
])
def test_config_errors_exit_2(capsys, argv, msg):
    rc, _, err = run(argv, capsys)
    assert rc == 2 and msg in err


def test_unknown_config_key_rejected(tmp_path, capsys):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps({"mode": "asymptotic", "sizes": [32]}))
    rc, _, err = run(["poisson", "--config", str(p)], capsys)
    assert rc == 2 and "unknown config key 'sizes'" in err


def test_nested_config_rejected(tmp_path, capsys):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps({"mode": "asymptotic", "size": [[32]]}))
    rc, _, err = run(["poisson", "--config", str(p)], capsys)
    assert rc == 2 and "nesting" in err


def test_flags_override_config():
    cfg = cli.load_config("ns", None, {"mode": "temporal", "dt": "1/10,1/20", "order": 2})
    assert cfg["dt"] == [0.1, 0.05] and cfg["order"] == 2 and cfg["re"] is None
    cfg2 = cli.load_config("poisson", None, {"mode": "algebraic", "size": "256,512"})
    assert cfg2["size"] == [256, 512]


def test_missing_ghia_names_path(capsys):
    rc, _, err = run(["ns", "--mode", "cavity", "--ghia", "/nonexistent/ghia.txt"], capsys)
    assert rc == 2 and "/nonexistent/ghia.txt" in err


def test_csv_shortest_roundtrip():
    for x in (0.1, 1e-300, 2.0 / 3.0, 1.7400000000000002e-3):
        assert float(cli.fmt(x)) == x and cli.fmt(x) == repr(x)
    buf = io.StringIO()
    c = cli.Csv("poisson", cli.load_config("poisson", None, {"mode": "algebraic"}), buf)
    c.row(a=1, b=0.5, c="")
    c.row(a=2, b=float("nan"), c=None)
    lines = buf.getvalue().splitlines()
    assert lines[1:] == ["a,b,c", "1,0.5,", "2,nan,"]


def test_ghia_reader(tmp_path):
    p = tmp_path / "g.txt"
    p.write_text("# comment\n0.0 0.0 0.0 0.0\n1.0 1.0 1.0 1.0\n\n0.0 0.0 0.0 0.0\n1.0 0.0 0.0 0.0\n")
    u, v = cli._read_ghia(str(p))
    assert u.shape == (2, 4) and v.shape == (2, 4)
