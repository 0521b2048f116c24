"""Experiment command line over the B200 FAS path (module
``bench-cli``: the caller of the hot path).

    python -m paper_2510_11152_b200 poisson --mode asymptotic --dim 3 --size 32,64,128
    python -m paper_2510_11152_b200 poisson --mode algebraic --size 256,512,1024
    python -m paper_2510_11152_b200 smoother-compare --size 512
    python -m paper_2510_11152_b200 ns --mode temporal --order 2 --size 512
    python -m paper_2510_11152_b200 ns --mode divergence --size 128 --steps 500
    python -m paper_2510_11152_b200 ns --mode cavity --re 100 --size 256 --ghia data/ghia1982.txt
    python -m paper_2510_11152_b200 ns --mode schedule-audit
    python -m paper_2510_11152_b200 timing --dim 3 --size 128,256,512

Every run is one experiment.  Configuration: a flat JSON object
(``--config PATH``; unknown keys rejected) overridden by flags.  Output: CSV
with a ``#`` provenance line (command, config SHA-256, seed, device), a
header row, shortest round-trip floats, '.' decimal separator.  Exit codes:
0 success, 2 configuration error, 3 not converged (with ``--strict``).
All numerics run on the GPU through the package's public API; there is no
CPU path (the SPEC's thread count is accepted and recorded only).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys

import numpy as np

# config key -> (type, default)
KEYS = {
    "mode": (str, None),
    "dim": (int, 2),
    "size": (list, None),
    "dt": (list, None),
    "re": (float, None),
    "tol": (float, None),
    "kmax": (int, None),
    "smooth_steps": (int, 2),
    "mesh_level": (int, None),
    "smoother": (str, "x"),
    "sequence": (str, "ff"),
    "order": (int, 1),
    "schedule": (str, "efficient"),
    "threads": (int, 1),
    "seed": (int, 0),
    "out": (str, None),
    "steps": (int, None),
    "t_end": (float, None),
    "ghia": (str, None),
    "profiles_only": (bool, False),
    "strict": (bool, False),
    "cycles": (int, 10),
    "forcing": (str, "trap"),
}

MODES = {"poisson": ("algebraic", "asymptotic"),
         "ns": ("temporal", "cavity", "divergence", "schedule-audit")}

GHIA_DEFAULT = os.path.join("data", "ghia1982.txt")


class ConfigError(Exception):
    pass


class NotConverged(Exception):
    pass


def _num_list(v, cast):
    if isinstance(v, str):
        v = [x for x in v.split(",") if x.strip()]
    if isinstance(v, (int, float)):
        v = [v]
    out = []
    for x in v:
        if isinstance(x, str) and "/" in x:
            a, b = x.split("/")
            out.append(cast(float(a) / float(b)))
        else:
            out.append(cast(x))
    return out


def load_config(cmd: str, path: str | None, flags: dict) -> dict:
    """Flat JSON config + flag overrides (flags win), schema-checked."""
    cfg = {}
    if path:
        try:
            with open(path) as fh:
                raw = json.load(fh)
        except (OSError, ValueError) as e:
            raise ConfigError(f"cannot read config {path}: {e}")
        if not isinstance(raw, dict):
            raise ConfigError("config must be a flat JSON object")
        for k, v in raw.items():
            if k not in KEYS:
                raise ConfigError(f"unknown config key {k!r}")
            if isinstance(v, (dict,)) or (isinstance(v, list) and any(isinstance(x, (dict, list)) for x in v)):
                raise ConfigError(f"config key {k!r}: nesting beyond one level")
            cfg[k] = v
    for k, v in flags.items():
        if v is not None:
            cfg[k] = v
    out = {}
    for k, (typ, dflt) in KEYS.items():
        v = cfg.get(k, dflt)
        if v is None:
            out[k] = None
            continue
        try:
            if k == "size":
                v = _num_list(v, int)
            elif k == "dt":
                v = _num_list(v, float)
            elif typ is bool:
                v = bool(v)
            else:
                v = typ(v)
        except (TypeError, ValueError):
            raise ConfigError(f"config key {k!r}: bad value {cfg.get(k)!r}")
        out[k] = v
    if cmd in MODES:
        if out["mode"] is None:
            raise ConfigError(f"{cmd}: --mode is required ({'|'.join(MODES[cmd])})")
        if out["mode"] not in MODES[cmd]:
            raise ConfigError(f"{cmd}: unknown mode {out['mode']!r}")
    if out["dim"] not in (2, 3):
        raise ConfigError("dim must be 2 or 3")
    if out["smoother"] not in ("x", "rbgs", "u", "z"):
        raise ConfigError(f"unknown smoother {out['smoother']!r}")
    if out["sequence"] not in ("ff", "fb"):
        raise ConfigError(f"unknown sequence {out['sequence']!r}")
    if out["forcing"] not in ("mid", "trap"):
        raise ConfigError(f"unknown forcing rule {out['forcing']!r}")
    if out["order"] not in (1, 2):
        raise ConfigError("order must be 1 or 2")
    if out["schedule"] not in ("classical", "efficient"):
        raise ConfigError(f"unknown schedule {out['schedule']!r}")
    if out["size"] is not None:
        if not out["size"]:
            raise ConfigError("empty size list")
        if any(n < 4 or n & (n - 1) for n in out["size"]):
            raise ConfigError("sizes must be powers of two >= 4")
    return out


def fmt(v) -> str:
    """Shortest round-trip text of a CSV cell."""
    if isinstance(v, bool):
        return "1" if v else "0"
    if isinstance(v, float):
        if math.isnan(v):
            return "nan"
        return repr(v)
    if v is None:
        return ""
    return str(v)


class Csv:
    def __init__(self, cmd: str, cfg: dict, stream):
        self.stream = stream
        blob = json.dumps(cfg, sort_keys=True).encode()
        dev = "none"
        try:
            import torch
            if torch.cuda.is_available():
                dev = torch.cuda.get_device_name(0).replace(",", " ")
        except Exception:
            pass
        self.stream.write(f"# fasmg-b200 {cmd}; config_sha256={hashlib.sha256(blob).hexdigest()}; "
                          f"seed={cfg['seed']}; threads={cfg['threads']}; device={dev}\n")
        self.header = None

    def row(self, **kv):
        if self.header is None:
            self.header = list(kv)
            self.stream.write(",".join(self.header) + "\n")
        self.stream.write(",".join(fmt(kv[k]) for k in self.header) + "\n")
        self.stream.flush()


# ---------------------------------------------------------------- helpers
def _pkg():
    import paper_2510_11152_b200 as P
    return P


def _l2(grid, e) -> float:
    return float(grid.h ** (grid.dim / 2.0) * np.sqrt(np.sum(np.asarray(e) ** 2)))


def _ml(cfg, n):
    return cfg["mesh_level"] or int(math.log2(n)) - 1


def _solve_params(cfg, n, tol=1e-9, kmax=20):
    P = _pkg()
    return P.FasParams(cfg["tol"] or tol, cfg["kmax"] or kmax, cfg["smooth_steps"], _ml(cfg, n))


# ---------------------------------------------------------------- poisson
def cmd_poisson(cfg, out: Csv):
    """algebraic: residual + error per cycle (Fig. algebraic2D/3D,
    PAPER.md:376-410); asymptotic: error and order per size (Tables
    err_2D/err_3D)."""
    P = _pkg()
    from . import manufactured as M
    dim = cfg["dim"]
    sizes = cfg["size"] or ([256, 512, 1024] if dim == 2 else [32, 64, 128])
    plan = P.make_plan(cfg["smoother"], dim, cfg["sequence"])
    bc = P.BoundaryCondition.dirichlet(dim)
    coeffs = P.OperatorCoeffs(1.0, 1.0)
    prev = None
    converged = True
    for n in sizes:
        g = P.unit_grid((n,) * dim)
        exact = M.poisson_exact_array(g)
        prm = _solve_params(cfg, n)
        if cfg["mode"] == "asymptotic":
            p = P.Field(g, P.Location.CELL)
            f = M.poisson_rhs_continuous(g)
            _, rep = P.solve(p, f, coeffs, prm, plan, bc)
            err = _l2(g, p.interior.cpu().numpy() - exact)
            order = "" if prev is None else math.log(prev[1] / err) / math.log(n / prev[0])
            out.row(dim=dim, size=n, iterations=rep.iterations, final_residual=rep.final_residual,
                    error=err, order=order)
            prev = (n, err)
            converged &= rep.converged
        else:
            rng = np.random.default_rng(cfg["seed"])
            p0 = np.zeros(tuple(x + 2 for x in g.shape))
            p0[(slice(1, -1),) * dim] = rng.random(g.shape)
            p = P.Field(g, P.Location.CELL, 1, p0)
            f = M.poisson_rhs_discrete(g)
            S = P.FasSolver(P.make_hierarchy(g, prm.mesh_level), P.Location.CELL, bc, plan, coeffs)
            one = P.FasParams(prm.tol, 1, prm.s, prm.mesh_level)
            P.fill_ghosts(p, bc)
            res = P.norm_l2_scaled(P.residual(f, p, coeffs))
            out.row(dim=dim, size=n, cycle=0, residual=float(res),
                    error=_l2(g, p.interior.cpu().numpy() - exact))
            k = 0
            while k < prm.k_max and res >= prm.tol:
                rep = S.solve(p, f, one)
                k += 1
                res = rep.final_residual
                out.row(dim=dim, size=n, cycle=k, residual=res,
                        error=_l2(g, p.interior.cpu().numpy() - exact))
            converged &= res < prm.tol
    if not converged:
        raise NotConverged("poisson: a solve hit kMax")


def cmd_smoother_compare(cfg, out: Csv):
    """Total V-cycles of the six ordering configurations (Fig.
    smoothing-test)."""
    P = _pkg()
    from . import manufactured as M
    dim = cfg["dim"]
    n = (cfg["size"] or [512])[0]
    g = P.unit_grid((n,) * dim)
    rng = np.random.default_rng(cfg["seed"])
    p0 = np.zeros(tuple(x + 2 for x in g.shape))
    p0[(slice(1, -1),) * dim] = rng.random(g.shape)
    f0 = M.poisson_rhs_discrete(g)
    prm = _solve_params(cfg, n, kmax=100)
    for shape in ("x", "u", "z"):
        for seq in ("ff", "fb"):
            p = P.Field(g, P.Location.CELL, 1, p0.copy())
            _, rep = P.solve(p, f0.copy(), P.OperatorCoeffs(1.0, 1.0), prm,
                             P.make_plan(shape, dim, seq), P.BoundaryCondition.dirichlet(dim))
            out.row(dim=dim, size=n, shape=shape, sequence=seq, iterations=rep.iterations,
                    final_residual=rep.final_residual, converged=rep.converged)


# ---------------------------------------------------------------- ns
def _ns_params(cfg, n, re, dt, tol):
    from .ns import NSParams
    return NSParams(re=re, dt=dt, order=cfg["order"], mode=cfg["schedule"],
                    tol=cfg["tol"] or tol, k_max=cfg["kmax"] or 20, s=cfg["smooth_steps"],
                    mesh_level=_ml(cfg, n))


def ns_temporal(cfg, out: Csv):
    """Asymptotic-in-time test (Tables 7-8): Re=10,
    manufactured 2D solution with body force, errors at t=1 per dt."""
    P = _pkg()
    from . import manufactured as M
    from .ns import ProjectionStepper
    n = (cfg["size"] or [512])[0]
    re = cfg["re"] or 10.0
    dts = cfg["dt"] or [1 / 10, 1 / 20, 1 / 40, 1 / 80, 1 / 160]
    t_end = cfg["t_end"] or 1.0
    g = P.unit_grid((n, n))
    bcs = {"u": P.BoundaryCondition.dirichlet(2), "v": P.BoundaryCondition.dirichlet(2),
           "p": P.BoundaryCondition.neumann(2)}
    # The body force is sin(t)*A + cos(t)*B + sin(t)^2*C per component
    # (PKG/manufactured.py:115-147): tabulate A, B, C once on the device
    # (from t = pi/2, 0, -pi/2) so each step's force is three fused
    # multiply-adds instead of a host evaluation and upload.
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    parts = {}
    for c in ("u", "v"):
        f1, f2, f3 = (torch.as_tensor(M.flow_forcing(c, g, t, re), device=dev)
                      for t in (math.pi / 2, 0.0, -math.pi / 2))
        parts[c] = (0.5 * (f1 - f3), f2, 0.5 * (f1 + f3))

    def force(c, t):
        a, b, q = parts[c]
        s_, c_ = math.sin(t), math.cos(t)
        return a * s_ + b * c_ + q * (s_ * s_)

    prev = None
    for dt in dts:
        steps = int(round(t_end / dt))
        st = ProjectionStepper(g, _ns_params(cfg, n, re, dt, 1e-9), bcs, forcing=force)
        st.forcing_rule = cfg["forcing"]
        st.set_state({})
        worst = 0
        for _ in range(steps):
            rep = st.step()
            worst = max([worst, rep.pressure.iterations]
                        + [r.iterations for r in rep.momentum.values()])
        T = steps * dt
        eu = _l2(g, st.velocity("u").interior.cpu().numpy() - M.flow_exact_u(g, T))
        ev = _l2(g, st.velocity("v").interior.cpu().numpy() - M.flow_exact_v(g, T))
        ep = _l2(g, st.pressure().interior.cpu().numpy() - M.flow_exact_p(g, T))
        row = dict(order=cfg["order"], size=n, re=re, dt=dt, steps=steps, err_u=eu, err_v=ev,
                   err_p=ep, order_u="", order_v="", order_p="", max_cycles=worst)
        if prev is not None:
            r = math.log(prev[0] / dt)
            row.update(order_u=math.log(prev[1] / eu) / r, order_v=math.log(prev[2] / ev) / r,
                       order_p=math.log(prev[3] / ep) / r)
        out.row(**row)
        prev = (dt, eu, ev, ep)


def _read_ghia(path):
    """Ghia et al. (1982) centerline table: '#' comments,
    then rows 'y u_Re100 u_Re400 u_Re1000', a blank line, rows
    'x v_Re100 v_Re400 v_Re1000'."""
    blocks, cur = [], []
    with open(path) as fh:
        for line in fh:
            s = line.strip()
            if s.startswith("#"):
                continue
            if not s:
                if cur:
                    blocks.append(np.array(cur))
                    cur = []
                continue
            cur.append([float(x) for x in s.split()])
    if cur:
        blocks.append(np.array(cur))
    if len(blocks) != 2:
        raise ConfigError(f"{path}: expected two blocks (u and v profiles)")
    return blocks


def ns_cavity(cfg, out: Csv):
    """Lid-driven cavity to steady state: centerline
    u(y) and v(x) plus deltas to the Ghia table."""
    P = _pkg()
    from .ns import ProjectionStepper, cavity_bcs, centerline_profiles
    dim = cfg["dim"]
    n = (cfg["size"] or [256])[0]
    re = cfg["re"] or 100.0
    dt = (cfg["dt"] or [1e-3])[0]
    ghia = None
    if not cfg["profiles_only"]:
        path = cfg["ghia"] or GHIA_DEFAULT
        if not os.path.exists(path):
            raise ConfigError(f"Ghia reference data not found at {path!r} (expected the "
                              f"SPEC.md:521-523 format; pass --ghia PATH or --profiles-only)")
        ghia = _read_ghia(path)
    g = P.unit_grid((n,) * dim)
    st = ProjectionStepper(g, _ns_params(cfg, n, re, dt, 1e-10), cavity_bcs(dim))
    st.set_state({})
    t_end = cfg["t_end"] or 50.0
    max_steps = cfg["steps"] or int(round(t_end / dt))
    prev = st.velocity("u").interior.clone()
    steady = False
    k = 0
    for k in range(1, max_steps + 1):
        st.step()
        if k % 10 == 0:
            u = st.velocity("u").interior
            d = float((u - prev).pow(2).sum().sqrt()) * g.h ** (dim / 2.0) / (10 * dt)
            prev = u.clone()
            if d < 1e-7:
                steady = True
                break
    u_line, v_line = centerline_profiles(st)
    yc = (np.arange(n) + 0.5) / n      # cell centers (u along the vertical line)
    xe = np.arange(1, n) / n           # v-edge positions along the horizontal line
    if len(v_line) == n:
        xe = yc
    delta = {"u": None, "v": None}
    if ghia is not None:
        ci = {100.0: 1, 400.0: 2, 1000.0: 3}.get(float(re))
        if ci is None:
            raise ConfigError("Ghia data covers Re = 100, 400, 1000")
        gu, gv = ghia
        delta["u"] = (gu[:, 0], np.interp(gu[:, 0], yc, u_line) - gu[:, ci])
        delta["v"] = (gv[:, 0], np.interp(gv[:, 0], xe, v_line) - gv[:, ci])
    for name, coord, line in (("u", yc, u_line), ("v", xe, v_line)):
        for x, val in zip(coord, line):
            out.row(re=re, size=n, steps=k, steady=steady, profile=name, coord=float(x),
                    value=float(val), ghia_coord="", ghia_delta="")
        if delta[name] is not None:
            for x, d in zip(*delta[name]):
                out.row(re=re, size=n, steps=k, steady=steady, profile=name + "_ghia",
                        coord="", value="", ghia_coord=float(x), ghia_delta=float(d))
    if ghia is not None:
        out.stream.write(f"# max|u-ghia|={float(np.abs(delta['u'][1]).max())!r} "
                         f"max|v-ghia|={float(np.abs(delta['v'][1]).max())!r}\n")


def ns_divergence(cfg, out: Csv):
    """integral_divergence per step of a cavity run (Fig. div-u; SPEC.md
    acceptance 7: |.| <= 1e-12 at every step)."""
    P = _pkg()
    from .ns import ProjectionStepper, cavity_bcs
    dim = cfg["dim"]
    n = (cfg["size"] or [128])[0]
    re = cfg["re"] or 100.0
    dt = (cfg["dt"] or [1e-3])[0]
    g = P.unit_grid((n,) * dim)
    st = ProjectionStepper(g, _ns_params(cfg, n, re, dt, 1e-10), cavity_bcs(dim))
    st.set_state({})
    for k in range(1, (cfg["steps"] or 500) + 1):
        rep = st.step()
        out.row(step=k, t=k * dt, integral_divergence=st.divergence(),
                pressure_cycles=rep.pressure.iterations,
                momentum_cycles=max(r.iterations for r in rep.momentum.values()))


def ns_schedule_audit(cfg, out: Csv):
    """Validator report for the four slot schedules (Tables 2-5)."""
    from .schedule import build_schedule, validate_schedule
    for dim in (2, 3):
        for order in (1, 2):
            ref = build_schedule(order, "classical", dim)
            for mode in ("classical", "efficient"):
                sch = build_schedule(order, mode, dim)
                probs = validate_schedule(sch, None if mode == "classical" else ref)
                out.row(dim=dim, order=order, mode=mode, slots=len(sch.slots),
                        status="ok" if not probs else "; ".join(probs).replace(",", ";"))


def cmd_ns(cfg, out: Csv):
    {"temporal": ns_temporal, "cavity": ns_cavity, "divergence": ns_divergence,
     "schedule-audit": ns_schedule_audit}[cfg["mode"]](cfg, out)


# ---------------------------------------------------------------- timing
def cmd_timing(cfg, out: Csv):
    """Per-V-cycle device time: 10 timed cycles per size
    (CUDA events on the solver stream, inputs resident), mean and stddev."""
    import torch
    P = _pkg()
    dim = cfg["dim"]
    sizes = cfg["size"] or ([1024, 2048, 4096] if dim == 2 else [128, 256, 512])
    for n in sizes:
        g = P.unit_grid((n,) * dim)
        p = P.Field(g, P.Location.CELL)
        f = P.Field(g, P.Location.CELL)
        gen = torch.Generator(device=p.device).manual_seed(cfg["seed"])
        p.interior = torch.rand(p.interior.shape, dtype=torch.float64, device=p.device,
                                generator=gen)
        f.interior = torch.rand(f.interior.shape, dtype=torch.float64, device=p.device,
                                generator=gen)
        S = P.FasSolver(P.make_hierarchy(g, _ml(cfg, n)), P.Location.CELL,
                        P.BoundaryCondition.dirichlet(dim),
                        P.make_plan(cfg["smoother"], dim, cfg["sequence"]),
                        P.OperatorCoeffs(1.0, 1.0))
        e = S.engine(cfg["smooth_steps"], p.device)
        e.load(p, f)
        e.run(2, True)
        st = torch.cuda.ExternalStream(e.stream.value)
        ts = []
        for _ in range(cfg["cycles"]):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            e.run(1, True)
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts = np.array(ts)
        dof = n ** dim
        out.row(dim=dim, size=n, cycles=len(ts), mean_ms=float(ts.mean()), std_ms=float(ts.std()),
                min_ms=float(ts.min()), mdof_per_s=dof / float(ts.mean()) / 1e3,
                kernels_per_cycle=e.kernels_per_vcycle(), threads=cfg["threads"])


COMMANDS = {"poisson": cmd_poisson, "smoother-compare": cmd_smoother_compare, "ns": cmd_ns,
            "timing": cmd_timing}


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2510_11152_b200",
                                 description="FAS multigrid experiments on the B200 path")
    ap.add_argument("command", choices=sorted(COMMANDS))
    ap.add_argument("--config")
    ap.add_argument("--mode")
    ap.add_argument("--dim", type=int)
    ap.add_argument("--size")
    ap.add_argument("--dt")
    ap.add_argument("--re", type=float)
    ap.add_argument("--tol", type=float)
    ap.add_argument("--kmax", type=int)
    ap.add_argument("--smooth-steps", dest="smooth_steps", type=int)
    ap.add_argument("--mesh-level", dest="mesh_level", type=int)
    ap.add_argument("--smoother")
    ap.add_argument("--sequence")
    ap.add_argument("--order", type=int)
    ap.add_argument("--schedule")
    ap.add_argument("--threads", type=int)
    ap.add_argument("--seed", type=int)
    ap.add_argument("--steps", type=int)
    ap.add_argument("--t-end", dest="t_end", type=float)
    ap.add_argument("--cycles", type=int)
    ap.add_argument("--forcing", help="order-2 body-force rule: trap ((F^n+F^{n+1})/2, default: reproduces "
                         "Table 8) | mid (F(t^{n+1/2}))")
    ap.add_argument("--ghia")
    ap.add_argument("--profiles-only", dest="profiles_only", action="store_true", default=None)
    ap.add_argument("--strict", action="store_true", default=None)
    ap.add_argument("--out")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    flags = {k: v for k, v in vars(a).items() if k not in ("command", "config")}
    try:
        cfg = load_config(a.command, a.config, flags)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    stream = open(cfg["out"], "w") if cfg["out"] else sys.stdout
    try:
        COMMANDS[a.command](cfg, Csv(a.command, cfg, stream))
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except NotConverged as e:
        print(f"not converged: {e}", file=sys.stderr)
        return 3 if cfg["strict"] else 0
    finally:
        if stream is not sys.stdout:
            stream.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
