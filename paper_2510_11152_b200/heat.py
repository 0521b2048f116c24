"""Backward-Euler heat-equation driver.

Each step solves ``p^{n+1} - dt*Lap(p^{n+1}) = p^n`` (a = 1, b = dt) with the
FAS solver, starting from ``p^n``; with dt = 1 and f = p^n this is exactly
the paper's benchmark operator ``p - Lap p = f`` (PAPER.md:122-127,
476-515).  The reference ships no heat driver; this is the thin loop over
FasSolver.solve it implies.
"""

from __future__ import annotations

import numpy as np

from .boundary import BoundaryCondition
from .elementwise import COPY, elem
from .fas import FasParams, FasSolver, SolveReport
from .grid import Field, GridLevel, Location, make_hierarchy
from .smoothers import make_plan
from .stencil import OperatorCoeffs


class HeatStepper:
    def __init__(self, grid: GridLevel, dt: float = 1.0, bc: BoundaryCondition | None = None,
                 tol: float = 1e-9, k_max: int = 20, s: int = 2, mesh_level: int | None = None,
                 plan=None, device=None):
        self.grid = grid
        self.dt = dt
        self.bc = bc or BoundaryCondition.dirichlet(grid.dim)
        ml = mesh_level or int(np.log2(min(grid.shape))) - 1
        self.params = FasParams(tol, k_max, s, ml)
        self.solver = FasSolver(make_hierarchy(grid, ml), Location.CELL, self.bc,
                                plan or make_plan("x", grid.dim, "ff"), OperatorCoeffs(1.0, dt))
        self.rhs = Field(grid, Location.CELL, 1, device=device)
        self.reports: list = []

    def step(self, p: Field) -> SolveReport:
        """Advance ``p`` (in place) by one backward-Euler step."""
        elem(COPY, self.rhs.interior, [p.interior])
        rep = self.solver.solve(p, self.rhs, self.params)
        self.reports.append(rep)
        return rep

    def run(self, p: Field, steps: int):
        for _ in range(steps):
            self.step(p)
        return p
