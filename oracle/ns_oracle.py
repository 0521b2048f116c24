"""CPU oracle of the projection time steppers -- TEST INFRASTRUCTURE ONLY.

The reference ships no NS driver: this is a
straight-line transcription of the memory-efficient schemes of
PAPER.md Table 3 (first order) and Table 5 (second order,
PAPER.md:867-922) composed from reference primitives restated in
oracle.py (weno3_convect, gradient_axis, divergence_edges_to_cc, FAS
solve), with the source-term association order documented in
paper_2510_11152_b200/ns.py.  Parity at the driver level is therefore
"composed, unpinned"; every primitive underneath is pinned to the reference
golden vectors.  It deliberately does NOT execute schedule Step lists, so it
also checks the product's schedule executor.
"""

from __future__ import annotations

import numpy as np

import oracle as O

LOC = {"u": "edge_ew", "v": "edge_ns", "w": "edge_tb"}
AX = {"u": 0, "v": 1, "w": 2}


def cavity_faces(dim, lid=1.0):
    names = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")[: 2 * dim]
    vel = {nm: ("dirichlet", 0.0) for nm in names}
    u = dict(vel)
    u["yhi" if dim == 2 else "zhi"] = ("dirichlet", lid)
    out = {"u": u, "v": dict(vel), "p": {nm: ("neumann", 0.0) for nm in names}}
    if dim == 3:
        out["w"] = dict(vel)
    return out


def laplacian(F: O.OField) -> np.ndarray:
    """(nsum - 2d c) * inv_h2 at interior points (KER/numpy_backend.py:66-88)."""
    h = 1.0 / F.n[0]
    inv_h2 = 1.0 / (h * h)
    c = F.core
    ext = O.interior_extent(F.n, F.loc)
    sl = lambda d: tuple(slice(1 + d[a], 1 + d[a] + ext[a]) for a in range(F.dim))  # noqa
    z = [0] * F.dim

    def sh(a, s):
        d = list(z)
        d[a] = s
        return c[sl(d)]

    ns = (sh(0, 1) + sh(0, -1)) + sh(1, 1)
    ns = ns + sh(1, -1)
    if F.dim == 3:
        ns = (ns + sh(2, 1)) + sh(2, -1)
    return (ns - (6.0 if F.dim == 3 else 4.0) * c[sl(z)]) * inv_h2


class NSOracle:
    def __init__(self, n, re, dt, order, tol=1e-10, k_max=20, s=2, mesh_level=None, lid=1.0):
        self.n = tuple(n)
        self.dim = len(n)
        self.comps = ("u", "v", "w")[: self.dim]
        self.re, self.dt, self.order = re, dt, order
        self.tol, self.k_max, self.s = tol, k_max, s
        self.ml = mesh_level or int(np.log2(min(n))) - 1
        self.faces = cavity_faces(self.dim, lid)
        self.colors = O.plan_colors("x", self.dim)
        self.un = {c: O.OField(self.n, LOC[c], 2) for c in self.comps}
        self.unm1 = {c: O.OField(self.n, LOC[c], 2) for c in self.comps}
        self.p = O.OField(self.n, "cell", 1)
        self.pt = O.OField(self.n, "cell", 1)  # previous increment (guess)
        for c in self.comps:
            O.fill_ghosts(self.un[c], self.faces[c])
            self.unm1[c].data[...] = self.un[c].data

    def _mix(self, c, a, b, kind):
        M = O.OField(self.n, LOC[c], 2)
        if kind == "ext":
            M.interior[...] = (3.0 * a.interior - b.interior) * 0.5
        else:
            M.interior[...] = (a.interior + b.interior) * 0.5
        O.fill_ghosts(M, self.faces[c])
        return M

    def rhs(self, c, tld):
        dt = self.dt
        vel = []
        for o in self.comps:
            if self.order == 1:
                O.fill_ghosts(self.un[o], self.faces[o])
                vel.append(self.un[o])
            elif o in tld:
                vel.append(self._mix(o, self.un[o], tld[o], "avg"))
            else:
                vel.append(self._mix(o, self.un[o], self.unm1[o], "ext"))
        conv = O.weno3_convect(vel, AX[c])
        gp = O.gradient_axis(self.p, AX[c])
        un = self.un[c].interior
        f = O.OField(self.n, LOC[c], 1)
        if self.order == 1:
            f.interior[...] = (un - dt * conv) - dt * gp
        else:
            O.fill_ghosts(self.un[c], self.faces[c])
            lap = laplacian(self.un[c])
            f.interior[...] = ((un - dt * conv) - dt * gp) + (dt / (2.0 * self.re)) * lap
        return f

    def step(self):
        dt = self.dt
        b_mom = dt / self.re if self.order == 1 else dt / (2.0 * self.re)
        tld = {}
        hist = {}
        for c in self.comps:
            f = self.rhs(c, tld)
            ut = O.OField(self.n, LOC[c], 2, self.un[c].data.copy())  # guess u^n
            it, h = O.fas_solve(ut, f, 1.0, b_mom, self.faces[c], self.colors, self.tol,
                                self.k_max, self.s, self.ml)
            hist[c] = h
            tld[c] = ut
        div = O.OField(self.n, "cell", 1)
        div.interior[...] = -O.divergence_edges_to_cc([tld[c] for c in self.comps])
        it, h = O.fas_solve(self.pt, div, 0.0, dt, self.faces["p"], self.colors, self.tol,
                            self.k_max, self.s, self.ml)
        hist["p"] = h
        for c in self.comps:
            new = O.OField(self.n, LOC[c], 2)
            new.data[...] = self.un[c].data
            new.interior[...] = tld[c].interior - dt * O.gradient_axis(self.pt, AX[c])
            O.fill_ghosts(new, self.faces[c])
            self.unm1[c] = self.un[c]
            self.un[c] = new
        self.p.interior[...] = self.p.interior + self.pt.interior
        return hist
