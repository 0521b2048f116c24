"""Navier-Stokes projection on axis-0 slabs (ns_slab.py; BASELINE.json
configs[4], the 1024^3 cavity across 8 B200) checked on one device:

* the slab ghost fill (exchange + fasmg_fill_ghosts_slab) equals the
  whole-field fill_ghosts on every local row, every location, halo and BC;
* P virtual ranks (one process, device-copy exchanges, VirtualSlabSolver)
  and 2 real processes (DistRanks over gloo, DistSlabSolver over CUDA IPC)
  give fields bitwise equal to the single-GPU stepper and residual
  histories within 1e-12."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cases as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11152_b200 as pkg
    return pkg


@pytest.mark.parametrize("loc", ["cell", "edge_ew", "edge_ns", "edge_tb"])
@pytest.mark.parametrize("halo", [1, 2])
@pytest.mark.parametrize("bc", ["dirichlet", "dirichlet_val", "neumann", "lid"])
@pytest.mark.parametrize("parts", [2, 4])
def test_slab_fill_equals_whole_field_fill(P, loc, halo, bc, parts):
    from paper_2510_11152_b200.ns_slab import SlabField, SlabGeom, VirtualRanks
    from paper_2510_11152_b200.ns import ProjectionStepper  # noqa: F401
    n = (16, 8, 12)
    g = P.GridLevel(0, n, (0.0,) * 3, tuple(x / n[-1] for x in n))
    L = getattr(P.Location, loc.upper())
    faces = C.bc_faces(3, bc)
    bcond = P.BoundaryCondition(3, tuple((k, P.FaceRule(*v)) for k, v in faces.items()))
    ref = P.Field(g, L, halo, C.rand_field(7, n, loc, halo))
    P.fill_ghosts(ref, bcond)
    geom = SlabGeom(g, parts)
    comm = VirtualRanks(parts)
    F = SlabField(geom, L, halo, comm.ranks, ref.device)
    for r in comm.ranks:
        lo = geom.lo(r) - 1
        rows = geom.rows(L, r)
        F.parts[r].fill_(float("nan"))
        F.interior(r)[...] = ref.interior[lo: lo + rows]

    class _S:  # the stepper's refresh on a bare geometry
        pass
    st = _S()
    st.comm, st.geom, st.grid = comm, geom, g
    from paper_2510_11152_b200.ns_slab import SlabProjectionStepper
    SlabProjectionStepper._refresh(st, F, bcond)
    for r in comm.ranks:
        t = F.parts[r]
        # global data rows of this slab's local rows (those that exist globally)
        d0 = geom.lo(r) - 1  # global data row of local row 0
        nrow = min(t.shape[0], ref.data.shape[0] - d0)
        got = t[:nrow]
        want = ref.data[d0: d0 + nrow]
        if L.edge_axis == 0 and r == parts - 1:
            pass  # the last slab also holds the wall node and the rings beyond
        assert torch.equal(torch.nan_to_num(got, nan=1e300), torch.nan_to_num(want, nan=1e300)), \
            (r, (got != want).nonzero()[:5].tolist())


def _single(P, n, order, dt=1e-3):
    from paper_2510_11152_b200.ns import NSParams, ProjectionStepper
    st = ProjectionStepper(P.unit_grid(n), NSParams(re=100.0, dt=dt, order=order, tol=1e-10,
                                                    k_max=20))
    st.set_state({})
    return st


@pytest.mark.parametrize("n,parts,order", [((32, 32, 32), 2, 2), ((32, 32, 32), 4, 2),
                                           ((32, 32, 32), 2, 1), ((64, 64, 64), 4, 2),
                                           ((64, 32, 96), 2, 2)])
def test_virtual_slab_ns_matches_single_gpu(P, n, parts, order):
    from paper_2510_11152_b200.ns import NSParams
    from paper_2510_11152_b200.ns_slab import SlabProjectionStepper, VirtualRanks
    g = P.GridLevel(0, n, (0.0,) * 3, tuple(x / n[-1] for x in n))
    from paper_2510_11152_b200.ns import ProjectionStepper
    ref = ProjectionStepper(g, NSParams(re=100.0, dt=1e-3, order=order, tol=1e-10, k_max=20))
    ref.set_state({})
    sl = SlabProjectionStepper(g, NSParams(re=100.0, dt=1e-3, order=order, tol=1e-10, k_max=20),
                               VirtualRanks(parts))
    sl.set_state({})
    for k in range(2):
        a = ref.step()
        b = sl.step()
        for c in ref.comps:
            np.testing.assert_allclose(b.momentum[c].residual_history,
                                       a.momentum[c].residual_history, rtol=1e-12, atol=0)
        np.testing.assert_allclose(b.pressure.residual_history, a.pressure.residual_history,
                                   rtol=1e-12, atol=0)
        for c in ref.comps:
            assert torch.equal(sl.velocity_global(c), ref.velocity(c).interior), (k, c)
        assert torch.equal(sl.pressure_global(), ref.pressure().interior), k
    assert sl.divergence() == ref.divergence()
    sl.close()


@pytest.mark.parametrize("world", [2, 4])
def test_process_slab_ns_matches_single_gpu(world):
    """``world`` processes sharing the device (gloo for the row exchanges,
    CUDA IPC for the solver's halo push): every rank's gathered fields equal
    the single-GPU stepper's bitwise (scripts/ns_slab_selftest.py)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = 29700 + world
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "scripts", "ns_slab_selftest.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, NS_SLAB_N="32"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("bitwise True") == world, r.stdout
