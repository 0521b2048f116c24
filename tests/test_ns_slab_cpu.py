"""Host-side protocol of the slab Navier-Stokes stepper on CPU: the row
exchange of DistRanks and the rank-ordered chunk-sum gather over real gloo
process groups (world size 2 and 3), against VirtualRanks on the same data
and against slicing the whole array."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_11152_b200.grid import GridLevel, Location
from paper_2510_11152_b200.ns_slab import DistRanks, SlabField, SlabGeom, VirtualRanks

N = (12, 5, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fill_rows(F, full):
    """Local slabs with the interior rows of the whole array and NaN halos."""
    h = F.halo
    for r, t in F.parts.items():
        t.fill_(float("nan"))
        lo = F.geom.lo(r) - 1 + h  # global data row of the rank's first interior row
        m = F.geom.rows(F.location, r)
        t[h: h + m] = full[lo: lo + m]


def _expected(F, full, rows, r):
    """Local array after an exchange of ``rows`` rows: interior + the
    neighbours' rows (whole-array rows), NaN elsewhere."""
    h, geom = F.halo, F.geom
    t = torch.full_like(F.parts[r], float("nan"))
    d0 = geom.lo(r) - 1  # global data row of local row 0
    m = geom.rows(F.location, r)
    t[h: h + m] = full[d0 + h: d0 + h + m]
    if r > 0:
        t[h - rows: h] = full[d0 + h - rows: d0 + h]
    if r < geom.P - 1:
        t[geom.m0 + h: geom.m0 + h + rows] = full[d0 + geom.m0 + h: d0 + geom.m0 + h + rows]
    return t


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = GridLevel(0, N, (0.0,) * 3, tuple(x / N[-1] for x in N))
    geom = SlabGeom(g, world)
    comm = DistRanks()
    ok = True
    for loc, h in ((Location.CELL, 1), (Location.EDGE_EW, 2), (Location.EDGE_NS, 2)):
        F = SlabField(geom, loc, h, comm.ranks, "cpu")
        full = torch.arange(float((N[0] + 2 * h) * F.parts[rank].shape[1] * F.parts[rank].shape[2]),
                            dtype=torch.float64).reshape(-1, *F.parts[rank].shape[1:])
        _fill_rows(F, full)
        for rows in range(1, h + 1):
            comm.exchange(F, rows)
            want = _expected(F, full, rows, rank)
            ok &= torch.equal(torch.nan_to_num(F.parts[rank], nan=-1.0),
                              torch.nan_to_num(want, nan=-1.0))
    sums = comm.gather_chunk_sums({rank: torch.tensor([float(rank), 10.0 + rank],
                                                      dtype=torch.float64)})
    ok &= [s.tolist() for s in sums] == [[float(r), 10.0 + r] for r in range(world)]
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res.values()), res


def test_dist_rank_exchange_gloo_world2():
    _run(2)


def test_dist_rank_exchange_gloo_world3():
    _run(3)


def test_virtual_rank_exchange_matches_slicing():
    g = GridLevel(0, N, (0.0,) * 3, tuple(x / N[-1] for x in N))
    for P in (2, 3):
        geom = SlabGeom(g, P)
        comm = VirtualRanks(P)
        for loc, h in ((Location.CELL, 1), (Location.EDGE_EW, 2), (Location.EDGE_TB, 2)):
            F = SlabField(geom, loc, h, comm.ranks, "cpu")
            shp = F.parts[0].shape
            full = torch.arange(float((N[0] + 2 * h) * shp[1] * shp[2]),
                                dtype=torch.float64).reshape(-1, *shp[1:])
            _fill_rows(F, full)
            comm.exchange(F, h)
            for r in comm.ranks:
                want = _expected(F, full, h, r)
                assert torch.equal(torch.nan_to_num(F.parts[r], nan=-1.0),
                                   torch.nan_to_num(want, nan=-1.0)), (P, loc, r)
