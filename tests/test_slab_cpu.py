"""Host-side logic of the multi-GPU slab decomposition on CPU: slab ranges
and views, and the CUDA-IPC pointer exchange protocol run over a real
world-size-2 gloo process group (fake handle functions stand in for the
device calls)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_11152_b200 import slab as S


def test_slab_cells_and_views():
    assert S.slab_cells(512, 8, 0) == (1, 64)
    assert S.slab_cells(512, 8, 7) == (449, 512)
    assert S.slab_cells(64, 4, 2) == (33, 48)
    with pytest.raises(ValueError):
        S.slab_cells(64, 3, 0)
    data = torch.arange(66 * 4).reshape(66, 4)
    v = S.slab_view(data, 1, 64, 4, 1)            # cells 17..32 + ghosts 16, 33
    assert v.shape[0] == 18 and int(v[0, 0]) == 16 * 4 and int(v[-1, 0]) == 33 * 4
    data2 = torch.arange(68 * 2).reshape(68, 2)    # halo 2: core index x at data x+1
    v2 = S.slab_view(data2, 2, 64, 2, 1)
    assert v2.shape[0] == 34 and int(v2[0, 0]) == (32 + 1) * 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = 1000 * (rank + 1)
    exports = [base + i for i in range(5)]          # this rank's "device pointers"
    handle_of = lambda ptr: f"h{rank}:{ptr}".encode()  # noqa: E731
    opened = {}

    def open_handle(hd):
        r, ptr = hd.decode()[1:].split(":")
        opened[hd] = 10 ** 6 * (int(r) + 1) + int(ptr)  # "mapped" address
        return opened[hd]

    out = S.exchange_ipc(exports, handle_of, open_handle,
                         lambda o, obj: dist.all_gather_object(o, obj), rank, world)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_exchange_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        table = res[r]
        assert len(table) == world
        for src in range(world):
            if src == r:
                assert table[src] == [1000 * (r + 1) + i for i in range(5)]
            else:  # peer pointers come from opening the peer's handles
                assert table[src] == [10 ** 6 * (src + 1) + 1000 * (src + 1) + i for i in range(5)]


def test_slab_view_edge_axis0():
    """Edge axis along the slab axis: core 0..n (walls 0 and n); the last
    rank's view ends at the wall node when the array has no ring beyond it."""
    n = 64
    data = torch.arange((n + 1) * 3).reshape(n + 1, 3)  # halo 1: core x at data x
    v0 = S.slab_view(data, 1, n, 4, 0)
    v3 = S.slab_view(data, 1, n, 4, 3)
    assert int(v0[0, 0]) == 0 and v0.shape[0] == 18           # nodes 0..17
    assert int(v3[0, 0]) == 48 * 3 and v3.shape[0] == 17      # nodes 48..64 (wall)


def _np_chunk(ext):
    B = 8192
    for k in range(len(ext)):
        P = 1
        for a in range(k, len(ext)):
            P *= ext[a]
        if P <= 8192:
            return (8192 // P) * P
    return B


def _mean_worker(rank, world, port, q):
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 32
    full = np.random.default_rng(5).standard_normal((n + 2,) * 3)
    interior = full[1:-1, 1:-1, 1:-1]                     # non-contiguous: buffered reduce
    B = _np_chunk(interior.shape)
    rows = n // world
    mine = np.ascontiguousarray(interior[rank * rows:(rank + 1) * rows]).ravel()
    sums = torch.tensor([np.sum(mine[i:i + B]) for i in range(0, mine.size, B)])
    out = [torch.empty_like(sums) for _ in range(world)]
    dist.all_gather(out, sums)
    q.put((rank, S.ordered_total(out), float(np.sum(interior))))
    dist.barrier()
    dist.destroy_process_group()


def test_ordered_mean_gloo_world2():
    """Distributed ordered mean (SURVEY.md section 8e item v): per-rank chunk
    sums gathered in rank order and totalled in chunk order equal numpy's
    sum of the whole interior view bitwise."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mean_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, tot, ref in res:
        assert tot == ref
