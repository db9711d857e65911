"""Multi-process (gloo, world size 2 and 3) tests of the host logic of the z-slab decomposition:
the library's cgks_decompose (pure host code, no GPU) gives each rank its slab and neighbours;
a 2-plane ghost exchange in the library's send/receive order (send low planes to the lower
neighbour, high planes to the upper, receive the high ghost from the upper, the low ghost from
the lower) must reproduce the periodic global field around every slab.  Also checks the bench's
max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch

    import bench
    from paper_2508_19911_b200.binding import decompose
    off, nl, (lo, hi) = decompose(n, (1, 1, world), rank)
    rng = np.random.default_rng(11)
    glob = rng.standard_normal((n[2], 3, n[1], n[0]))  # [z][field][y][x], as in HBM
    nz = nl[2]
    z0 = off[2]
    loc = np.zeros((nz + 4,) + glob.shape[1:])
    loc[2:nz + 2] = glob[z0:z0 + nz]
    sends = [torch.from_numpy(np.ascontiguousarray(loc[2:4])), torch.from_numpy(np.ascontiguousarray(loc[nz:nz + 2]))]
    rhi = torch.zeros_like(sends[0])
    rlo = torch.zeros_like(sends[0])
    reqs = [dist.isend(sends[0], lo), dist.isend(sends[1], hi), dist.irecv(rhi, hi), dist.irecv(rlo, lo)]
    for r in reqs:
        r.wait()
    loc[nz + 2:nz + 4] = rhi.numpy()
    loc[0:2] = rlo.numpy()
    want = glob[np.arange(z0 - 2, z0 + nz + 2) % n[2]]
    ok = bool(np.array_equal(loc, want))
    t = bench.max_over_ranks(float(rank + 1), world)
    out[rank] = (ok, t, off, nl)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_halo_exchange_gloo(world):
    n = (6, 5, 4 * world * 2)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, out), nprocs=world, join=True)
    for r in range(world):
        ok, t, off, nl = out[r]
        assert ok, f"rank {r} ghost planes wrong"
        assert t == float(world)  # max over ranks
        assert nl == (n[0], n[1], n[2] // world) and off == (0, 0, r * (n[2] // world))


def test_decompose_rejects_unsupported():
    from paper_2508_19911_b200.binding import CgksError, decompose
    with pytest.raises(CgksError):
        decompose((8, 8, 10), (1, 1, 4), 0)  # 10 planes not divisible by 4
    with pytest.raises(CgksError):
        decompose((8, 8, 8), (2, 1, 1), 0)  # only z-slabs
