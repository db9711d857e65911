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


# ---------------------------------------------------------------------------
# pencils / y-slabs, nproc = (1, Py, Pz): cgks_decompose_pencil and the library's exchange order (the y strips of
# the own planes first, then whole z planes including the fresh y ghost rows, which carry the edge ghosts along)
# ---------------------------------------------------------------------------
def _pencil_local(glob, off, nl):
    """[z + 4][field][y + 4][x] block of a rank with empty ghosts (the library's storage of a pencil rank)."""
    y0, ny, z0, nz = off[1], nl[1], off[2], nl[2]
    loc = np.full((nz + 4, glob.shape[1], ny + 4, glob.shape[3]), np.nan)
    loc[2:nz + 2, :, 2:ny + 2] = glob[z0:z0 + nz, :, y0:y0 + ny]
    return loc


def _pencil_want(glob, off, nl, n):
    y0, ny, z0, nz = off[1], nl[1], off[2], nl[2]
    zi = np.arange(z0 - 2, z0 + nz + 2) % n[2]
    yi = np.arange(y0 - 2, y0 + ny + 2) % n[1]
    return glob[zi][:, :, yi]


@pytest.mark.parametrize("Py,Pz", [(2, 1), (2, 2), (3, 2), (1, 3)])
def test_pencil_decomposition_and_exchange_order(Py, Pz):
    from paper_2508_19911_b200.binding import decompose_pencil
    n = (5, 4 * Py, 4 * Pz)
    P = Py * Pz
    rng = np.random.default_rng(12)
    glob = rng.standard_normal((n[2], 3, n[1], n[0]))
    info = [decompose_pencil(n, (1, Py, Pz), r) for r in range(P)]
    # the blocks tile the grid, rank = ry + Py rz, neighbours are reciprocal
    cover = np.zeros((n[2], n[1]), dtype=int)
    for r, (off, nl, nb) in enumerate(info):
        assert nl == (n[0], n[1] // Py, n[2] // Pz) and off == (0, (r % Py) * nl[1], (r // Py) * nl[2])
        cover[off[2]:off[2] + nl[2], off[1]:off[1] + nl[1]] += 1
        assert info[nb[0]][2][1] == r and info[nb[1]][2][0] == r  # y lower's upper is me, y upper's lower is me
        assert info[nb[2]][2][3] == r and info[nb[3]][2][2] == r
    assert (cover == 1).all()
    loc = [_pencil_local(glob, off, nl) for off, nl, _ in info]
    # 1. y strips of the own planes; 2. whole z planes (with their y ghost rows)
    for r, (off, nl, nb) in enumerate(info):
        ny, nz = nl[1], nl[2]
        loc[r][2:nz + 2, :, 0:2] = loc[nb[0]][2:nz + 2, :, ny:ny + 2]
        loc[r][2:nz + 2, :, ny + 2:ny + 4] = loc[nb[1]][2:nz + 2, :, 2:4]
    for r, (off, nl, nb) in enumerate(info):
        nz = nl[2]
        loc[r][0:2] = loc[nb[2]][nz:nz + 2]
        loc[r][nz + 2:nz + 4] = loc[nb[3]][2:4]
    for r, (off, nl, _) in enumerate(info):
        assert np.array_equal(loc[r], _pencil_want(glob, off, nl, n)), f"rank {r}: ghosts (edges included) wrong"
    # the other order (z planes first) leaves the edge ghosts unset: the order is what the test pins
    loc = [_pencil_local(glob, off, nl) for off, nl, _ in info]
    for r, (off, nl, nb) in enumerate(info):
        nz = nl[2]
        loc[r][0:2] = loc[nb[2]][nz:nz + 2]
        loc[r][nz + 2:nz + 4] = loc[nb[3]][2:4]
    for r, (off, nl, nb) in enumerate(info):
        ny, nz = nl[1], nl[2]
        loc[r][2:nz + 2, :, 0:2] = loc[nb[0]][2:nz + 2, :, ny:ny + 2]
        loc[r][2:nz + 2, :, ny + 2:ny + 4] = loc[nb[1]][2:nz + 2, :, 2:4]
    assert any(np.isnan(loc[r]).any() for r in range(P))


def test_decompose_pencil_rejects_unsupported():
    from paper_2508_19911_b200.binding import CgksError, decompose_pencil
    with pytest.raises(CgksError):
        decompose_pencil((8, 10, 8), (1, 4, 1), 0)  # 10 rows not divisible by 4
    with pytest.raises(CgksError):
        decompose_pencil((8, 8, 8), (2, 2, 1), 0)  # x is never split
    with pytest.raises(CgksError):
        decompose_pencil((8, 8, 8), (1, 2, 2), 4)  # rank out of range


def _pencil_worker(rank, world, port, n, Py, Pz, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch

    from paper_2508_19911_b200.binding import decompose_pencil
    off, nl, nb = decompose_pencil(n, (1, Py, Pz), rank)
    rng = np.random.default_rng(13)
    glob = rng.standard_normal((n[2], 3, n[1], n[0]))
    loc = _pencil_local(glob, off, nl)
    ny, nz = nl[1], nl[2]

    def xchg(send_lo, send_hi, lo, hi):
        s = [torch.from_numpy(np.ascontiguousarray(send_lo)), torch.from_numpy(np.ascontiguousarray(send_hi))]
        rhi, rlo = torch.zeros_like(s[0]), torch.zeros_like(s[0])
        reqs = [dist.isend(s[0], lo), dist.isend(s[1], hi), dist.irecv(rhi, hi), dist.irecv(rlo, lo)]
        for q in reqs:
            q.wait()
        return rlo.numpy(), rhi.numpy()

    # the library's order: dense y strips of the own planes (send low, send high, receive high, receive low) ...
    rlo, rhi = xchg(loc[2:nz + 2, :, 2:4], loc[2:nz + 2, :, ny:ny + 2], nb[0], nb[1])
    loc[2:nz + 2, :, 0:2] = rlo
    loc[2:nz + 2, :, ny + 2:ny + 4] = rhi
    # ... then the contiguous 2-plane z blocks with their y ghost rows
    if Pz > 1:
        rlo, rhi = xchg(loc[2:4], loc[nz:nz + 2], nb[2], nb[3])
    else:
        rlo, rhi = loc[nz:nz + 2].copy(), loc[2:4].copy()  # periodic z of an undivided axis
    loc[0:2] = rlo
    loc[nz + 2:nz + 4] = rhi
    out[rank] = bool(np.array_equal(loc, _pencil_want(glob, off, nl, n)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("Py,Pz", [(2, 1), (2, 2)])
def test_pencil_halo_exchange_gloo(Py, Pz):
    world = Py * Pz
    n = (6, 4 * Py, 4 * Pz)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pencil_worker, args=(world, _free_port(), n, Py, Pz, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r], f"rank {r} ghosts wrong"
