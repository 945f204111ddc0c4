"""Host logic of the multi-GPU path on CPU: world size 2 over gloo (127.0.0.1).  The single
broadcast delivers identical reflectors, the column shards tile [0, nev), and per-shard
application (the oracle stands in for the GPU here) concatenates bitwise to the 1-rank
result — the invariant the NCCL/GPU path relies on."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from inputs import synthetic_reflectors, synthetic_q_np


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nbw, nev, seed, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1811_01277_b200.dist import shard_range, pack_reflectors, unpack_reflectors, broadcast_reflectors
    s, L = oracle.schedule(n, nbw)
    R = len(s)
    if rank == 0:
        hv, tau = synthetic_reflectors(R, nbw, seed)
        packed = pack_reflectors(torch.from_numpy(hv), torch.from_numpy(tau))
    else:
        packed = torch.full((R * (nbw + 1),), float("nan"), dtype=torch.float64)
    broadcast_reflectors(packed, src=0)
    hv_r, tau_r = unpack_reflectors(packed, R, nbw)
    c0, c1 = shard_range(nev, rank, world)
    Ql = synthetic_q_np(n, c0, c1, seed)
    out = oracle.apply(hv_r.numpy(), tau_r.numpy(), s, L, Ql, nthreads=1)
    np.save(os.path.join(outdir, f"shard{rank}.npy"), out)
    np.save(os.path.join(outdir, f"hh{rank}.npy"), packed.numpy())
    dist.destroy_process_group()


def test_shard_range_tiles_columns():
    from paper_1811_01277_b200.dist import shard_range
    for nev in (0, 1, 7, 20000, 30000):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(nev, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nev
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_gloo_world2_broadcast_and_shards(tmp_path):
    n, nbw, nev, seed = 160, 16, 21, 77
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), n, nbw, nev, seed, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    h0, h1 = np.load(tmp_path / "hh0.npy"), np.load(tmp_path / "hh1.npy")
    assert np.array_equal(h0, h1)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors(len(s), nbw, seed)
    want = oracle.apply(hv, tau, s, L, synthetic_q_np(n, 0, nev, seed), nthreads=4)
    assert np.array_equal(got, want)


def test_sweep_chunks_cover_and_balance():
    """The broadcast's sweep ranges tile [0, n-2], are strictly increasing, and hold about R/C
    reflectors each (the last sweeps are short: a range may hold a few more sweeps)."""
    import paper_1811_01277_b200 as eb
    from paper_1811_01277_b200.dist import sweep_chunks
    for (n, nbw, C) in [(20000, 64, 8), (4096, 32, 8), (300, 16, 3), (50, 8, 8), (5, 2, 4)]:
        b = sweep_chunks(n, nbw, C)
        assert b[0] == 0 and b[-1] == n - 2
        assert all(x < y for x, y in zip(b[:-1], b[1:]))
        R = eb.hh_count(n, nbw)
        offs = [eb.hh_offset(n, nbw, j) for j in b]
        assert offs[0] == 0 and offs[-1] == R
        sizes = [y - x for x, y in zip(offs[:-1], offs[1:])]
        assert max(sizes) <= R // C + 2 * (n // nbw + 2), sizes
    n, b = 300, 16
    for j in (0, 1, 17, 200, 297, 298):                # off(j) = reflectors of the sweeps before j
        before = sum(len(range(jj + 1, n - 1, b)) for jj in range(min(j, n - 2)))
        assert eb.hh_offset(n, b, j) == before
    assert eb.hh_offset(n, b, n - 2) == oracle.count(n, b)


def _chunk_worker(rank, world, port, n, nbw, seed, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1811_01277_b200 as eb
    from paper_1811_01277_b200.dist import pack_reflectors, broadcast_chunks
    R = eb.hh_count(n, nbw)
    if rank == 0:
        hv, tau = synthetic_reflectors(R, nbw, seed)
        packed = pack_reflectors(torch.from_numpy(hv), torch.from_numpy(tau))
    else:
        packed = torch.full((R * (nbw + 1),), float("nan"), dtype=torch.float64)
    for j0, j1, works in broadcast_chunks(n, nbw, packed, R, src=0, chunks=5):
        for w in works:
            w.wait()
    np.save(os.path.join(outdir, f"chunked{rank}.npy"), packed.numpy())
    dist.destroy_process_group()


def test_gloo_world2_chunked_broadcast(tmp_path):
    """The chunked broadcast delivers exactly the source's packed reflectors (every row and tau
    of every sweep range, nothing else)."""
    n, nbw, seed, world = 301, 16, 5, 2
    mp.start_processes(_chunk_worker, args=(world, _free_port(), n, nbw, seed, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    a, b = np.load(tmp_path / "chunked0.npy"), np.load(tmp_path / "chunked1.npy")
    assert np.array_equal(a, b) and np.isfinite(b).all()
