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
