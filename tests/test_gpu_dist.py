"""Multi-GPU path on real GPUs, world size 2 over NCCL: the broadcast delivers the
reflectors, apply_sharded on a NON-default stream waits for it (torch's NCCL
collectives only order the current stream), and the shards equal the oracle's columns.
Needs two GPUs (gpurun --gpus 2); skipped on a one-GPU box."""
import os
import socket

import numpy as np
import pytest

import oracle
from inputs import synthetic_reflectors, synthetic_q_np

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nbw, nev, seed, outdir, use_ws):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1811_01277_b200 as eb
    from paper_1811_01277_b200.dist import shard_range, pack_reflectors, apply_sharded
    R = eb.hh_count(n, nbw)
    if rank == 0:
        hv, tau = synthetic_reflectors(R, nbw, seed)
        packed = pack_reflectors(torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda())
    else:
        packed = torch.full((R * (nbw + 1),), float("nan"), dtype=torch.float64, device="cuda")
    c0, c1 = shard_range(nev, rank, world)
    Q = torch.from_numpy(synthetic_q_np(n, c0, c1, seed)).cuda()
    side = torch.cuda.Stream()
    ws = torch.empty(eb.workspace_bytes(n, nbw), dtype=torch.uint8, device="cuda") if use_ws else None
    torch.cuda.synchronize()
    # delay the broadcast's source on rank 0 (its NCCL stream waits for `side`), so a receiving
    # rank whose apply did not wait for the broadcast would read the NaN-filled buffer
    if rank == 0:
        with torch.cuda.stream(side):
            torch.cuda._sleep(50_000_000)
    apply_sharded(n, nbw, packed, R, Q, src=0, stream=side, workspace=ws)
    side.synchronize()
    np.save(os.path.join(outdir, f"shard{rank}_{int(use_ws)}.npy"), Q.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("use_ws", [False, True])
def test_nccl_world2_side_stream(tmp_path, use_ws):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    n, nbw, nev, seed, world = 700, 32, 90, 123, 2
    mp.start_processes(_worker, args=(world, _free_port(), n, nbw, nev, seed, str(tmp_path), use_ws),
                       nprocs=world, join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"shard{r}_{int(use_ws)}.npy") for r in range(world)])
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors(len(s), nbw, seed)
    want = oracle.apply(hv, tau, s, L, synthetic_q_np(n, 0, nev, seed))
    assert np.isfinite(got).all()
    assert float(np.abs(got - want).max() / np.abs(want).max()) <= 1e-12
