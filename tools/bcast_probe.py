"""NCCL broadcast bandwidth probe (development): times dist.broadcast of the C3/C5 packed
reflector sizes with CUDA events, max over ranks; one JSON line per size from rank 0."""
import json, os, sys
import torch
import torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=dev)
for nbytes in (1_630_000_000, 203_000_000, 14_640_000_000):
    x = torch.ones(nbytes // 8, dtype=torch.float64, device=dev)
    for _ in range(3):
        dist.broadcast(x, src=0)
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        dist.broadcast(x, src=0)
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps(dict(world=world, bytes=nbytes, ms=float(t.item()), GBps=nbytes / float(t.item()) / 1e6)), flush=True)
    del x
    torch.cuda.empty_cache()
dist.destroy_process_group()
