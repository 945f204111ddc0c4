"""Timeline probe of the multi-GPU preamble at C3 (development): broadcast alone (1 and C
chunks), preparation alone (whole and chunked), and the chunked pipeline; CUDA events on the
compute stream, max over ranks; rank 0 prints one JSON line per variant."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import torch.distributed as dist
import paper_1811_01277_b200 as eb
from paper_1811_01277_b200.dist import broadcast_chunks, broadcast_and_prepare, sweep_chunks, unpack_reflectors
from inputs import synthetic_reflectors_torch
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
n, nbw = 20000, 64
R = eb.hh_count(n, nbw)
hh = torch.empty(R * (nbw + 1), dtype=torch.float64, device=dev)
hv, tau = synthetic_reflectors_torch(R, nbw, 3, device=dev)
hh[:R * nbw].copy_(hv.reshape(-1)); hh[R * nbw:].copy_(tau)
del hv, tau
ws = torch.empty(eb.workspace_bytes(n, nbw), dtype=torch.uint8, device=dev)
hh_v, hh_tau = unpack_reflectors(hh, R, nbw)
s = torch.cuda.current_stream(dev)
C = int(os.environ.get("CHUNKS", "8"))

def bcast(c):
    for _, _, w in broadcast_chunks(n, nbw, hh, R, chunks=c):
        for x in w:
            x.wait()

def prep_chunks(c):
    b = sweep_chunks(n, nbw, c)
    for j0, j1 in zip(b[:-1], b[1:]):
        eb.prepare_sweeps(n, nbw, hh_v, hh_tau, ws, j0, j1)

variants = {"bcast_1": lambda: bcast(1), f"bcast_{C}": lambda: bcast(C), "prep_1": lambda: eb.prepare(n, nbw, hh_v, hh_tau, ws),
            f"prep_{C}": lambda: prep_chunks(C), f"pipeline_{C}": lambda: broadcast_and_prepare(n, nbw, hh, R, ws, chunks=C),
            "bcast_then_prep": lambda: (bcast(1), eb.prepare(n, nbw, hh_v, hh_tau, ws))}
for name, f in variants.items():
    for _ in range(2):
        f()
    torch.cuda.synchronize(); dist.barrier(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(s)
    for _ in range(reps):
        f()
    e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps(dict(world=world, variant=name, ms=round(float(t.item()), 3))), flush=True)
dist.destroy_process_group()
