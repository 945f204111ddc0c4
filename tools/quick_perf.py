"""Quick timing sweep of the DMMA kernel configs (development tool, not the bench)."""
import itertools, json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors, synthetic_q_torch, config_seed

def bench(n, nbw, nev, opts, reps=3):
    R = eb.hh_count(n, nbw)
    hv, tau = synthetic_reflectors(R, nbw, 1)
    dv, dt = torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda()
    ws = torch.empty(eb.workspace_bytes(n, nbw, opts), dtype=torch.uint8, device='cuda')
    dq = synthetic_q_torch(n, 0, nev, 2, device='cuda')
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    eb.prepare(n, nbw, dv, dt, ws, opts=opts)
    eb.apply_prepared(n, nbw, ws, dq, opts=opts)
    torch.cuda.synchronize()
    best = 1e30; tprep = 0
    for _ in range(reps):
        e0.record(); eb.prepare(n, nbw, dv, dt, ws, opts=opts); e1.record()
        eb.apply_prepared(n, nbw, ws, dq, opts=opts); e2.record(); torch.cuda.synchronize()
        best = min(best, e1.elapsed_time(e2)); tprep = e0.elapsed_time(e1)
    fl = eb.credited_flops(n, nbw, nev)
    return best, tprep, fl / best / 1e9

cfgs = [(20000, 64, 20000), (20000, 64, 2000), (4096, 32, 4096)]
shapes = [(1,8,2), (2,4,2), (2,2,4), (4,2,2), (4,2,4), (4,1,4), (8,1,2), (8,1,4), (4,4,1), (8,2,1)]
for (n, nbw, nev) in cfgs:
    for sh in [None] + shapes:
        opts = None if sh is None else dict(kernel=2, depth_warps=sh[0], col_warps=sh[1], tiles_per_warp=sh[2])
        try:
            ms, tp, tf = bench(n, nbw, nev, opts, reps=2 if n == 20000 and nev == 20000 else 3)
            print(json.dumps(dict(n=n, nbw=nbw, nev=nev, shape=sh, desc=eb.describe(n, nbw, nev, opts)[1], ms=round(ms, 3), prep_ms=round(tp, 3), tflops=round(tf, 3))), flush=True)
        except Exception as e:
            print(json.dumps(dict(n=n, nbw=nbw, nev=nev, shape=sh, error=str(e))), flush=True)
