"""Timing sweep of DMMA kernel shapes per config (development tool, not the bench)."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors, synthetic_q_torch

import os
SHAPES = [tuple(int(v) for v in t.split(',')) for t in os.environ['SHAPES'].split()] if os.environ.get('SHAPES') else [(1,2,4,1), (2,2,4,1), (4,2,4,1), (8,1,4,1), (2,4,2,1), (2,2,3,1), (2,2,2,1), (4,4,2,1), (2,4,3,1), (2,1,2,1), (1,2,2,1), (4,2,2,1), (2,1,4,1), (1,1,4,1), (1,1,2,1), (1,4,2,1), (2,1,3,1)]
REPS = int(os.environ.get('REPS', '2'))
cfgs = [(20000, 64, 20000), (20000, 64, 2000), (4096, 32, 4096), (20000, 64, 2500), (60000, 64, 3750)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in a.split(',')) for a in sys.argv[1:]]
for (n, nbw, nev) in cfgs:
    R = eb.hh_count(n, nbw)
    hv, tau = synthetic_reflectors(R, nbw, 1)
    dv, dt = torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda()
    del hv, tau
    ws = torch.empty(eb.workspace_bytes(n, nbw), dtype=torch.uint8, device='cuda')
    dq = synthetic_q_torch(n, 0, nev, 2, device='cuda')
    eb.prepare(n, nbw, dv, dt, ws)
    fl = eb.credited_flops(n, nbw, nev)
    for sh in [None] + SHAPES:
        for grid in ([0] if sh is None else [int(g) for g in os.environ.get('GRIDS', '0').split()]):
            opts = None if sh is None else dict(kernel=int(os.environ.get('KERNEL', '2')), depth_warps=sh[0], col_warps=sh[1], tiles_per_warp=sh[2], grid_ctas=grid, groups_per_step=sh[3])
            try:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                eb.apply_prepared(n, nbw, ws, dq, opts=opts); torch.cuda.synchronize()
                best = 1e30
                for _ in range(REPS):
                    e0.record(); eb.apply_prepared(n, nbw, ws, dq, opts=opts); e1.record(); torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                print(json.dumps(dict(n=n, nbw=nbw, nev=nev, shape=sh, grid=grid, ms=round(best, 3), tflops=round(fl / best / 1e9, 3),
                                      desc=eb.describe(n, nbw, nev, opts)[1])), flush=True)
            except Exception as ex:
                print(json.dumps(dict(n=n, nbw=nbw, nev=nev, shape=sh, error=str(ex))), flush=True)
    del dv, dt, ws, dq
    torch.cuda.empty_cache()
