"""DFMA kernel timing probe (development): apply-only time; grid 1 = serial items."""
import sys, os, json; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch
for (n, nbw, nev, kf, grid, kern) in [(4000, 64, 64, 8, 1, 3), (4000, 64, 64, 8, 0, 3), (4000, 64, 64, 8, 1, 2), (4000, 64, 64, 8, 0, 2),
                                      (4000, 32, 64, 8, 1, 3), (4000, 32, 64, 8, 0, 3)]:
    R = eb.hh_count(n, nbw)
    dv, dt = synthetic_reflectors_torch(R, nbw, 2, device='cuda')
    dq = synthetic_q_torch(n, 0, nev, 3, device='cuda')
    opts = dict(kernel=kern, fused_k=kf if kern == 3 else 0, grid_ctas=grid)
    ws = torch.empty(eb.workspace_bytes(n, nbw, opts), dtype=torch.uint8, device='cuda')
    eb.prepare(n, nbw, dv, dt, ws, opts=opts)
    eb.apply_prepared(n, nbw, ws, dq, opts=opts); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eb.apply_prepared(n, nbw, ws, dq, opts=opts); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps(dict(n=n, nbw=nbw, nev=nev, kf=kf, grid=grid, kernel=kern, pub=os.environ.get('ELPA_B200_PUB'), ms=round(ms, 3),
                          tflops=round(eb.credited_flops(n, nbw, nev) / ms / 1e9, 3), desc=eb.describe(n, nbw, nev, opts)[1])), flush=True)
