"""The k-blocking sweep of the FP64 CUDA-core (DFMA) kernel against the tensor-core (DMMA)
kernel (north_star item 3; BASELINE config 2 "k=2/4/6 reflector-blocking sweep"): for each
config, the apply kernel alone (reflectors prepared once per kernel) timed with CUDA events,
best of REPS, credited flops 4*nbw*nev per reflector.  Development tool; one JSON line per
(config, kernel, k).  usage: python tools/dfma_sweep.py [n,nbw,nev ...]"""
import json, os, sys
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch

REPS = int(os.environ.get('REPS', '3'))
cfgs = [(4096, 32, 4096), (20000, 64, 20000), (20000, 64, 2000)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in a.split(',')) for a in sys.argv[1:]]
variants = [("dmma", None)] + [("dfma", kf) for kf in (2, 4, 6, 8)]
for (n, nbw, nev) in cfgs:
    R = eb.hh_count(n, nbw)
    dv, dt = synthetic_reflectors_torch(R, nbw, 2, device='cuda')
    dq = synthetic_q_torch(n, 0, nev, 3, device='cuda')
    fl = eb.credited_flops(n, nbw, nev)
    for name, kf in variants:
        opts = dict(kernel=eb.KERNEL_DMMA) if kf is None else dict(kernel=eb.KERNEL_DFMA, fused_k=kf)
        try:
            ws = torch.empty(eb.workspace_bytes(n, nbw, opts), dtype=torch.uint8, device='cuda')
            eb.prepare(n, nbw, dv, dt, ws, opts=opts)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eb.apply_prepared(n, nbw, ws, dq, opts=opts)
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(REPS):
                e0.record(); eb.apply_prepared(n, nbw, ws, dq, opts=opts); e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            tf = fl / best / 1e9
            print(json.dumps(dict(n=n, nbw=nbw, nev=nev, kernel=name, k=kf or 8, ms=round(best, 3), tflops=round(tf, 3),
                                  frac_fp64_peak=round(tf / 36.98, 4), desc=eb.describe(n, nbw, nev, opts)[1])), flush=True)
            del ws
        except Exception as ex:
            print(json.dumps(dict(n=n, nbw=nbw, nev=nev, kernel=name, k=kf, error=str(ex))), flush=True)
    del dv, dt, dq
    torch.cuda.empty_cache()
