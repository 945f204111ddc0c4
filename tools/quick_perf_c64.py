"""Timing sweep of the complex variant's shapes (NEXT-3; development tool).  Whole call (prep +
apply); credited flops 16*nbw*nev per reflector (4x the real count: a complex multiply-add is
4 real ones)."""
import json, os, sys
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_c, synthetic_q_c_np

SHAPES = [tuple(int(v) for v in t.split(',')) for t in os.environ['SHAPES'].split()] if os.environ.get('SHAPES') else \
    [(1, 2, 2), (2, 2, 1), (1, 2, 1), (2, 1, 2), (1, 4, 1), (2, 2, 2), (1, 1, 2)]
REPS = int(os.environ.get('REPS', '2'))
cfgs = [(20000, 64, 20000), (20000, 64, 2000), (4096, 32, 4096)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(v) for v in a.split(',')) for a in sys.argv[1:]]
for (n, nbw, nev) in cfgs:
    R = eb.hh_count(n, nbw)
    hv, tau = synthetic_reflectors_c(R, nbw, 1)
    dv, dt = torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda()
    del hv, tau
    dq = torch.empty((nev, n), dtype=torch.complex128, device='cuda')
    for a in range(0, nev, 2000):
        dq[a:a + 2000] = torch.from_numpy(synthetic_q_c_np(n, a, min(nev, a + 2000), 2)).cuda()
    fl = 4 * eb.credited_flops(n, nbw, nev)
    for sh in [None] + SHAPES:
        opts = None if sh is None else dict(kernel=eb.KERNEL_DMMA, depth_warps=sh[0], col_warps=sh[1], tiles_per_warp=sh[2],
                                            groups_per_step=sh[3] if len(sh) > 3 else 1)
        try:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eb.trans_ev_tridi_to_band(n, nbw, dv, dt, dq, opts=opts); torch.cuda.synchronize()
            best = 1e30
            for _ in range(REPS):
                e0.record(); eb.trans_ev_tridi_to_band(n, nbw, dv, dt, dq, opts=opts); e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(json.dumps(dict(dtype="c64", n=n, nbw=nbw, nev=nev, shape=sh, ms=round(best, 3),
                                  tflops=round(fl / best / 1e9, 3), desc=eb.describe_c64(n, nbw, nev, opts)[1])), flush=True)
        except Exception as ex:
            print(json.dumps(dict(n=n, nbw=nbw, nev=nev, shape=sh, error=str(ex))), flush=True)
    del dv, dt, dq
    torch.cuda.empty_cache()
