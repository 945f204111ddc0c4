"""One FP32 call at the given size for an ncu capture (development tool).
usage: python tools/prof_f32.py n nbw nev [D CW NC K]"""
import sys; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch
n, nbw, nev = (int(a) for a in sys.argv[1:4])
opts = None
if len(sys.argv) > 7:
    D, CW, NC, K = (int(a) for a in sys.argv[4:8])
    opts = dict(kernel=eb.KERNEL_FFMA2, depth_warps=D, col_warps=CW, tiles_per_warp=NC, groups_per_step=K)
R = eb.hh_count(n, nbw)
dv, dt = synthetic_reflectors_torch(R, nbw, 1, device='cuda')
dv, dt = dv.float(), dt.float()
dq = synthetic_q_torch(n, 0, nev, 2, device='cuda').float()
eb.trans_ev_tridi_to_band(n, nbw, dv, dt, dq, opts=opts)
torch.cuda.synchronize()
