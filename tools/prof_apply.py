"""One DMMA apply (prepared once) for an ncu capture (development tool).
usage: python tools/prof_apply.py n nbw nev [D CW NCT [K]]"""
import sys; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch
n, nbw, nev = (int(a) for a in sys.argv[1:4])
opts = None
if len(sys.argv) > 6:
    D, CW, NCT = (int(a) for a in sys.argv[4:7])
    K = int(sys.argv[7]) if len(sys.argv) > 7 else 1
    opts = dict(kernel=eb.KERNEL_DMMA, depth_warps=D, col_warps=CW, tiles_per_warp=NCT, groups_per_step=K)
R = eb.hh_count(n, nbw)
dv, dt = synthetic_reflectors_torch(R, nbw, 2, device='cuda')
dq = synthetic_q_torch(n, 0, nev, 3, device='cuda')
ws = torch.empty(eb.workspace_bytes(n, nbw), dtype=torch.uint8, device='cuda')
eb.prepare(n, nbw, dv, dt, ws)
eb.apply_prepared(n, nbw, ws, dq, opts=opts)
torch.cuda.synchronize()
