"""One DFMA-kernel apply at C2 (n=4096, nbw=32) for an ncu capture (development tool)."""
import sys; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch
n, nbw, nev, kf = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 32, 4096, 8)))
R = eb.hh_count(n, nbw)
dv, dt = synthetic_reflectors_torch(R, nbw, 2, device='cuda')
dq = synthetic_q_torch(n, 0, nev, 3, device='cuda')
opts = dict(kernel=eb.KERNEL_DFMA, fused_k=kf)
ws = torch.empty(eb.workspace_bytes(n, nbw, opts), dtype=torch.uint8, device='cuda')
eb.prepare(n, nbw, dv, dt, ws, opts=opts)
eb.apply_prepared(n, nbw, ws, dq, opts=opts)
torch.cuda.synchronize()
