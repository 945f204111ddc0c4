"""One C3 preparation (prep_dmma_kernel) for an ncu capture (development tool)."""
import sys; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch
n, nbw = 20000, 64
R = eb.hh_count(n, nbw)
dv, dt = synthetic_reflectors_torch(R, nbw, 2, device='cuda')
ws = torch.empty(eb.workspace_bytes(n, nbw), dtype=torch.uint8, device='cuda')
eb.prepare(n, nbw, dv, dt, ws)
torch.cuda.synchronize()
