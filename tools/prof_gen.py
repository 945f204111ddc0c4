"""One generalized back-transformation at n = nev = 20000 for an ncu launch list (development tool)."""
import sys; sys.path.insert(0, '.')
import torch
import paper_1811_01277_b200 as eb
from inputs import lower_triangular_cm_torch, synthetic_q_torch
n, nev = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (20000, 20000)))
dL = lower_triangular_cm_torch(n, 0, n, 5, device="cuda")
dq = synthetic_q_torch(n, 0, nev, 6, device="cuda")
torch.cuda.synchronize()
eb.generalized_back_transform(n, dL, dq)
torch.cuda.synchronize()
