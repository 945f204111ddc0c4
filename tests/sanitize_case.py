"""Small cases for compute-sanitizer runs (memcheck / racecheck / synccheck), one process; kept under
tests/ because it checks results against the oracle.  Not collected by pytest (no test_ prefix)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
import oracle
from inputs import synthetic_reflectors, synthetic_q_np

def run(n, nbw, nev, opts):
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors(len(s), nbw, 3)
    Q = synthetic_q_np(n, 0, nev, 3, ldq=n + (n & 1))
    want = oracle.apply(hv, tau, s, L, Q)
    dq = torch.from_numpy(Q).cuda()
    eb.trans_ev_tridi_to_band(n, nbw, torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda(), dq, opts=opts)
    torch.cuda.synchronize()
    err = np.abs(dq.cpu().numpy() - want).max() / np.abs(want).max()
    print(n, nbw, nev, opts, "err", err, flush=True)
    assert err < 1e-12

for opts in [None, dict(kernel=2, depth_warps=2, col_warps=2, tiles_per_warp=2, grid_ctas=3),
             dict(kernel=2, depth_warps=4, col_warps=2, tiles_per_warp=4, grid_ctas=2),
             dict(kernel=2, depth_warps=1, col_warps=2, tiles_per_warp=4), dict(kernel=3), dict(kernel=1)]:
    run(301, 64, 45, opts)
    run(200, 16, 33, opts)
print("sanitize cases ok")
