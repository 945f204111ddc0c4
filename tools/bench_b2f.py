"""NEXT-1 measurement: elpa_trans_ev_band_to_full at a BASELINE size (synthetic stage-1
reflectors generated on the device), FP64 TFLOP/s of the exact flop count
sum_j 4 * (n - j - nbw) * nev against the measured DMMA peak.  Timing only: parity against the
oracle is tests/test_gpu_parity.py::test_band_to_full_vs_oracle (only tests/, smoke() and bench.py's
cpu_baseline leg may use oracle/)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import uniform_pm1_torch, synthetic_q_torch, config_seed

n, nbw, nev = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 64, 20000)))
seed = config_seed(3)
K = eb.b2f_count(n, nbw)
V = torch.zeros((K, n), dtype=torch.float64, device="cuda")
for j0 in range(0, K, 512):
    j1 = min(K, j0 + 512)
    cnt = torch.arange(j0 * n, j1 * n, dtype=torch.int64, device="cuda")
    V[j0:j1] = uniform_pm1_torch(seed ^ 0x77, cnt).reshape(j1 - j0, n)
rows = torch.arange(n, device="cuda")[None, :]
start = (torch.arange(K, device="cuda") + nbw)[:, None]
V = torch.where(rows < start, torch.zeros_like(V), V)
V[torch.arange(K), torch.arange(K) + nbw] = 1.0
tau = 2.0 / (V * V).sum(dim=1)
Q = synthetic_q_torch(n, 0, nev, seed, device="cuda")
flops = sum(4.0 * (n - j - nbw) * nev for j in range(K))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    eb.trans_ev_band_to_full(n, nbw, V, tau, Q)
torch.cuda.synchronize()
times = []
for _ in range(3):
    e0.record(); eb.trans_ev_band_to_full(n, nbw, V, tau, Q); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = min(times)
print(json.dumps(dict(path="trans_ev_band_to_full", n=n, nbw=nbw, nev=nev, K=K, ms=ms, tflops=flops / ms / 1e9,
                      frac_of_dmma_peak=flops / ms / 1e9 / 36.983, times=times)))
