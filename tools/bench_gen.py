"""NEXT-4 timing: elpa_generalized_back_transform (V = L^-T Vtilde) at C3/C4 sizes, CUDA
events; flops credited n^2 * nev (the triangular solve)."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import lower_triangular_cm_torch, synthetic_q_torch

for (n, nev) in [(20000, 20000), (20000, 2000), (4096, 4096)]:
    dL = lower_triangular_cm_torch(n, 0, n, 5, device="cuda")
    dq = synthetic_q_torch(n, 0, nev, 6, device="cuda")
    eb.generalized_back_transform(n, dL, dq); torch.cuda.synchronize()
    times = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eb.generalized_back_transform(n, dL, dq); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = min(times)
    print(json.dumps(dict(path="generalized_back_transform", n=n, nev=nev, ms=ms, tflops=n * n * nev / ms / 1e9,
                          frac_of_dmma_peak=n * n * nev / ms / 1e9 / 36.983, times=times)), flush=True)
    del dL, dq
    torch.cuda.empty_cache()
