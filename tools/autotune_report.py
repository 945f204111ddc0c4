"""NEXT-2 evidence: run the MEDIUM autotuning loop (elpa_b200_autotune_run_dtype) for the FP64,
FP32 and complex paths at the BASELINE shapes and print each best choice (development tool)."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch, synthetic_reflectors_c, synthetic_q_c_np

cases = [("f64", 20000, 64, 20000), ("f64", 20000, 64, 2000), ("f64", 4096, 32, 4096),
         ("f32", 20000, 64, 20000), ("f32", 20000, 64, 2000), ("c64", 20000, 64, 2000), ("c64", 4096, 32, 4096)]
for dt, n, nbw, nev in cases:
    R = eb.hh_count(n, nbw)
    if dt == "c64":
        hv, tau = synthetic_reflectors_c(R, nbw, 1)
        dv, dtau = torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda()
        Q = torch.empty((nev, n), dtype=torch.complex128, device="cuda")
        for a in range(0, nev, 2000):
            Q[a:a + 2000] = torch.from_numpy(synthetic_q_c_np(n, a, min(nev, a + 2000), 2)).cuda()
    else:
        dv, dtau = synthetic_reflectors_torch(R, nbw, 1, device="cuda")
        Q = synthetic_q_torch(n, 0, nev, 2, device="cuda")
        if dt == "f32":
            dv, dtau, Q = dv.float(), dtau.float(), Q.float()
    t0 = time.time()
    best, ms = eb.autotune(n, nbw, dv, dtau, Q, level=eb.AUTOTUNE_MEDIUM, reps=2)
    flops = eb.credited_flops(n, nbw, nev) * (4 if dt == "c64" else 1)
    print(json.dumps(dict(dtype=dt, n=n, nbw=nbw, nev=nev, best=best, best_ms=round(ms, 3),
                          best_tflops=round(flops / ms / 1e9, 2), tuning_s=round(time.time() - t0, 1))), flush=True)
    del dv, dtau, Q
    torch.cuda.empty_cache()
