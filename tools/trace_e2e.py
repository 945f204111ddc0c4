"""Stage timeline of the host-buffer entry point (elpa_trans_ev_tridi_to_band_host) at C3 with
ELPA_B200_TRACE=1: prints the library's trace line (ms after buffer allocation) and the wall
time of the call.  Development tool for the e2e path."""
import os, sys, time
os.environ["ELPA_B200_TRACE"] = "1"
import torch
sys.path.insert(0, '.')
import paper_1811_01277_b200 as eb
from inputs import synthetic_reflectors_torch, synthetic_q_torch, CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n, nbw, nev = CONFIGS[cfg]
R = eb.hh_count(n, nbw)
dv, dt = synthetic_reflectors_torch(R, nbw, 1, device="cuda")
hv, ht = dv.cpu().pin_memory(), dt.cpu().pin_memory()
del dv, dt
Qh = synthetic_q_torch(n, 0, nev, 2, device="cuda").cpu().pin_memory()
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    eb.trans_ev_tridi_to_band_host(n, nbw, hv, ht, Qh)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms wall, "
          f"{4.0 * nbw * nev * R / (time.perf_counter() - t0) / 1e12:.2f} TF/s", file=sys.stderr, flush=True)
