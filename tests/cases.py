"""Disk cache of real-chase oracle cases (the chase and the tridiagonal eigensolve
are the slow part of the oracle, so a case is computed once per box and reused).  Test
infrastructure: it only stores what oracle.make_case returns; nothing here computes.

Cache directory: $ELPA_B200_CASE_CACHE, else /tmp/elpa_b200_cases (per box: a fresh gpurun
box recomputes, a second test in the same session reuses)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle

CACHE = os.environ.get("ELPA_B200_CASE_CACHE", "/tmp/elpa_b200_cases")
_KEYS = ("band", "hh_v", "hh_tau", "s", "L", "d", "e", "lam", "Qin", "Qref")


def real_case(n, nbw, nev, seed):
    """oracle.make_case(n, nbw, nev, seed), cached as an .npz keyed by its arguments."""
    path = os.path.join(CACHE, f"case_n{n}_b{nbw}_k{nev}_s{seed}.npz")
    if os.path.exists(path):
        z = np.load(path)
        case = {k: z[k] for k in _KEYS}
        case.update(n=n, nbw=nbw, nev=nev, seed=seed, secs=0.0)
        return case
    case = oracle.make_case(n, nbw, nev, seed)
    os.makedirs(CACHE, exist_ok=True)
    tmp = path + ".tmp.npz"
    np.savez(tmp, **{k: case[k] for k in _KEYS})
    os.replace(tmp, path)
    return case


def residual_parallel(band, Q, lam, chunk=256, workers=None):
    """oracle.residual over column chunks on host threads (numpy releases the GIL): the squared
    Frobenius numerators add over columns and the denominator n ||B||_F is shared, so
    sqrt(sum_chunks r_chunk^2) is exactly the full residual."""
    nev = Q.shape[0]
    chunks = [(c, min(nev, c + chunk)) for c in range(0, nev, chunk)]
    with ThreadPoolExecutor(workers or os.cpu_count() or 1) as ex:
        parts = list(ex.map(lambda cc: oracle.residual(band, Q[cc[0]:cc[1]], lam[cc[0]:cc[1]]), chunks))
    return float(np.sqrt(np.sum(np.square(parts))))
