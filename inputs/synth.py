"""Counter-based splitmix64 generators ("seeded
splitmix-style generator").

Element t of stream `seed` is splitmix64(seed + (t+1)*GAMMA) — a pure function of
(seed, t), so any sub-block of any input (a column range of Q, a sampled column) can be
regenerated independently on host (numpy) or device (torch) with identical bits.

u = (z >> 11) * 2^-53 in [0, 1);  a = 2u - 1 in [-1, 1).
"""
import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_TWO53 = float(2 ** -53)

# Stream tags: independent streams for the different inputs of one config seed.
TAG_BAND = 0x0
TAG_HHV = 0x5F1A2B3C4D5E6F70
TAG_Q = 0x2A7B9C1D3E5F7081

# BASELINE.json configs: name -> (n, nbw, nev); seeds S_i = 1811012770 + i
CONFIGS = {
    "C1": (512, 16, 512),
    "C2": (4096, 32, 4096),
    "C3": (20000, 64, 20000),
    "C4": (20000, 64, 2000),
    "C5": (60000, 64, 30000),
}


def config_seed(i):
    return 1811012770 + int(i)


def splitmix64_np(seed, counters):
    """splitmix64 output for counters (uint64 array)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (counters.astype(np.uint64) + np.uint64(1)) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1_np(seed, counters):
    z = splitmix64_np(seed, counters)
    u = (z >> np.uint64(11)).astype(np.float64) * _TWO53
    return 2.0 * u - 1.0


def _s64(x):
    x &= 0xFFFFFFFFFFFFFFFF
    return x - (1 << 64) if x >= (1 << 63) else x


def uniform_pm1_torch(seed, counters):
    """Same stream as uniform_pm1_np, computed with torch int64 (wrapping) arithmetic.
    `counters` is an int64 torch tensor (any device)."""
    import torch
    def lsr(z, k):  # logical shift right on int64
        return (z >> k) & ((1 << (64 - k)) - 1)
    z = (counters + 1) * _s64(GAMMA) + _s64(seed)
    z = (z ^ lsr(z, 30)) * _s64(_M1)
    z = (z ^ lsr(z, 27)) * _s64(_M2)
    z = z ^ lsr(z, 31)
    u = lsr(z, 11).to(torch.float64) * _TWO53
    return 2.0 * u - 1.0


def band_matrix(n, nbw, seed):
    """Random symmetric band matrix, entries i.i.d. uniform [-1,1).

    Returns LAPACK-style lower band storage `band` of shape (nbw+1, n):
    band[d, c] = B[c+d, c] for c+d < n (zero otherwise).  Draw order: c ascending, then
    d ascending, skipping c+d >= n without drawing (one draw per stored entry)."""
    n, nbw = int(n), int(nbw)
    band = np.zeros((nbw + 1, n), dtype=np.float64)
    if n == 0:
        return band
    cnt = np.minimum(nbw + 1, n - np.arange(n))            # entries drawn in column c
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    c_idx = np.repeat(np.arange(n), cnt)
    d_idx = np.arange(cnt.sum()) - np.repeat(off, cnt)
    vals = uniform_pm1_np(seed ^ TAG_BAND, np.arange(cnt.sum(), dtype=np.uint64))
    band[d_idx, c_idx] = vals
    return band


TAG_DENSE = 0x3C4D5E6F708192A3


def dense_symmetric(n, seed):
    """Random dense symmetric n x n matrix, entries uniform [-1,1) drawn for the lower triangle
    column by column (c ascending, then row r >= c ascending), mirrored."""
    n = int(n)
    rows, cols = np.tril_indices(n)
    order = np.lexsort((rows, cols))                 # column-major order of the lower triangle
    vals = uniform_pm1_np(seed ^ TAG_DENSE, np.arange(len(order), dtype=np.uint64))
    A = np.zeros((n, n))
    A[rows[order], cols[order]] = vals
    A = A + np.tril(A, -1).T
    return A


def synthetic_reflectors(R, nbw, seed):
    """Synthetic Householder reflectors for timing / sampled parity at sizes where the
    oracle's chase is too slow: v[0] = 1, v[1:] uniform [-1,1),
    tau = 2/||v||^2 over the full nbw entries (so every truncated reflector is a
    contraction and every full one orthogonal).  Returns (hh_v (R, nbw) C-order ==
    nbw x R column-major, hh_tau (R,))."""
    R, nbw = int(R), int(nbw)
    v = uniform_pm1_np(seed ^ TAG_HHV, np.arange(R * nbw, dtype=np.uint64)).reshape(R, nbw)
    v[:, 0] = 1.0
    tau = 2.0 / np.einsum("ij,ij->i", v, v)
    return v, tau


def synthetic_reflectors_torch(R, nbw, seed, device="cpu", chunk=1 << 22):
    """torch version of synthetic_reflectors (bitwise identical), generated on `device`
    in chunks of reflectors (C5 has 28M reflectors = 14.4 GB)."""
    import torch
    R, nbw = int(R), int(nbw)
    v = torch.empty((R, nbw), dtype=torch.float64, device=device)
    tau = torch.empty((R,), dtype=torch.float64, device=device)
    for a in range(0, R, chunk):
        b = min(R, a + chunk)
        cnt = torch.arange(a * nbw, b * nbw, dtype=torch.int64, device=device)
        blk = uniform_pm1_torch(seed ^ TAG_HHV, cnt).reshape(b - a, nbw)
        blk[:, 0] = 1.0
        v[a:b] = blk
        tau[a:b] = 2.0 / (blk * blk).sum(dim=1)
    return v, tau


def synthetic_q_np(n, c0, c1, seed, ldq=None):
    """Columns [c0, c1) of the synthetic n x nev eigenvector block, uniform [-1,1):
    element (i, c) = stream(seed^TAG_Q)[c*n + i].  Returns (c1-c0, ldq) C-order array
    (the row-major view of a column-major n x (c1-c0) block with leading dim ldq)."""
    ldq = n if ldq is None else ldq
    out = np.zeros((c1 - c0, ldq), dtype=np.float64)
    if c1 > c0 and n > 0:
        cnt = np.arange(c0 * n, c1 * n, dtype=np.uint64)
        out[:, :n] = uniform_pm1_np(seed ^ TAG_Q, cnt).reshape(c1 - c0, n)
    return out


def synthetic_q_torch(n, c0, c1, seed, ldq=None, device="cpu", chunk_cols=1024):
    """torch version of synthetic_q_np (bitwise identical), generated on `device`."""
    import torch
    ldq = n if ldq is None else ldq
    out = torch.zeros((c1 - c0, ldq), dtype=torch.float64, device=device)
    for a in range(c0, c1, chunk_cols):
        b = min(c1, a + chunk_cols)
        cnt = torch.arange(a * n, b * n, dtype=torch.int64, device=device)
        out[a - c0:b - c0, :n] = uniform_pm1_torch(seed ^ TAG_Q, cnt).reshape(b - a, n)
    return out


# ---- generalized EVP inputs (NEXT-4) -----------------------------------------------------
TAG_SPD = 0x6A5B4C3D2E1F0918
TAG_TRIL = 0x19283746AFBECDD0


def spd_matrix(n, seed):
    """Random symmetric positive definite B = C C^T / n + I, C uniform [-1,1) (row-major
    stream), so cond(B) = O(1) and its Cholesky factor is well conditioned."""
    n = int(n)
    C = uniform_pm1_np(seed ^ TAG_SPD, np.arange(n * n, dtype=np.uint64)).reshape(n, n)
    return C @ C.T / max(n, 1) + np.eye(n)


def lower_triangular_cm_np(n, c0, c1, seed, ldl=None):
    """Columns [c0, c1) of a well-conditioned random lower-triangular n x n matrix, as the
    (c1-c0, ldl) row-major view of its column-major storage: L[i][c] = 1.5 + u/2 on the
    diagonal, u/n below it, 0 above (u uniform [-1,1) from element counter c*n + i), so
    L = D (I + N) with ||N||_2 < 1/2."""
    ldl = n if ldl is None else ldl
    out = np.zeros((c1 - c0, ldl), dtype=np.float64)
    if c1 > c0 and n > 0:
        u = uniform_pm1_np(seed ^ TAG_TRIL, np.arange(c0 * n, c1 * n, dtype=np.uint64)).reshape(c1 - c0, n)
        rows = np.arange(n)[None, :]
        cols = np.arange(c0, c1)[:, None]
        out[:, :n] = np.where(rows > cols, u / n, np.where(rows == cols, 1.5 + 0.5 * u, 0.0))
    return out


def lower_triangular_cm_torch(n, c0, c1, seed, ldl=None, device="cpu", chunk_cols=1024):
    """torch version of lower_triangular_cm_np (bitwise identical), generated on `device`."""
    import torch
    ldl = n if ldl is None else ldl
    out = torch.zeros((c1 - c0, ldl), dtype=torch.float64, device=device)
    rows = torch.arange(n, device=device)[None, :]
    for a in range(c0, c1, chunk_cols):
        b = min(c1, a + chunk_cols)
        u = uniform_pm1_torch(seed ^ TAG_TRIL, torch.arange(a * n, b * n, dtype=torch.int64, device=device)).reshape(b - a, n)
        cols = torch.arange(a, b, device=device)[:, None]
        out[a - c0:b - c0, :n] = torch.where(rows > cols, u / n, torch.where(rows == cols, 1.5 + 0.5 * u,
                                                                              torch.zeros_like(u)))
    return out


# ---- complex (NEXT-3, Hermitian) inputs ---------------------------------------------------
TAG_BAND_C = 0x4E3D2C1B0A998877
TAG_HHV_C = 0x7A6B5C4D3E2F1001
TAG_TAU_C = 0x1122334455667788
TAG_Q_C = 0x0F1E2D3C4B5A6978


def band_matrix_c(n, nbw, seed):
    """Random Hermitian band matrix in lower band storage ((nbw+1, n) complex, row d = d-th
    sub-diagonal): real and imaginary parts uniform [-1,1) from element counters 2k, 2k+1 of
    the flattened storage (k = d*n + c); the diagonal is real."""
    n, nbw = int(n), int(nbw)
    u = uniform_pm1_np(seed ^ TAG_BAND_C, np.arange(2 * (nbw + 1) * n, dtype=np.uint64)).reshape(nbw + 1, n, 2)
    band = u[..., 0] + 1j * u[..., 1]
    band[0] = band[0].real
    for dd in range(1, nbw + 1):
        band[dd, n - dd:] = 0.0
    return band


def synthetic_reflectors_c(R, nbw, seed):
    """Complex synthetic reflectors: v_0 = 1, v_i (i >= 1) complex uniform [-1,1)^2,
    tau = (1 + exp(i phi)) / ||v||^2 with phi uniform [-pi, pi) (then H = I - tau v v^H is
    unitary).  Returns (hh_v (R, nbw) complex128, hh_tau (R,) complex128)."""
    R, nbw = int(R), int(nbw)
    u = uniform_pm1_np(seed ^ TAG_HHV_C, np.arange(2 * R * nbw, dtype=np.uint64)).reshape(R, nbw, 2)
    v = u[..., 0] + 1j * u[..., 1]
    v[:, 0] = 1.0
    phi = np.pi * uniform_pm1_np(seed ^ TAG_TAU_C, np.arange(R, dtype=np.uint64))
    tau = (1.0 + np.exp(1j * phi)) / np.sum(np.abs(v) ** 2, axis=1)
    return v, tau


def synthetic_q_c_np(n, c0, c1, seed, ldq=None):
    """Columns [c0, c1) of a complex synthetic n x nev block: element (i, c) = u[2(c*n+i)] +
    i u[2(c*n+i)+1].  Returns (c1-c0, ldq) complex128 (row c = column c)."""
    ldq = n if ldq is None else ldq
    out = np.zeros((c1 - c0, ldq), dtype=np.complex128)
    if c1 > c0 and n > 0:
        u = uniform_pm1_np(seed ^ TAG_Q_C, np.arange(2 * c0 * n, 2 * c1 * n, dtype=np.uint64)).reshape(c1 - c0, n, 2)
        out[:, :n] = u[..., 0] + 1j * u[..., 1]
    return out
