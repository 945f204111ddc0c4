"""CPU oracle for trans_ev_tridi_to_band — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  It shares no code with the CUDA path
(paper_1811_01277_b200/) and never imports it; the product path never imports this.

What it computes (PAPER.md = /root/reference/PAPER.md):
  * make_case: the two-stage pipeline's inputs to the hot path — random symmetric band
    matrix B (inputs.band_matrix), band->tridiagonal chase recording reflectors (P:141-144,
    oracle.c), tridiagonal eigensolve T Vhat = Vhat Lambda (Eq. 5) with a
    library dense/tridiagonal eigensolver, lowest nev pairs ascending (R7).
  * apply: Q_out = H_0 H_1 ... H_{R-1} Q, one reflector at a time in exact reverse
    generation order (Eq. 6) — oracle.c:oracle_apply.
  * gen_back: V = L^-T Vtilde for the generalized EVP (Eq. 7; NEXT-4).
  * chase_c / apply_c / make_case_c: the complex Hermitian case (NEXT-3, DESIGN R15).
Pins (tests/test_oracle_*.py) tie every function to mathematics other than itself:
explicit reflector products, LAPACK dsytrd/dormqr at nbw = n-1, similarity, residual,
closed-form Toeplitz spectra, SPEC worked examples (tests/golden/).
"""
import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lib = None

BUILD_CMD = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
             "-o", _SO, _SRC, "-lm"]


def ensure_built(force=False):
    """Compile oracle.c with gcc (plain, -ffp-contract=off) if the .so is missing/stale."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _SO


def _load():
    global _lib
    if _lib is None:
        ensure_built()
        lib = ctypes.CDLL(_SO)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        lib.oracle_schedule.restype = i64
        lib.oracle_schedule.argtypes = [i64, i64, p, p]
        lib.oracle_chase.restype = i64
        lib.oracle_chase.argtypes = [i64, i64, p, p, p, p, p, p, p]
        lib.oracle_apply.restype = None
        lib.oracle_apply.argtypes = [i64, i64, i64, i64, p, p, p, p, p, i64, ctypes.c_int]
        lib.oracle_reduce_to_band.restype = i64
        lib.oracle_reduce_to_band.argtypes = [i64, i64, p, p, p, p]
        lib.oracle_apply_full.restype = None
        lib.oracle_apply_full.argtypes = [i64, i64, p, i64, p, p, p, i64, i64, ctypes.c_int]
        lib.oracle_chase_c.restype = i64
        lib.oracle_chase_c.argtypes = [i64, i64, p, p, p, p, p, p, p]
        lib.oracle_apply_c.restype = None
        lib.oracle_apply_c.argtypes = [i64, i64, i64, p, p, p, p, p, i64, ctypes.c_int]
        lib.oracle_gen_back.restype = None
        lib.oracle_gen_back.argtypes = [i64, i64, p, i64, p, i64, ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def schedule(n, nbw):
    """Explicit reflector schedule by plain enumeration: (s, L) arrays of length R."""
    lib = _load()
    R = lib.oracle_schedule(n, nbw, None, None)
    s = np.zeros(max(R, 1), dtype=np.int64)
    L = np.zeros(max(R, 1), dtype=np.int64)
    lib.oracle_schedule(n, nbw, _ptr(s), _ptr(L))
    return s[:R], L[:R]


def count(n, nbw):
    return int(_load().oracle_schedule(n, nbw, None, None))


def chase(band):
    """Band -> tridiagonal chase of the lower band (nbw+1, n).  Returns
    (hh_v (R, nbw), hh_tau (R,), s (R,), L (R,), d (n,), e (n-1,))."""
    lib = _load()
    band = np.ascontiguousarray(band, dtype=np.float64)
    nb1, n = band.shape
    nbw = nb1 - 1
    R = count(n, nbw)
    hh_v = np.zeros((max(R, 1), max(nbw, 1)), dtype=np.float64)
    tau = np.zeros(max(R, 1), dtype=np.float64)
    s = np.zeros(max(R, 1), dtype=np.int64)
    L = np.zeros(max(R, 1), dtype=np.int64)
    d = np.zeros(max(n, 1), dtype=np.float64)
    e = np.zeros(max(n - 1, 1), dtype=np.float64)
    r = lib.oracle_chase(n, nbw, _ptr(band), _ptr(hh_v), _ptr(tau), _ptr(s), _ptr(L), _ptr(d), _ptr(e))
    if r != R:
        raise RuntimeError(f"oracle_chase returned {r}, expected {R}")
    return hh_v[:R, :nbw], tau[:R], s[:R], L[:R], d[:n], e[:max(n - 1, 0)]


def apply(hh_v, hh_tau, s, L, Q, nthreads=None):
    """Q (nev, ldq) row-major view of column-major n x nev; returns a new array
    Q_out = H_0 ... H_{R-1} Q (reverse generation order)."""
    lib = _load()
    Q = np.array(Q, dtype=np.float64, order="C", copy=True)
    nev, ldq = Q.shape
    hh_v = np.ascontiguousarray(hh_v, dtype=np.float64)
    R, nbw = hh_v.shape if hh_v.ndim == 2 else (0, 1)
    hh_tau = np.ascontiguousarray(hh_tau, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.int64)
    L = np.ascontiguousarray(L, dtype=np.int64)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    if R > 0 and nev > 0:
        lib.oracle_apply(ldq, nbw, nev, R, _ptr(hh_v), _ptr(hh_tau), _ptr(s), _ptr(L),
                         _ptr(Q), ldq, int(nthreads))
    return Q


def tridiag_eig(d, e, nev):
    """Lowest nev eigenpairs of the symmetric tridiagonal T(d, e), ascending (Eq. 5;
    DESIGN.md R7).  Library solver: numpy dense eigh for n <= 1024, scipy stemr beyond.
    Returns (lam (nev,), Vhat (n, nev))."""
    n = len(d)
    if nev == 0:
        return np.zeros(0), np.zeros((n, 0))
    if n <= 1024:
        T = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
        lam, V = np.linalg.eigh(T)
        return lam[:nev].copy(), np.ascontiguousarray(V[:, :nev])
    from scipy.linalg import eigh_tridiagonal
    lam, V = eigh_tridiagonal(d, e, select="i", select_range=(0, nev - 1), lapack_driver="stemr")
    return lam, np.ascontiguousarray(V)


def dense_from_band(band):
    nb1, n = band.shape
    B = np.zeros((n, n))
    for dd in range(nb1):
        idx = np.arange(n - dd)
        B[idx + dd, idx] = band[dd, :n - dd]
        B[idx, idx + dd] = band[dd, :n - dd]
    return B


def make_case(n, nbw, nev, seed):
    """Full oracle case: returns dict(B band, hh_v, hh_tau, s, L, d, e, lam, Vhat, Q_ref)
    where Q_ref = apply(reflectors, Vhat) holds the band matrix's eigenvectors."""
    from inputs import band_matrix
    t0 = time.time()
    band = band_matrix(n, nbw, seed)
    hh_v, hh_tau, s, L, d, e = chase(band)
    lam, Vhat = tridiag_eig(d, e, nev)
    Qin = np.ascontiguousarray(Vhat.T)               # (nev, n): column-major n x nev
    Qref = apply(hh_v, hh_tau, s, L, Qin)
    return dict(n=n, nbw=nbw, nev=nev, seed=seed, band=band, hh_v=hh_v, hh_tau=hh_tau,
                s=s, L=L, d=d, e=e, lam=lam, Qin=Qin, Qref=Qref, secs=time.time() - t0)


def residual(band, Q, lam):
    """||B Q - Q Lambda||_F / (n ||B||_F) with Q given as (nev, n) rows = eigenvectors
    (R8: Frobenius on both).  Uses the band structure (B applied via its
    diagonals), no dense n x n matrix."""
    nb1, n = band.shape
    X = np.asarray(Q)[:, :n].T                       # n x nev
    BX = band[0][:, None] * X
    for dd in range(1, nb1):
        bd = band[dd, :n - dd][:, None]
        BX[dd:] += bd * X[:-dd]
        BX[:-dd] += bd * X[dd:]
    nrmB = np.sqrt(np.sum(band[0] ** 2) + 2.0 * np.sum(band[1:] ** 2))
    return float(np.linalg.norm(BX - X * lam[None, :]) / (n * nrmB))


# ------------------------------------------------------------------ stage 1 (NEXT-1)
def reduce_to_band(A, nbw):
    """Full symmetric A (n x n) -> band (half-bandwidth nbw), one reflector per column
    (oracle.c:oracle_reduce_to_band).  Returns (band lower storage
    (nbw+1, n), V (K, n) rows = reflector vectors (zeros before s, v[s] = 1), tau (K,), s (K,),
    the reduced full matrix)."""
    lib = _load()
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    n = A.shape[0]
    K = max(n - nbw - 1, 0)
    V = np.zeros((max(K, 1), n), dtype=np.float64)
    tau = np.zeros(max(K, 1))
    s = np.zeros(max(K, 1), dtype=np.int64)
    k = lib.oracle_reduce_to_band(n, nbw, A.ctypes.data_as(ctypes.c_void_p), _ptr(V), _ptr(tau), _ptr(s))
    assert k == K
    band = np.zeros((nbw + 1, n))
    for dd in range(nbw + 1):
        band[dd, :n - dd] = np.diagonal(A, -dd)
    return band, V[:K], tau[:K], s[:K], A


def apply_full(V, tau, s, Q, n, nthreads=None):
    """Q (nev, ldq) -> H_0 ... H_{K-1} Q for the stage-1 reflectors (oracle_apply_full)."""
    lib = _load()
    Q = np.array(Q, dtype=np.float64, order="C", copy=True)
    nev, ldq = Q.shape
    V = np.ascontiguousarray(V, dtype=np.float64)
    K = V.shape[0] if V.ndim == 2 else 0
    if K and nev:
        lib.oracle_apply_full(n, K, _ptr(V), V.shape[1], _ptr(np.ascontiguousarray(tau, dtype=np.float64)),
                              _ptr(np.ascontiguousarray(s, dtype=np.int64)), _ptr(Q), ldq, nev,
                              int(nthreads or os.cpu_count() or 1))
    return Q


def make_case_full(n, nbw, nev, seed):
    """The whole two-stage pipeline on a random dense symmetric A (inputs.dense_symmetric):
    A -> band (stage 1) -> tridiagonal (stage 2 chase) -> lowest nev eigenpairs of T ->
    back-transformed twice.  Returns a dict with every intermediate."""
    from inputs import dense_symmetric
    A = dense_symmetric(n, seed)
    band, V1, tau1, s1, _ = reduce_to_band(A, nbw)
    hh_v, hh_tau, s2, L2, d, e = chase(band)
    lam, Vhat = tridiag_eig(d, e, nev)
    Qin = np.ascontiguousarray(Vhat.T)
    Qband = apply(hh_v, hh_tau, s2, L2, Qin)
    Qfull = apply_full(V1, tau1, s1, Qband, n)
    return dict(A=A, band=band, V1=V1, tau1=tau1, s1=s1, hh_v=hh_v, hh_tau=hh_tau, s2=s2, L2=L2, d=d, e=e,
                lam=lam, Qin=Qin, Qband=Qband, Qfull=Qfull)


# ------------------------------------------------------------------ generalized EVP (NEXT-4)
def gen_back(L, Q, nthreads=None):
    """V = (L^{-1})^T Vtilde (Eq. 7) by backward substitution per column
    (oracle.c:oracle_gen_back).  L: (n, n) lower-triangular numpy matrix (mathematical layout);
    Q: (nev, ldq) row-major view of the column-major n x nev block.  Returns a new array."""
    lib = _load()
    L = np.asarray(L, dtype=np.float64)
    n = L.shape[0]
    Lcm = np.ascontiguousarray(L.T)                  # row i = column i of L (column-major storage)
    Q = np.array(Q, dtype=np.float64, order="C", copy=True)
    nev, ldq = Q.shape
    if n and nev:
        lib.oracle_gen_back(n, nev, _ptr(Lcm), n, _ptr(Q), ldq, int(nthreads or os.cpu_count() or 1))
    return Q


def make_case_generalized(n, nbw, nev, seed):
    """The generalized EVP A V = B V Lambda through the whole two-stage pipeline:
    B = L L^T (Cholesky, library), Atilde = L^-1 A L^-T (library triangular solves), the
    two-stage solve of make_case_full on Atilde, then V = L^-T Vtilde (gen_back)."""
    from inputs import dense_symmetric, spd_matrix
    from scipy.linalg import solve_triangular
    A = dense_symmetric(n, seed)
    B = spd_matrix(n, seed)
    L = np.linalg.cholesky(B)
    X = solve_triangular(L, A, lower=True)
    At = solve_triangular(L, X.T, lower=True).T
    At = 0.5 * (At + At.T)
    band, V1, tau1, s1, _ = reduce_to_band(At, nbw)
    hh_v, hh_tau, s2, L2, d, e = chase(band)
    lam, Vhat = tridiag_eig(d, e, nev)
    Qin = np.ascontiguousarray(Vhat.T)
    Qband = apply(hh_v, hh_tau, s2, L2, Qin)
    Qt = apply_full(V1, tau1, s1, Qband, n)
    V = gen_back(L, Qt)
    return dict(A=A, B=B, L=L, At=At, lam=lam, Qt=Qt, V=V, band=band, hh_v=hh_v, hh_tau=hh_tau, s2=s2, L2=L2,
                V1=V1, tau1=tau1, s1=s1, Qin=Qin, Qband=Qband)


# ------------------------------------------------------------------ complex Hermitian (NEXT-3)
def chase_c(band):
    """Hermitian band -> tridiagonal chase (oracle.c:oracle_chase_c, zlarfg convention).
    band: (nbw+1, n) complex lower band storage.  Returns (hh_v (R, nbw) complex, hh_tau (R,)
    complex, s, L, d (n,) real, e (n-1,) complex)."""
    lib = _load()
    band = np.ascontiguousarray(band, dtype=np.complex128)
    nb1, n = band.shape
    nbw = nb1 - 1
    R = count(n, nbw)
    hh_v = np.zeros((max(R, 1), max(nbw, 1)), dtype=np.complex128)
    tau = np.zeros(max(R, 1), dtype=np.complex128)
    s = np.zeros(max(R, 1), dtype=np.int64)
    L = np.zeros(max(R, 1), dtype=np.int64)
    d = np.zeros(max(n, 1), dtype=np.float64)
    e = np.zeros(max(n - 1, 1), dtype=np.complex128)
    r = lib.oracle_chase_c(n, nbw, _ptr(band), _ptr(hh_v), _ptr(tau), _ptr(s), _ptr(L), _ptr(d), _ptr(e))
    if r != R:
        raise RuntimeError(f"oracle_chase_c returned {r}, expected {R}")
    return hh_v[:R, :nbw], tau[:R], s[:R], L[:R], d[:n], e[:max(n - 1, 0)]


def apply_c(hh_v, hh_tau, s, L, Q, nthreads=None):
    """Q (nev, ldq) complex; returns H_0 ... H_{R-1} Q (H_r = I - tau_r v_r v_r^H)."""
    lib = _load()
    Q = np.array(Q, dtype=np.complex128, order="C", copy=True)
    nev, ldq = Q.shape
    hh_v = np.ascontiguousarray(hh_v, dtype=np.complex128)
    R, nbw = hh_v.shape if hh_v.ndim == 2 else (0, 1)
    if R > 0 and nev > 0:
        lib.oracle_apply_c(nbw, nev, R, _ptr(hh_v), _ptr(np.ascontiguousarray(hh_tau, dtype=np.complex128)),
                           _ptr(np.ascontiguousarray(s, dtype=np.int64)), _ptr(np.ascontiguousarray(L, dtype=np.int64)),
                           _ptr(Q), ldq, int(nthreads or os.cpu_count() or 1))
    return Q


def tridiag_eig_c(d, e, nev):
    """Lowest nev eigenpairs of the Hermitian tridiagonal T (real d, complex e = T(i+1, i)).
    T = D T_r D^H with the unitary diagonal D (D_0 = 1, D_{i+1} = D_i e_i / |e_i|, 1 where
    e_i = 0) and the real symmetric tridiagonal T_r (d, |e|): eigenvectors D Vhat_r
    (R15).  Returns (lam, Vhat (n, nev) complex)."""
    n = len(d)
    ph = np.ones(n, dtype=np.complex128)
    ae = np.abs(e)
    for i in range(n - 1):
        ph[i + 1] = ph[i] * (e[i] / ae[i] if ae[i] != 0 else 1.0)
    lam, Vr = tridiag_eig(np.asarray(d, dtype=np.float64), ae, nev)
    return lam, ph[:, None] * Vr


def dense_from_band_c(band):
    nb1, n = band.shape
    B = np.zeros((n, n), dtype=np.complex128)
    for dd in range(nb1):
        idx = np.arange(n - dd)
        B[idx + dd, idx] = band[dd, :n - dd]
        B[idx, idx + dd] = np.conj(band[dd, :n - dd])
    return B


def residual_c(band, Q, lam):
    """||B X - X Lambda||_F / (n ||B||_F), X = Q[:, :n]^T (columns = eigenvectors), B Hermitian band."""
    nb1, n = band.shape
    X = np.asarray(Q)[:, :n].T
    BX = band[0].real[:, None] * X
    for dd in range(1, nb1):
        bd = band[dd, :n - dd][:, None]
        BX[dd:] += bd * X[:-dd]
        BX[:-dd] += np.conj(bd) * X[dd:]
    nrmB = np.sqrt(np.sum(band[0].real ** 2) + 2.0 * np.sum(np.abs(band[1:]) ** 2))
    return float(np.linalg.norm(BX - X * lam[None, :]) / (n * nrmB))


def make_case_c(n, nbw, nev, seed):
    """Complex Hermitian case: band -> chase -> tridiagonal eig (with the phase scaling) ->
    back-transformation.  Returns dict(band, hh_v, hh_tau, s, L, d, e, lam, Qin, Qref)."""
    from inputs import band_matrix_c
    band = band_matrix_c(n, nbw, seed)
    hh_v, hh_tau, s, L, d, e = chase_c(band)
    lam, Vhat = tridiag_eig_c(d, e, nev)
    Qin = np.ascontiguousarray(Vhat.T)
    Qref = apply_c(hh_v, hh_tau, s, L, Qin)
    return dict(n=n, nbw=nbw, nev=nev, band=band, hh_v=hh_v, hh_tau=hh_tau, s=s, L=L, d=d, e=e, lam=lam,
                Qin=Qin, Qref=Qref)
