"""Pins for the CPU oracle — every check ties the oracle to
something other than itself: explicit dense reflector products, LAPACK, orthogonal
similarity invariants, closed forms, SPEC worked examples (tests/golden/)."""
import os

import numpy as np
import pytest

import oracle
from inputs import band_matrix, synthetic_reflectors, synthetic_q_np

EPS = np.finfo(np.float64).eps
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, *vals = line.split()
        out[k] = vals
    return out


def explicit_Qbc(n, hh_v, tau, s, L):
    """Q_bc = H_0 H_1 ... H_{R-1}, each H_r = I - tau_r v_r v_r^T formed densely
    (PAPER.md P:117-121 definition, generation order)."""
    Q = np.eye(n)
    for r in range(len(tau)):
        v = np.zeros(n)
        v[s[r]:s[r] + L[r]] = hh_v[r, :L[r]]
        v[s[r]] = 1.0
        Q = Q @ (np.eye(n) - tau[r] * np.outer(v, v))
    return Q


def closed_form_R(n, b):
    """R(n, b) = (n-2) + F(n-3), F(x) = sum_{t=0}^{x} floor(t/b)."""
    if n < 3 or b < 2:
        return 0
    x = n - 3
    q = x // b
    F = b * q * (q - 1) // 2 + q * (x % b + 1)
    return (n - 2) + F


SMALL = [(12, 3), (40, 5), (64, 8), (33, 32), (20, 19), (57, 6), (30, 2), (16, 4)]


# ---------------------------------------------------------------- counts / schedule
@pytest.mark.parametrize("n,b", SMALL + [(3, 2), (4, 3), (100, 16), (513, 16), (1000, 64)])
def test_count_matches_closed_form(n, b):
    assert oracle.count(n, b) == closed_form_R(n, b)


def test_config_counts_golden():
    for line in open(os.path.join(GOLD, "paper_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, n, b, nev, R, sumL = line.split()
        n, b, R, sumL = int(n), int(b), int(R), int(sumL)
        assert closed_form_R(n, b) == R, name
        if n <= 20000:
            s, L = oracle.schedule(n, b)
            assert len(s) == R and int(L.sum()) == sumL, name
            assert L.min() >= 2 and L.max() <= b


def test_degenerate_counts():
    for n in range(0, 3):
        assert oracle.count(n, 4) == 0
    assert oracle.count(50, 1) == 0            # nbw = 1: already tridiagonal


# ---------------------------------------------------------------- P1 explicit product
@pytest.mark.parametrize("n,b", SMALL)
def test_P1_apply_equals_explicit_product(n, b):
    band = band_matrix(n, b, 1000 + n * 7 + b)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    assert len(tau) == closed_form_R(n, b)
    rng = np.random.default_rng(n * 31 + b)
    Vhat = rng.standard_normal((n, 5))
    got = oracle.apply(hh_v, tau, s, L, Vhat.T.copy()).T
    want = explicit_Qbc(n, hh_v, tau, s, L) @ Vhat
    assert np.abs(got - want).max() <= 10 * n * EPS * max(1.0, np.abs(want).max())


def test_P1_catches_wrong_order():
    """The explicit product in generation order distinguishes a reversed order."""
    n, b = 40, 5
    band = band_matrix(n, b, 3)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    Vhat = np.eye(n)[:, :6]
    got = oracle.apply(hh_v, tau, s, L, Vhat.T.copy()).T
    rev = oracle.apply(hh_v[::-1], tau[::-1], s[::-1], L[::-1], Vhat.T.copy()).T
    want = explicit_Qbc(n, hh_v, tau, s, L) @ Vhat
    assert np.abs(got - want).max() < 1e-13
    assert np.abs(rev - want).max() > 1e-3


# ---------------------------------------------------------------- P2 similarity
@pytest.mark.parametrize("n,b", SMALL)
def test_P2_similarity_tridiagonal(n, b):
    band = band_matrix(n, b, 77 + n + b)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    B = oracle.dense_from_band(band)
    Q = explicit_Qbc(n, hh_v, tau, s, L)
    T = Q.T @ B @ Q
    Tt = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
    nrm = np.linalg.norm(B)
    assert np.abs(T - Tt).max() <= 10 * n * EPS * nrm
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 10 * n * EPS


# ---------------------------------------------------------------- P3 LAPACK special case
def test_P3_full_band_equals_lapack_dsytrd_dormqr():
    from scipy.linalg import lapack
    n = 24
    band = band_matrix(n, n - 1, 2024)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    assert len(tau) == n - 2 and np.all(L == np.arange(n - 1, 1, -1))
    A = oracle.dense_from_band(band)
    c, dd, ee, tt, info = lapack.dsytrd(A, lower=1)
    assert info == 0
    assert np.abs(tau - tt[:n - 2]).max() < 1e-13
    assert tt[n - 2] == 0.0                       # LAPACK's length-1 tail reflector
    assert np.abs(d - dd).max() < 1e-13 and np.abs(e - ee).max() < 1e-13
    for j in range(n - 2):                        # same vectors (LAPACK stores v below the subdiagonal)
        assert np.abs(hh_v[j, 1:L[j]] - c[j + 2:, j]).max() < 1e-12
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, 7))
    got = oracle.apply(hh_v, tau, s, L, X.T.copy()).T
    want = X.copy()
    qa = np.asfortranarray(c[1:, :n - 1])
    lw = lapack.dormqr("L", "N", qa, tt[:n - 1], np.asfortranarray(want[1:]), lwork=-1)[1]
    cq, work, info = lapack.dormqr("L", "N", qa, tt[:n - 1], np.asfortranarray(want[1:]), lwork=int(lw[0]))
    assert info == 0
    want[1:] = cq
    assert np.abs(got - want).max() < 1e-13


# ---------------------------------------------------------------- P4 trivial cases
def test_P4_no_op_cases_bitwise():
    n = 30
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((4, n))
    # all tau = 0
    s, L = oracle.schedule(n, 5)
    hv, tau = synthetic_reflectors(len(s), 5, 9)
    out = oracle.apply(hv, np.zeros_like(tau), s, L, Q)
    assert np.array_equal(out, Q)
    # nbw = 1: R = 0
    band = band_matrix(n, 1, 3)
    hv, tau, s, L, d, e = oracle.chase(band)
    assert len(tau) == 0
    assert np.array_equal(d, band[0]) and np.array_equal(e, band[1, :n - 1])
    # an already tridiagonal matrix given with nbw = 4: every reflector is the identity
    band = band_matrix(n, 4, 3)
    band[2:] = 0.0
    hv, tau, s, L, d, e = oracle.chase(band)
    assert np.all(tau == 0.0)
    assert np.array_equal(oracle.apply(hv, tau, s, L, Q), Q)


# ---------------------------------------------------------------- P5 inverse replay
@pytest.mark.parametrize("n,b", [(40, 5), (64, 8), (57, 6)])
def test_P5_inverse_replay(n, b):
    band = band_matrix(n, b, 5 + n)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    rng = np.random.default_rng(2)
    Q = rng.standard_normal((6, n))
    fwd = oracle.apply(hh_v, tau, s, L, Q)                       # H_0 ... H_{R-1} Q
    back = oracle.apply(hh_v[::-1], tau[::-1], s[::-1], L[::-1], fwd)  # H_{R-1} ... H_0 (.)
    assert np.abs(back - Q).max() <= 20 * n * EPS * np.abs(Q).max()


# ---------------------------------------------------------------- P6 invariants
@pytest.mark.parametrize("n,b", [(64, 8), (100, 16), (33, 32)])
def test_P6_invariants(n, b):
    band = band_matrix(n, b, 11 + n)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    nz = tau != 0
    vn = np.array([1.0 + np.sum(hh_v[r, 1:L[r]] ** 2) for r in range(len(tau))])
    assert np.abs(tau[nz] * vn[nz] - 2.0).max() < 1e-13      # dlarfg: tau ||v||^2 = 2
    assert np.all(hh_v[:, 0] == 1.0)
    for r in range(len(tau)):
        assert np.all(hh_v[r, L[r]:] == 0.0)
    B = oracle.dense_from_band(band)
    Tt = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
    nrm = np.linalg.norm(B)
    assert np.abs(np.linalg.eigvalsh(Tt) - np.linalg.eigvalsh(B)).max() <= 10 * n * EPS * nrm
    lam, Vh = oracle.tridiag_eig(d, e, n)
    Qo = oracle.apply(hh_v, tau, s, L, Vh.T.copy())
    assert np.abs(Qo @ Qo.T - np.eye(n)).max() <= 20 * n * EPS
    assert np.abs(np.linalg.norm(Qo, axis=1) - 1.0).max() <= 10 * n * EPS


# ---------------------------------------------------------------- P7 residual
@pytest.mark.parametrize("n,b,nev", [(64, 8, 64), (200, 16, 50), (512, 16, 512)])
def test_P7_residual(n, b, nev):
    case = oracle.make_case(n, b, nev, 1811012771 if n == 512 else 99 + n)
    res = oracle.residual(case["band"], case["Qref"], case["lam"])
    assert res <= 1e-13, res
    # the un-back-transformed Vhat is NOT an eigenbasis of B (the check has teeth)
    assert oracle.residual(case["band"], case["Qin"], case["lam"]) > 1e-6


def _residual_mutants(band, Q, lam):
    """Plausible mis-normalisations of oracle.residual (each must fail the pins below):
    off-diagonals counted once in ||B||_F, the 1/n dropped, the max-norm for ||B||."""
    nb1, n = band.shape
    X = np.asarray(Q)[:, :n].T
    B = oracle.dense_from_band(band)
    num = np.linalg.norm(B @ X - X * lam[None, :])
    once = np.sqrt(np.sum(band ** 2))
    return {"offdiag_once": num / (n * once), "no_1_over_n": num / np.linalg.norm(B),
            "max_norm": num / (n * np.abs(B).max())}


def test_P7_residual_closed_form_toeplitz():
    """R8 pinned by a closed form: B = tridiag(-1, 2, -1) (nbw = 1 storage widened to nbw = 3
    with zero diagonals), X = the first k unit vectors, Lambda = 0.  Then B X = the first k
    columns of B: ||B X||_F^2 = 5 + 6 (k - 1) for k < n (column 0 has 2^2 + 1, the others
    1 + 4 + 1), ||B||_F^2 = 4 n + 2 (n - 1), so the residual is sqrt(5 + 6(k-1)) / (n sqrt(6n - 2))."""
    n, k = 40, 7
    band = np.zeros((4, n))
    band[0] = 2.0
    band[1, :n - 1] = -1.0
    Q = np.zeros((k, n))
    Q[np.arange(k), np.arange(k)] = 1.0
    lam = np.zeros(k)
    want = np.sqrt(5.0 + 6.0 * (k - 1)) / (n * np.sqrt(6.0 * n - 2.0))
    got = oracle.residual(band, Q, lam)
    assert abs(got - want) <= 1e-15 * want
    for name, bad in _residual_mutants(band, Q, lam).items():
        assert abs(bad - want) > 1e-3 * want, name


@pytest.mark.parametrize("n,b,nev,ldq", [(64, 8, 20, 64), (301, 16, 45, 302), (512, 64, 33, 512)])
def test_P7_residual_equals_dense_formula(n, b, nev, ldq):
    """oracle.residual (banded B applied by diagonals, ||B||_F from the stored band) equals the
    dense definition ||B X - X Lambda||_F / (n ||B||_F) with an explicit dense B built by
    numpy.  Random X and Lambda (not eigenpairs), so every term of B X enters the norm, and
    the ldq padding of Q is ignored."""
    rng = np.random.default_rng(n + b)
    band = rng.uniform(-1, 1, (b + 1, n))
    for dd in range(1, b + 1):
        band[dd, n - dd:] = 0.0                     # outside the matrix: never part of B
    Q = rng.uniform(-1, 1, (nev, ldq))
    lam = rng.uniform(-3, 3, nev)
    B = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - b), min(n, i + b + 1)):
            B[i, j] = band[abs(i - j), min(i, j)]
    X = Q[:, :n].T
    want = np.linalg.norm(B @ X - X @ np.diag(lam), "fro") / (n * np.linalg.norm(B, "fro"))
    got = oracle.residual(band, Q, lam)
    assert abs(got - want) <= 1e-13 * want
    for name, bad in _residual_mutants(band, Q, lam).items():
        assert abs(bad - want) > 1e-3 * want, name


# ---------------------------------------------------------------- P8/P9 column independence, threads
def test_P8_column_subset_bitwise_and_P9_threads():
    n, b = 300, 16
    s, L = oracle.schedule(n, b)
    hv, tau = synthetic_reflectors(len(s), b, 4)
    Q = synthetic_q_np(n, 0, 40, 8)
    full = oracle.apply(hv, tau, s, L, Q, nthreads=8)
    sub = oracle.apply(hv, tau, s, L, Q[13:21], nthreads=1)
    assert np.array_equal(full[13:21], sub)
    one = oracle.apply(hv, tau, s, L, Q, nthreads=1)
    assert np.array_equal(full, one)


def test_P8_ldq_padding_untouched():
    n, b, ldq = 50, 6, 56
    s, L = oracle.schedule(n, b)
    hv, tau = synthetic_reflectors(len(s), b, 4)
    Q = synthetic_q_np(n, 0, 5, 8, ldq=ldq)
    Q[:, n:] = 7.0
    out = oracle.apply(hv, tau, s, L, Q)
    assert np.all(out[:, n:] == 7.0)
    assert np.array_equal(out[:, :n], oracle.apply(hv, tau, s, L, Q[:, :n].copy()))


# ---------------------------------------------------------------- P10 hand example (golden)
def test_P10_spec_hand_reflector():
    g = _gold("spec_hand_reflector.txt")
    v = np.array(g["v"], dtype=float)
    beta = float(g["beta"][0])
    x = np.array(g["x"], dtype=float)
    want = np.array(g["expected"], dtype=float)
    # one reflector of length 2 on rows [1, 3) of an n = 3 system (row 0 untouched)
    hh_v = np.array([[1.0, v[1]]])
    out = oracle.apply(hh_v, np.array([beta]), np.array([1]), np.array([2]),
                       np.array([[5.0, x[0], x[1]]]))
    assert np.array_equal(out[0, 1:], want) and out[0, 0] == 5.0


def test_golden_spec_ones_plus_identity():
    g = _gold("spec_ones_plus_identity.txt")
    A = np.array(g["A"], dtype=float).reshape(3, 3)
    lam_want = np.array(g["eigenvalues"], dtype=float)
    band = np.zeros((3, 3))
    band[0] = np.diag(A)
    band[1, :2] = np.diag(A, -1)
    band[2, :1] = np.diag(A, -2)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    assert len(tau) == 1
    lam, Vh = oracle.tridiag_eig(d, e, 3)
    assert np.abs(lam - lam_want).max() < 1e-14
    Q = oracle.apply(hh_v, tau, s, L, Vh.T.copy())
    assert np.abs(A @ Q.T - Q.T * lam).max() < 1e-14


# ---------------------------------------------------------------- P11 closed-form Toeplitz
def test_P11_toeplitz_closed_form():
    """nbw = 1 Toeplitz input (d = 2, e = -1): R = 0, the pipeline is the
    tridiagonal solve alone; lambda_j = 2 - 2 cos(j pi/(n+1)),
    v_j(i) = sqrt(2/(n+1)) sin((i+1) j pi/(n+1))."""
    n = 40
    band = np.zeros((2, n))
    band[0] = 2.0
    band[1, :n - 1] = -1.0
    hh_v, tau, s, L, d, e = oracle.chase(band)
    assert len(tau) == 0
    lam, Vh = oracle.tridiag_eig(d, e, n)
    j = np.arange(1, n + 1)
    assert np.abs(lam - (2 - 2 * np.cos(j * np.pi / (n + 1)))).max() < 1e-13
    i = np.arange(n)[:, None]
    Vc = np.sqrt(2.0 / (n + 1)) * np.sin((i + 1) * j[None, :] * np.pi / (n + 1))
    sgn = np.sign(np.sum(Vh * Vc, axis=0))
    assert np.abs(Vh * sgn - Vc).max() < 1e-12
    Q = oracle.apply(hh_v, tau, s, L, Vh.T.copy())
    assert np.array_equal(Q, Vh.T)


def test_spec_chase_spectrum_n32_b4():
    """n = 32, b = 4 — the chase's d, e have the band matrix's spectrum."""
    band = band_matrix(32, 4, 32)
    hh_v, tau, s, L, d, e = oracle.chase(band)
    B = oracle.dense_from_band(band)
    lam = oracle.tridiag_eig(d, e, 32)[0]
    assert np.abs(lam - np.linalg.eigvalsh(B)).max() <= 10 * 32 * EPS * np.linalg.norm(B)
    assert abs(np.sum(d) - np.trace(B)) <= 10 * 32 * EPS * np.linalg.norm(B)


# ---------------------------------------------------------------- P12 compact k-group algebra
@pytest.mark.parametrize("k", [2, 4, 6, 8])
def test_P12_compact_group_equals_sequential(k):
    """k reflectors of one depth (each shifted one row, window b+k-1 rows) applied as
    Q <- Q - V (T^T (V^T Q)) with T the forward (dlarft) triangular factor equals
    applying them one by one, reflector a = 0 (lowest, largest j) first."""
    b, w = 16, 5
    rng = np.random.default_rng(k)
    Wr = b + k - 1
    V = np.zeros((Wr, k))
    tau = np.zeros(k)
    for a in range(k):
        v = rng.uniform(-1, 1, b)
        v[0] = 1.0
        V[k - 1 - a:k - 1 - a + b, a] = v
        tau[a] = 2.0 / (v @ v)
    Q = rng.standard_normal((Wr, w))
    seq = Q.copy()
    for a in range(k):
        seq -= tau[a] * np.outer(V[:, a], V[:, a] @ seq)
    G = V.T @ V
    T = np.zeros((k, k))                           # dlarft forward: H_0 ... H_{k-1} = I - V T V^T
    for a in range(k):
        T[a, a] = tau[a]
        T[:a, a] = -tau[a] * T[:a, :a] @ G[:a, a]
    comp = Q - V @ (T.T @ (V.T @ Q))
    assert np.abs(comp - seq).max() < 1e-13
    # the form the DMMA kernel evaluates: U = -V T prepared once, W^T = Q^T U, Q += V W
    U = -V @ T
    comp_u = Q + V @ (U.T @ Q)
    assert np.abs(comp_u - seq).max() < 1e-13


def test_residual_parallel_equals_residual():
    """tests/cases.residual_parallel (column chunks on threads) is exactly oracle.residual."""
    from cases import residual_parallel
    rng = np.random.default_rng(3)
    band = rng.uniform(-1, 1, (9, 300))
    Q = rng.uniform(-1, 1, (77, 300))
    lam = rng.uniform(-1, 1, 77)
    assert abs(residual_parallel(band, Q, lam, chunk=16) - oracle.residual(band, Q, lam)) <= 1e-15
