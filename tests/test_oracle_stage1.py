"""Pins for the stage-1 oracle (NEXT-1: full -> band reduction and band -> full
back-transformation): LAPACK dsytrd at nbw = 1, explicit products,
similarity, and the whole two-stage eigensolver's residual."""
import numpy as np
import pytest

import oracle
from inputs import dense_symmetric

EPS = np.finfo(np.float64).eps


def explicit_Q1(n, V, tau):
    Q = np.eye(n)
    for r in range(len(tau)):
        Q = Q @ (np.eye(n) - tau[r] * np.outer(V[r], V[r]))
    return Q


def test_nbw1_equals_lapack_dsytrd():
    """With nbw = 1 the band reduction IS tridiagonalisation: same reflectors as dsytrd."""
    from scipy.linalg import lapack
    n = 20
    A = dense_symmetric(n, 11)
    band, V, tau, s, _ = oracle.reduce_to_band(A, 1)
    c, d, e, tt, info = lapack.dsytrd(A, lower=1)
    assert info == 0 and len(tau) == n - 2
    assert np.abs(tau - tt[:n - 2]).max() < 1e-13
    assert np.abs(band[0] - d).max() < 1e-13 and np.abs(band[1, :n - 1] - e).max() < 1e-13
    for j in range(n - 2):
        assert np.abs(V[j, j + 2:] - c[j + 2:, j]).max() < 1e-12


@pytest.mark.parametrize("n,b", [(12, 3), (30, 4), (40, 8), (25, 20)])
def test_similarity_and_band_structure(n, b):
    A = dense_symmetric(n, n + b)
    band, V, tau, s, Ared = oracle.reduce_to_band(A, b)
    assert len(tau) == max(n - b - 1, 0)
    assert np.all(V[np.arange(len(tau)), s] == 1.0)
    for j in range(len(tau)):
        assert np.all(V[j, :s[j]] == 0.0) and s[j] == j + b
    i, jj = np.indices((n, n))
    assert np.all(Ared[np.abs(i - jj) > b] == 0.0)               # exact band structure
    Q1 = explicit_Q1(n, V, tau)
    assert np.abs(Q1.T @ A @ Q1 - Ared).max() <= 20 * n * EPS * np.linalg.norm(A)
    assert np.abs(Q1.T @ Q1 - np.eye(n)).max() <= 20 * n * EPS


@pytest.mark.parametrize("n,b", [(30, 4), (40, 8)])
def test_apply_full_equals_explicit_product(n, b):
    A = dense_symmetric(n, 3 * n + b)
    band, V, tau, s, _ = oracle.reduce_to_band(A, b)
    X = np.random.default_rng(1).standard_normal((n, 6))
    got = oracle.apply_full(V, tau, s, X.T.copy(), n).T
    want = explicit_Q1(n, V, tau) @ X
    assert np.abs(got - want).max() <= 20 * n * EPS * np.abs(want).max()
    rev = oracle.apply_full(V[::-1], tau[::-1], s[::-1], X.T.copy(), n).T      # negative control
    assert np.abs(rev - want).max() > 1e-6


@pytest.mark.parametrize("n,b,nev", [(64, 8, 64), (200, 16, 60), (300, 32, 300)])
def test_two_stage_pipeline_residual(n, b, nev):
    """A -> band -> tridiagonal -> eig -> back-transform twice: eigenpairs of A."""
    c = oracle.make_case_full(n, b, nev, 7 + n)
    A, Q, lam = c["A"], c["Qfull"].T, c["lam"]
    assert np.abs(lam - np.linalg.eigvalsh(A)[:nev]).max() <= 50 * n * EPS * np.linalg.norm(A)
    res = np.linalg.norm(A @ Q - Q * lam) / (n * np.linalg.norm(A))
    assert res <= 1e-13, res
    assert np.abs(Q.T @ Q - np.eye(nev)).max() <= 50 * n * EPS
    # only one of the two transforms is not enough (the check has teeth)
    Qb = c["Qband"].T
    assert np.linalg.norm(A @ Qb - Qb * lam) / (n * np.linalg.norm(A)) > 1e-6
