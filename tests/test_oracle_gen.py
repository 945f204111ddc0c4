"""Pins of the NEXT-4 oracle: the generalized back-transformation V = (L^{-1})^T Vtilde
(Eq. 7; B = L L^T; Atilde = L^-1 A L^-T).
oracle.gen_back is plain backward substitution (oracle.c); the pins below tie it to an
independent library routine, to special cases and to the generalized eigenproblem itself."""
import numpy as np
import pytest
from scipy.linalg import eigh, solve_triangular

import oracle
from inputs import dense_symmetric, lower_triangular_cm_np, spd_matrix


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("n,nev", [(1, 1), (7, 3), (64, 64), (200, 37)])
def test_gen_back_matches_library_triangular_solve(n, nev):
    rng = np.random.default_rng(n)
    L = np.linalg.cholesky(spd_matrix(n, 5 + n))
    Q = rng.uniform(-1, 1, (nev, n + 3))
    got = oracle.gen_back(L, Q)
    want = solve_triangular(L, Q[:, :n].T, trans="T", lower=True).T
    assert _rel(got[:, :n], want) <= 1e-12
    assert np.array_equal(got[:, n:], Q[:, n:])          # padding rows untouched


def test_gen_back_special_cases():
    rng = np.random.default_rng(1)
    Q = rng.uniform(-1, 1, (5, 9))
    assert np.array_equal(oracle.gen_back(np.eye(9), Q), Q)                  # L = I
    d = rng.uniform(1, 2, 9)
    assert np.allclose(oracle.gen_back(np.diag(d), Q), Q / d[None, :], rtol=0, atol=1e-15)
    # unit lower bidiagonal with -1: L^T v = q  <=>  v_i = q_i + v_{i+1} (suffix sums)
    L = np.eye(9) - np.eye(9, k=-1)
    assert np.allclose(oracle.gen_back(L, Q), np.cumsum(Q[:, ::-1], axis=1)[:, ::-1], atol=1e-14)


def test_gen_back_solves_the_generalized_eigenproblem():
    """eig of Atilde = L^-1 A L^-T, back-transformed with gen_back, solves A V = B V Lambda with
    the eigenvalues scipy's generalized solver finds, and V is B-orthonormal; the eigenvectors
    of Atilde without the back-transformation do not."""
    n = 120
    A = dense_symmetric(n, 3)
    B = spd_matrix(n, 4)
    L = np.linalg.cholesky(B)
    At = solve_triangular(L, solve_triangular(L, A, lower=True).T, lower=True).T
    lam, Vt = np.linalg.eigh(0.5 * (At + At.T))
    V = oracle.gen_back(L, np.ascontiguousarray(Vt.T)).T
    res = np.linalg.norm(A @ V - B @ V * lam[None, :]) / (np.linalg.norm(A) * np.linalg.norm(V))
    assert res <= 1e-14
    assert np.allclose(lam, eigh(A, B, eigvals_only=True), rtol=0, atol=1e-12 * np.abs(lam).max())
    assert np.abs(V.T @ B @ V - np.eye(n)).max() <= 1e-12
    res_no = np.linalg.norm(A @ Vt - B @ Vt * lam[None, :]) / (np.linalg.norm(A) * np.linalg.norm(Vt))
    assert res_no > 1e-3


def test_generalized_two_stage_pipeline():
    """A V = B V Lambda solved end to end by the oracle's two-stage path (stage 1, chase,
    tridiagonal eig, both back-transforms, then gen_back), against scipy's generalized eigh."""
    n, nbw, nev = 96, 8, 40
    case = oracle.make_case_generalized(n, nbw, nev, 11)
    A, B, lam, V = case["A"], case["B"], case["lam"], case["V"][:, :n].T
    res = np.linalg.norm(A @ V - B @ V * lam[None, :]) / (np.linalg.norm(A) * np.linalg.norm(V))
    assert res <= 1e-13
    assert np.allclose(lam, eigh(A, B, eigvals_only=True)[:nev], rtol=0, atol=1e-11 * np.abs(lam).max())


def test_lower_triangular_recipe():
    n = 50
    Lcm = lower_triangular_cm_np(n, 0, n, 9, ldl=52)
    L = Lcm[:, :n].T
    assert np.array_equal(L, np.tril(L))
    assert np.all(np.diag(L) >= 1.0) and np.abs(np.tril(L, -1)).max() <= 1.0 / n
    assert np.linalg.cond(L) < 10
    part = lower_triangular_cm_np(n, 10, 20, 9, ldl=52)
    assert np.array_equal(part, Lcm[10:20])
