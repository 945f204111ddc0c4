"""Pins of the complex Hermitian oracle (NEXT-3 second half, reflectors
Q_i = I - beta_i v_i v_i^H of P:117-121; R15).  Tied to: the real oracle on real
data, explicit dense reflector products, unitary similarity to the tridiagonal T, numpy's
Hermitian eigensolver, and the eigen-residual of the back-transformed eigenvectors."""
import numpy as np
import pytest

import oracle
from inputs import band_matrix, band_matrix_c, synthetic_reflectors_c, synthetic_q_c_np


def dense_H(n, v, tau, s, L):
    H = np.eye(n, dtype=np.complex128)
    vv = np.zeros(n, dtype=np.complex128)
    vv[s:s + L] = v[:L]
    vv[s] = 1.0
    return H - tau * np.outer(vv, vv.conj())


@pytest.mark.parametrize("n,nbw", [(12, 3), (40, 5), (33, 8)])
def test_complex_chase_on_real_data_equals_real_chase(n, nbw):
    band = band_matrix(n, nbw, 7)
    hv, tau, s, L, d, e = oracle.chase_c(band.astype(np.complex128))
    hv_r, tau_r, s_r, L_r, d_r, e_r = oracle.chase(band)
    assert np.array_equal(s, s_r) and np.array_equal(L, L_r)
    assert np.abs(hv.imag).max() == 0 and np.abs(tau.imag).max() == 0 and np.abs(e.imag).max() == 0
    assert np.allclose(hv.real, hv_r, rtol=0, atol=1e-13) and np.allclose(tau.real, tau_r, rtol=0, atol=1e-13)
    assert np.allclose(d, d_r, rtol=0, atol=1e-13) and np.allclose(e.real, e_r, rtol=0, atol=1e-13)


@pytest.mark.parametrize("n,nbw", [(10, 3), (24, 4), (31, 7)])
def test_complex_chase_is_a_unitary_similarity_to_T(n, nbw):
    band = band_matrix_c(n, nbw, 3 + n)
    hv, tau, s, L, d, e = oracle.chase_c(band)
    B = oracle.dense_from_band_c(band)
    P = np.eye(n, dtype=np.complex128)
    for r in range(len(s)):                               # P = H_0 H_1 ... H_{R-1}
        H = dense_H(n, hv[r], tau[r], s[r], L[r])
        assert np.abs(H.conj().T @ H - np.eye(n)).max() <= 1e-13     # each H unitary
        P = P @ H
    T = P.conj().T @ B @ P
    Tw = np.diag(d).astype(np.complex128) + np.diag(e, -1) + np.diag(e.conj(), 1)
    assert np.abs(T - Tw).max() <= 1e-12 * np.abs(B).max()
    assert np.abs(e[:-1].imag).max() == 0                  # zlarfg: real beta (R15)
    # apply_c reproduces the explicit product
    assert np.abs(oracle.apply_c(hv, tau, s, L, np.eye(n, dtype=np.complex128)).T - P).max() <= 1e-13


def test_complex_apply_matches_dense_products_synthetic():
    n, nbw, nev = 37, 5, 9
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors_c(len(s), nbw, 4)
    Q = synthetic_q_c_np(n, 0, nev, 4, ldq=40)
    got = oracle.apply_c(hv, tau, s, L, Q)
    P = np.eye(n, dtype=np.complex128)
    for r in range(len(s)):
        P = P @ dense_H(n, hv[r], tau[r], s[r], L[r])
    want = (P @ Q[:, :n].T).T
    assert np.abs(got[:, :n] - want).max() <= 1e-13 * np.abs(want).max()
    assert np.array_equal(got[:, n:], Q[:, n:])
    # full-length synthetic reflectors are unitary (tau = (1 + e^{i phi}) / ||v||^2 over all nbw
    # entries; truncated ones at the bottom are contractions, as in the real recipe)
    for r in range(len(s)):
        if L[r] == nbw:
            H = dense_H(n, hv[r], tau[r], s[r], L[r])
            assert np.abs(H.conj().T @ H - np.eye(n)).max() <= 1e-13
    # reversed order is a different operator (negative control)
    Prev = np.eye(n, dtype=np.complex128)
    for r in reversed(range(len(s))):
        Prev = Prev @ dense_H(n, hv[r], tau[r], s[r], L[r])
    assert np.abs((Prev @ Q[:, :n].T).T - want).max() > 1e-3


@pytest.mark.parametrize("n,nbw,nev", [(64, 4, 64), (200, 16, 50)])
def test_complex_eigenproblem_end_to_end(n, nbw, nev):
    case = oracle.make_case_c(n, nbw, nev, 5)
    B = oracle.dense_from_band_c(case["band"])
    assert np.allclose(case["lam"], np.linalg.eigvalsh(B)[:nev], rtol=0, atol=1e-12 * np.abs(case["lam"]).max())
    assert oracle.residual_c(case["band"], case["Qref"], case["lam"]) <= 1e-14
    X = case["Qref"][:, :n].T
    assert np.abs(X.conj().T @ X - np.eye(nev)).max() <= 1e-12
    # without the back-transformation the tridiagonal eigenvectors do not solve B
    assert oracle.residual_c(case["band"], case["Qin"], case["lam"]) > 1e-4


@pytest.mark.parametrize("n,b,nev", [(50, 4, 11), (130, 16, 30)])
def test_complex_residual_equals_dense_formula(n, b, nev):
    """oracle.residual_c equals ||B X - X Lambda||_F / (n ||B||_F) with an explicit dense
    Hermitian B written element by element (B[i, j] = band[i-j, j] below, its conjugate above),
    on random X and Lambda; counting each off-diagonal once in ||B||_F fails."""
    rng = np.random.default_rng(n)
    band = rng.uniform(-1, 1, (b + 1, n)) + 1j * rng.uniform(-1, 1, (b + 1, n))
    band[0] = band[0].real
    for dd in range(1, b + 1):
        band[dd, n - dd:] = 0.0
    Q = rng.uniform(-1, 1, (nev, n)) + 1j * rng.uniform(-1, 1, (nev, n))
    lam = rng.uniform(-2, 2, nev)
    B = np.zeros((n, n), dtype=np.complex128)
    for i in range(n):
        for j in range(max(0, i - b), i + 1):
            B[i, j] = band[i - j, j]
            B[j, i] = np.conj(band[i - j, j])
    X = Q.T
    num = np.linalg.norm(B @ X - X @ np.diag(lam), "fro")
    want = num / (n * np.linalg.norm(B, "fro"))
    got = oracle.residual_c(band, Q, lam)
    assert abs(got - want) <= 1e-13 * want
    once = num / (n * np.sqrt(np.sum(np.abs(band) ** 2)))
    assert abs(once - want) > 1e-3 * want
