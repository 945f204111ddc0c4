"""GPU parity of NEXT-4, the generalized back-transformation V = L^{-T} Vtilde (PAPER.md
P:136-139, Eq. 7; elpa_generalized_back_transform) against the CPU oracle's backward
substitution (oracle.gen_back), bar max|dV| / max|V| <= 1e-12 (north_star's parity bar)."""
import numpy as np
import pytest

import oracle
from inputs import lower_triangular_cm_np, synthetic_q_np

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def eb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import paper_1811_01277_b200 as m
    return m


def _rel(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def run_gen(eb, n, Lcm, Q):
    import torch
    dL = torch.from_numpy(np.ascontiguousarray(Lcm)).cuda()
    dq = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    eb.generalized_back_transform(n, dL, dq)
    torch.cuda.synchronize()
    return dq.cpu().numpy()


@pytest.mark.parametrize("n,nev", [(1, 1), (5, 3), (127, 40), (128, 128), (129, 7), (300, 300), (1000, 77)])
def test_gen_back_vs_oracle(eb, n, nev):
    ldl, ldq = n + 3, n + 5
    Lcm = lower_triangular_cm_np(n, 0, n, 100 + n, ldl=ldl)
    # Lcm[c, r] = L[r][c]: its strict lower triangle is L's strict upper one, never to be read
    Lcm[:, :n] += np.tril(np.full((n, n), np.nan), -1)
    Q = synthetic_q_np(n, 0, nev, 200 + n, ldq=ldq)
    Q[:, n:] = 7.0
    L = np.nan_to_num(Lcm[:, :n].T, nan=0.0)
    want = oracle.gen_back(L, Q)
    got = run_gen(eb, n, Lcm, Q)
    assert _rel(got[:, :n], want[:, :n]) <= TOL
    assert np.array_equal(got[:, n:], Q[:, n:])              # ldq padding untouched


def test_gen_back_generalized_pipeline(eb):
    """the oracle's whole generalized two-stage pipeline, with the last step on the GPU:
    A V = B V Lambda at the oracle's accuracy"""
    n, nbw, nev = 400, 16, 150
    case = oracle.make_case_generalized(n, nbw, nev, 21)
    Lcm = np.ascontiguousarray(case["L"].T)
    got = run_gen(eb, n, Lcm, case["Qt"])
    assert _rel(got, case["V"]) <= TOL
    A, B, lam = case["A"], case["B"], case["lam"]
    V = got[:, :n].T
    res = np.linalg.norm(A @ V - B @ V * lam[None, :]) / (np.linalg.norm(A) * np.linalg.norm(V))
    assert res <= 1e-13


def test_gen_back_full_size_sampled(eb):
    """C3-sized (n = nev = 20000): the oracle recomputes sampled columns"""
    import torch
    from inputs import lower_triangular_cm_torch, synthetic_q_torch
    n, nev = 20000, 20000
    dL = lower_triangular_cm_torch(n, 0, n, 5, device="cuda")
    dq = synthetic_q_torch(n, 0, nev, 6, device="cuda")
    eb.generalized_back_transform(n, dL, dq)
    torch.cuda.synchronize()
    cols = [0, 1, 9999, 19999]
    got = dq[cols].cpu().numpy()
    L = dL.cpu().numpy().T
    del dL
    Qs = np.concatenate([synthetic_q_np(n, c, c + 1, 6) for c in cols])
    want = oracle.gen_back(L, Qs)
    assert _rel(got, want) <= TOL
