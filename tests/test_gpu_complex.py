"""GPU parity of the complex Hermitian variant (NEXT-3 second half, R15;
elpa_trans_ev_tridi_to_band_c64) against the CPU oracle (oracle.apply_c).  Bar as for FP64:
max|dQ| / max|Q| <= 1e-12; the REFERENCE kernel is bitwise the oracle."""
import numpy as np
import pytest

import oracle
from inputs import config_seed, synthetic_q_c_np, synthetic_reflectors_c

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


def zcase(n, nbw, nev, seed, ldq=None):
    ldq = n if ldq is None else ldq
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors_c(len(s), nbw, seed)
    Q = synthetic_q_c_np(n, 0, nev, seed, ldq=ldq)
    return hv, tau, s, L, Q


def runz(eb, n, nbw, hv, tau, Q, opts=None):
    import torch
    dv = torch.from_numpy(np.ascontiguousarray(hv)).cuda()
    dt = torch.from_numpy(np.ascontiguousarray(tau)).cuda()
    dq = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    eb.trans_ev_tridi_to_band(n, nbw, dv, dt, dq, opts=opts)
    torch.cuda.synchronize()
    return dq.cpu().numpy()


@pytest.mark.parametrize("n,nbw,nev", [(64, 8, 16), (37, 5, 9), (100, 7, 33), (3, 2, 3)])
def test_complex_reference_kernel_bitwise(eb, n, nbw, nev):
    hv, tau, s, L, Q = zcase(n, nbw, nev, 3 + n, ldq=n + 1)
    want = oracle.apply_c(hv, tau, s, L, Q)
    got = runz(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_REFERENCE))
    assert np.array_equal(got, want)


SHAPES = [(1, 2, 2), (2, 2, 1), (1, 2, 1), (2, 1, 2), (1, 4, 1), (2, 2, 2), (1, 1, 2)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("nbw", [8, 16, 32, 64])
def test_complex_dmma_all_shapes(eb, shape, nbw):
    D, CW, NZ = shape
    n, nev = 301, 45
    hv, tau, s, L, Q = zcase(n, nbw, nev, nbw * 5 + D, ldq=303)
    want = oracle.apply_c(hv, tau, s, L, Q)
    for grid in (0, 1, 3):
        got = runz(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_DMMA, depth_warps=D, col_warps=CW,
                                                      tiles_per_warp=NZ, grid_ctas=grid))
        assert _rel(got[:, :n], want[:, :n]) <= TOL, (shape, grid)
        assert np.array_equal(got[:, n:], Q[:, n:])


KWIN_SHAPES = [(4, 1, 2), (2, 1, 2), (8, 1, 2)]


@pytest.mark.parametrize("shape", KWIN_SHAPES)
@pytest.mark.parametrize("nbw", [32, 64])
def test_complex_kwin_shapes(eb, shape, nbw):
    """The K-group register-window kernel on complex tiles (KIND_ZMMA): D = 1, two groups per
    step; grids of 1 and 3 CTAs exercise the per-warp progress words across items."""
    CW, NZ, K = shape
    for n, nev in ((301, 45), (130, 129), (17, 17)):
        hv, tau, s, L, Q = zcase(n, nbw, nev, nbw * 7 + CW + n, ldq=n + 2)
        want = oracle.apply_c(hv, tau, s, L, Q)
        for grid in (0, 1, 3):
            got = runz(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_DMMA, depth_warps=1, col_warps=CW,
                                                          tiles_per_warp=NZ, grid_ctas=grid, groups_per_step=K))
            assert _rel(got[:, :n], want[:, :n]) <= TOL, (shape, n, grid)
            assert np.array_equal(got[:, n:], Q[:, n:])


def test_complex_kwin_rejects_unsupported(eb):
    n, nbw, nev = 100, 16, 10
    hv, tau, s, L, Q = zcase(n, nbw, nev, 3)
    with pytest.raises(eb.ElpaB200Error):
        runz(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_DMMA, depth_warps=1, col_warps=4, tiles_per_warp=1,
                                               groups_per_step=2))


@pytest.mark.parametrize("nbw", [24, 40, 72, 128])
def test_complex_nbw_range(eb, nbw):
    n, nev = 400, 50
    hv, tau, s, L, Q = zcase(n, nbw, nev, 9 * nbw)
    want = oracle.apply_c(hv, tau, s, L, Q)
    assert _rel(runz(eb, n, nbw, hv, tau, Q), want) <= TOL


@pytest.mark.parametrize("n,nbw,nev", [(4, 8, 1), (9, 8, 9), (17, 16, 17), (65, 64, 33), (130, 64, 129)])
def test_complex_edge_sizes(eb, n, nbw, nev):
    hv, tau, s, L, Q = zcase(n, nbw, nev, 7 * n)
    want = oracle.apply_c(hv, tau, s, L, Q)
    assert _rel(runz(eb, n, nbw, hv, tau, Q), want) <= TOL


def test_complex_real_eigenproblem(eb):
    """a real complex Hermitian case (chase + phase-scaled tridiagonal eig): parity and the
    eigen-residual of the GPU result"""
    case = oracle.make_case_c(512, 16, 256, config_seed(1))
    got = runz(eb, 512, 16, case["hh_v"], case["hh_tau"], case["Qin"])
    assert _rel(got, case["Qref"]) <= TOL
    assert oracle.residual_c(case["band"], got, case["lam"]) <= 1e-13


def test_complex_guard_bands(eb):
    import torch
    n, nbw, nev = 301, 64, 45
    ldq = 305
    hv, tau, s, L, Q = zcase(n, nbw, nev, 55, ldq=ldq)
    Q[:, n:] = np.nan
    want = oracle.apply_c(hv, tau, s, L, Q[:, :n].copy())
    G = 2048
    big = torch.full((G + nev * ldq + G,), complex(float("nan"), float("nan")), dtype=torch.complex128, device="cuda")
    big[G:G + nev * ldq] = torch.from_numpy(Q.reshape(-1)).cuda()
    dq = big[G:G + nev * ldq].view(nev, ldq)
    for opts in (None, dict(kernel=eb.KERNEL_DMMA, depth_warps=2, col_warps=2, tiles_per_warp=1),
                 dict(kernel=eb.KERNEL_DMMA, depth_warps=1, col_warps=4, tiles_per_warp=1, groups_per_step=2)):
        dq.copy_(torch.from_numpy(Q).cuda())
        eb.trans_ev_tridi_to_band(n, nbw, torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda(), dq, opts=opts)
        torch.cuda.synchronize()
        got = dq.cpu().numpy()
        assert np.isnan(big[:G].cpu().numpy()).all() and np.isnan(big[G + nev * ldq:].cpu().numpy()).all()
        assert np.isnan(got[:, n:]).all()
        assert _rel(got[:, :n], want) <= TOL


def test_complex_full_size_C3_sampled(eb):
    """n = 20000, nbw = 64, nev = 20000 complex with the default launch; sampled columns"""
    import torch
    n, nbw, nev = 20000, 64, 20000
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors_c(len(s), nbw, config_seed(3))
    dq = torch.empty((nev, n), dtype=torch.complex128, device="cuda")
    for a in range(0, nev, 2000):
        dq[a:a + 2000] = torch.from_numpy(synthetic_q_c_np(n, a, min(nev, a + 2000), 8)).cuda()
    eb.trans_ev_tridi_to_band(n, nbw, torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda(), dq)
    torch.cuda.synchronize()
    cols = [0, 7, 8, 10000, 19999]
    got = dq[cols].cpu().numpy()
    Qs = np.concatenate([synthetic_q_c_np(n, c, c + 1, 8) for c in cols])
    want = oracle.apply_c(hv, tau, s, L, Qs)
    assert _rel(got, want) <= TOL
