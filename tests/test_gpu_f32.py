"""GPU parity of the FP32 variant (elpa_trans_ev_tridi_to_band_f32) against
the CPU oracle.  Both sides take the SAME float32 inputs (reflectors and Q rounded to FP32 once);
the oracle applies them in fp64 (its plain definition), the kernel in FP32.

Tolerance (R14), ELEMENTWISE: every entry of a column passes through ~n/2 reflector
applications (R * nbw / n per row), each one a length-nbw dot product plus an update, so about
n*nbw/2 independent roundings of relative size u32 = 2^-24 reach it; they add like a random walk
(probabilistic rounding model), giving a per-entry standard deviation of u32 sqrt(n nbw / 2)
times the column's rms entry ||q_c||_2 / sqrt(n).  The test bar is
    max_{i,c} |dQ_ic| / (EXT * ||q_c||_2 / sqrt(n))  <=  8 u32 sqrt(max(n nbw / 2, 16)),
EXT = 7 the extreme-value factor of up to 1e10 Gaussian entries (sqrt(2 ln 1e10) = 6.8) and 8
the safety factor.  A single wrong entry of one column (an indexing bug) is caught at any n: the
per-entry allowance is 7/sqrt(n) of the column-norm allowance the first version used."""
import numpy as np
import pytest

import oracle
from inputs import config_seed, synthetic_q_np, synthetic_reflectors

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def bound(n, nbw):
    return 8.0 * U32 * np.sqrt(max(n * nbw / 2.0, 16.0))


EXT = 7.0


def colerr(got, want):
    """Elementwise error in units of EXT x the column's rms entry (see the module docstring)."""
    n = want.shape[1]
    rms = np.maximum(np.linalg.norm(want, axis=1), 1e-30) / np.sqrt(n)
    return float((np.abs(got - want).max(axis=1) / (EXT * rms)).max())


@pytest.fixture(scope="module")
def eb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import paper_1811_01277_b200 as m
    return m


def f32_case(n, nbw, nev, seed, ldq=None):
    ldq = (n + 3) // 4 * 4 if ldq is None else ldq     # the FP32 ABI requires ldq % 4 == 0
    s, L = oracle.schedule(n, nbw)
    hv, tau = synthetic_reflectors(len(s), nbw, seed)
    Q = synthetic_q_np(n, 0, nev, seed, ldq=ldq)
    hv32, tau32, Q32 = hv.astype(np.float32), tau.astype(np.float32), Q.astype(np.float32)
    want = oracle.apply(hv32.astype(np.float64), tau32.astype(np.float64), s, L, Q32.astype(np.float64))
    return hv32, tau32, Q32, want


def run32(eb, n, nbw, hv, tau, Q, opts=None):
    import torch
    dv = torch.from_numpy(np.ascontiguousarray(hv)).cuda()
    dt = torch.from_numpy(np.ascontiguousarray(tau)).cuda()
    dq = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    eb.trans_ev_tridi_to_band(n, nbw, dv, dt, dq, opts=opts)
    torch.cuda.synchronize()
    return dq.cpu().numpy()


SHAPES = [(1, 2, 1, 1), (2, 2, 1, 1), (1, 4, 1, 1), (2, 1, 1, 1), (4, 2, 1, 1), (1, 1, 2, 1), (1, 2, 2, 1),
          (2, 1, 2, 1), (1, 1, 1, 1), (1, 2, 1, 2), (2, 2, 1, 2), (2, 1, 1, 2)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("nbw", [8, 16, 32, 64])
def test_f32_all_shapes(eb, shape, nbw):
    D, CW, NC, K = shape
    n, nev = 301, 45                          # ragged: n odd, nev not a multiple of 32
    hv, tau, Q, want = f32_case(n, nbw, nev, nbw * 11 + D, ldq=304)
    tol = bound(n, nbw)
    for grid in (0, 1, 2, 3):
        got = run32(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_FFMA2, depth_warps=D, col_warps=CW,
                                                       tiles_per_warp=NC, grid_ctas=grid, groups_per_step=K))
        assert colerr(got[:, :n], want[:, :n]) <= tol, (shape, grid)
        assert np.array_equal(got[:, n:], Q[:, n:])      # ldq padding untouched


@pytest.mark.parametrize("shape,grid", [((1, 2, 1, 1), 0), ((1, 2, 1, 1), 5), ((2, 2, 1, 1), 0), ((4, 2, 1, 1), 7),
                                        ((1, 2, 2, 1), 0), ((2, 1, 2, 1), 3), ((2, 2, 1, 2), 0), ((2, 1, 1, 2), 5)])
def test_f32_multi_item_at_scale(eb, shape, grid):
    """many items per CTA, passes of one column block pipelining across CTAs"""
    D, CW, NC, K = shape
    n, nbw, nev = 2000, 64, 700
    hv, tau, Q, want = f32_case(n, nbw, nev, 41 + D * CW + NC)
    got = run32(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_FFMA2, depth_warps=D, col_warps=CW,
                                                   tiles_per_warp=NC, grid_ctas=grid, groups_per_step=K))
    assert colerr(got, want) <= bound(n, nbw)


@pytest.mark.parametrize("nbw", [24, 40, 56, 72, 96, 128])
def test_f32_nbw_range(eb, nbw):
    n, nev = 400, 70
    hv, tau, Q, want = f32_case(n, nbw, nev, 3 * nbw)
    for opts in (None, dict(kernel=eb.KERNEL_FFMA2, depth_warps=1, col_warps=2, tiles_per_warp=1)):
        got = run32(eb, n, nbw, hv, tau, Q, opts=opts)
        assert colerr(got[:, :n], want[:, :n]) <= bound(n, nbw), opts


@pytest.mark.parametrize("n,nbw,nev", [(4, 8, 1), (9, 8, 9), (10, 8, 3), (17, 16, 17), (64, 64, 64),
                                       (65, 64, 33), (130, 64, 129), (3, 8, 3)])
def test_f32_edge_sizes(eb, n, nbw, nev):
    hv, tau, Q, want = f32_case(n, nbw, nev, 7 * n + nbw)
    got = run32(eb, n, nbw, hv, tau, Q)
    assert colerr(got[:, :n], want[:, :n]) <= bound(n, nbw)


@pytest.mark.parametrize("n,nbw,nev", [(512, 16, 64), (37, 5, 9), (100, 7, 33), (64, 63, 10)])
def test_f32_reference_kernel(eb, n, nbw, nev):
    hv, tau, Q, want = f32_case(n, nbw, nev, 5 + n)
    got = run32(eb, n, nbw, hv, tau, Q, opts=dict(kernel=eb.KERNEL_REFERENCE))
    assert colerr(got[:, :n], want[:, :n]) <= bound(n, nbw)


def test_f32_real_C1(eb):
    """real eigenvectors (C1 chase + tridiagonal solve), rounded to FP32: parity with the
    oracle on the rounded inputs, and the eigen-residual at FP32 level"""
    case = oracle.make_case(512, 16, 512, config_seed(1))
    hv, tau, Qin = (case[k].astype(np.float32) for k in ("hh_v", "hh_tau", "Qin"))
    want = oracle.apply(hv.astype(np.float64), tau.astype(np.float64), case["s"], case["L"], Qin.astype(np.float64))
    got = run32(eb, 512, 16, hv, tau, Qin)
    assert colerr(got, want) <= bound(512, 16)
    assert oracle.residual(case["band"], got.astype(np.float64), case["lam"]) <= 1e-7


def test_f32_guard_bands(eb):
    """stray writes change a NaN guard; stray reads of a guard propagate NaN"""
    import torch
    n, nbw, nev = 301, 64, 45
    ldq = 308
    hv, tau, Q, want = f32_case(n, nbw, nev, 99, ldq=ldq)
    Q[:, n:] = np.nan
    G = 4096
    big = torch.full((G + nev * ldq + G,), float("nan"), dtype=torch.float32, device="cuda")
    big[G:G + nev * ldq] = torch.from_numpy(Q.reshape(-1)).cuda()
    dq = big[G:G + nev * ldq].view(nev, ldq)
    for opts in (None, dict(kernel=eb.KERNEL_FFMA2, depth_warps=4, col_warps=2, tiles_per_warp=1),
                 dict(kernel=eb.KERNEL_FFMA2, depth_warps=1, col_warps=2, tiles_per_warp=2),
                 dict(kernel=eb.KERNEL_FFMA2, depth_warps=2, col_warps=2, tiles_per_warp=1, groups_per_step=2)):
        dq.copy_(torch.from_numpy(Q).cuda())
        eb.trans_ev_tridi_to_band(n, nbw, torch.from_numpy(hv).cuda(), torch.from_numpy(tau).cuda(), dq, opts=opts)
        torch.cuda.synchronize()
        got = dq.cpu().numpy()
        assert np.isnan(big[:G].cpu().numpy()).all() and np.isnan(big[G + nev * ldq:].cpu().numpy()).all()
        assert np.isnan(got[:, n:]).all()
        assert colerr(got[:, :n], want[:, :n]) <= bound(n, nbw), opts


def test_f32_full_size_C3_sampled_columns(eb):
    """C3 (n = 20000, nbw = 64, nev = 20000) in FP32 with the default launch: the oracle
    recomputes 8 sampled columns from the same FP32 inputs (columns are independent)."""
    import torch
    from inputs import synthetic_q_torch, synthetic_reflectors_torch
    n, nbw, nev = 20000, 64, 20000
    seed = config_seed(3)
    R = eb.hh_count(n, nbw)
    dv, dt = synthetic_reflectors_torch(R, nbw, seed, device="cuda")
    dv32, dt32 = dv.float(), dt.float()
    del dv, dt
    dq = synthetic_q_torch(n, 0, nev, seed, device="cuda").float()
    eb.trans_ev_tridi_to_band(n, nbw, dv32, dt32, dq)
    torch.cuda.synchronize()
    cols = [0, 31, 32, 4999, 10000, 15000, 19968, 19999]
    got = dq[cols].cpu().numpy()
    s, L = oracle.schedule(n, nbw)
    Qs = np.concatenate([synthetic_q_np(n, c, c + 1, seed) for c in cols]).astype(np.float32)
    want = oracle.apply(dv32.cpu().numpy().astype(np.float64), dt32.cpu().numpy().astype(np.float64), s, L,
                        Qs.astype(np.float64))
    assert colerr(got, want) <= bound(n, nbw)
