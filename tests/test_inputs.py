"""Input generators: splitmix64 reference values, numpy == torch bitwise, recipes."""
import numpy as np
import torch

from inputs import (splitmix64_np, uniform_pm1_np, uniform_pm1_torch, band_matrix,
                    synthetic_reflectors, synthetic_q_np, synthetic_q_torch)


def test_splitmix64_reference_vector():
    # splitmix64 from state 1234567: the widely published first five outputs
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    got = splitmix64_np(1234567, np.arange(5, dtype=np.uint64))
    assert [int(x) for x in got] == want


def test_numpy_torch_bitwise():
    cnt = np.arange(0, 100000, 7, dtype=np.uint64)
    a = uniform_pm1_np(0xDEADBEEF, cnt)
    b = uniform_pm1_torch(0xDEADBEEF, torch.from_numpy(cnt.astype(np.int64))).numpy()
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    q1 = synthetic_q_np(37, 3, 11, 5, ldq=40)
    q2 = synthetic_q_torch(37, 3, 11, 5, ldq=40, chunk_cols=3).numpy()
    assert np.array_equal(q1, q2)


def test_band_matrix_recipe():
    n, b = 10, 3
    band = band_matrix(n, b, 42)
    # draw order: column c ascending, then d ascending, skipping c+d >= n
    flat = uniform_pm1_np(42, np.arange(40, dtype=np.uint64))
    t = 0
    for c in range(n):
        for d in range(b + 1):
            if c + d < n:
                assert band[d, c] == flat[t]
                t += 1
            else:
                assert band[d, c] == 0.0


def test_synthetic_reflectors_recipe():
    v, tau = synthetic_reflectors(50, 8, 3)
    assert np.all(v[:, 0] == 1.0)
    assert np.allclose(tau * np.sum(v * v, axis=1), 2.0)
    q = synthetic_q_np(20, 0, 6, 1)
    assert np.array_equal(q[2:4], synthetic_q_np(20, 2, 4, 1))


def test_synthetic_reflectors_torch_bitwise():
    from inputs import synthetic_reflectors_torch
    v, tau = synthetic_reflectors(123, 16, 9)
    vt, taut = synthetic_reflectors_torch(123, 16, 9, chunk=50)
    assert np.array_equal(v, vt.numpy())
    # tau = 2/||v||^2: same value up to the summation order of the norm
    assert np.allclose(tau, taut.numpy(), rtol=1e-15, atol=0)


def test_lower_triangular_torch_matches_numpy():
    import torch
    from inputs import lower_triangular_cm_np, lower_triangular_cm_torch
    a = lower_triangular_cm_np(37, 3, 30, 77, ldl=40)
    b = lower_triangular_cm_torch(37, 3, 30, 77, ldl=40, chunk_cols=5).numpy()
    assert np.array_equal(a, b)
