"""paper_1811_01277_b200 — B200-native trans_ev_tridi_to_band (ELPA two-stage eigensolver,
arXiv 1811.01277).  Thin ctypes binding over the C-ABI library libelpa_b200.so
(include/elpa_b200.h): argument marshalling only — every step of the path runs in the
library's sm_100a kernels.  There is no CPU fallback: importing fails loudly if the
library cannot be loaded.

Tensors: Q is a float64 CUDA tensor of shape (nev, ldq) — the row-major view of the
column-major n x nev eigenvector block (row c = eigenvector c, first n entries used).
hh_v is (R, nbw) (== nbw x R column-major), hh_tau is (R,).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libelpa_b200.so")          # the in-tree build, nothing else

OK, ERR_ARG, ERR_NULL, ERR_ALIGN, ERR_DEVICE, ERR_CUDA, ERR_SPACE = 0, -1, -2, -3, -4, -5, -6
KERNEL_AUTO, KERNEL_REFERENCE, KERNEL_DMMA, KERNEL_DFMA, KERNEL_FFMA2 = 0, 1, 2, 3, 4


def _load():
    if not os.path.exists(_SO):
        from . import build as _build
        _build.build()
    lib = ctypes.CDLL(_SO)
    i64, p, i32, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.elpa_b200_release_cache.restype = i32
    lib.elpa_b200_release_cache.argtypes = []
    lib.elpa_b200_set_workspace_cache.restype = i32
    lib.elpa_b200_set_workspace_cache.argtypes = [i32]
    lib.elpa_hh_count.restype = i64
    lib.elpa_hh_count.argtypes = [i64, i64]
    lib.elpa_hh_offset.restype = i64
    lib.elpa_hh_offset.argtypes = [i64, i64, i64]
    lib.elpa_b200_prepare_sweeps.restype = i32
    lib.elpa_b200_prepare_sweeps.argtypes = [i64, i64, p, p, p, sz, i64, i64, p, p]
    lib.elpa_trans_ev_tridi_to_band.restype = i32
    lib.elpa_trans_ev_tridi_to_band.argtypes = [i64, i64, i64, p, p, p, i64, p]
    for f in (lib.elpa_trans_ev_tridi_to_band_ex, lib.elpa_trans_ev_tridi_to_band_host):
        f.restype = i32
        f.argtypes = [i64, i64, i64, p, p, p, i64, p, p]
    lib.elpa_generalized_back_transform.restype = i32
    lib.elpa_generalized_back_transform.argtypes = [i64, i64, p, i64, p, i64, p]
    lib.elpa_trans_ev_tridi_to_band_c64.restype = i32
    lib.elpa_trans_ev_tridi_to_band_c64.argtypes = [i64, i64, i64, p, p, p, i64, p, p]
    lib.elpa_b200_describe_c64.restype = i32
    lib.elpa_b200_describe_c64.argtypes = [i64, i64, i64, p, ctypes.c_char_p, sz]
    lib.elpa_trans_ev_tridi_to_band_f32.restype = i32
    lib.elpa_trans_ev_tridi_to_band_f32.argtypes = [i64, i64, i64, p, p, p, i64, p, p]
    lib.elpa_b200_describe_f32.restype = i32
    lib.elpa_b200_describe_f32.argtypes = [i64, i64, i64, p, ctypes.c_char_p, sz]
    lib.elpa_b200_workspace_bytes.restype = i64
    lib.elpa_b200_workspace_bytes.argtypes = [i64, i64, p]
    lib.elpa_b200_prepare.restype = i32
    lib.elpa_b200_prepare.argtypes = [i64, i64, p, p, p, sz, p, p]
    lib.elpa_b200_apply_prepared.restype = i32
    lib.elpa_b200_apply_prepared.argtypes = [i64, i64, i64, p, p, p, sz, p, i64, p, p]
    lib.elpa_b200_describe.restype = i32
    lib.elpa_b200_describe.argtypes = [i64, i64, i64, p, ctypes.c_char_p, sz]
    lib.elpa_b200_strerror.restype = ctypes.c_char_p
    lib.elpa_b200_strerror.argtypes = [i32]
    pi = ctypes.POINTER(ctypes.c_int)
    lib.elpa_b200_autotune_setup.restype = p
    lib.elpa_b200_autotune_setup.argtypes = [i64, i64, i64, i32, pi]
    lib.elpa_b200_autotune_step.restype = i32
    lib.elpa_b200_autotune_step.argtypes = [p, p]
    lib.elpa_b200_autotune_report.restype = i32
    lib.elpa_b200_autotune_report.argtypes = [p, ctypes.c_double]
    lib.elpa_b200_autotune_best.restype = i32
    lib.elpa_b200_autotune_best.argtypes = [p, p, ctypes.POINTER(ctypes.c_double)]
    lib.elpa_b200_autotune_progress.restype = i32
    lib.elpa_b200_autotune_progress.argtypes = [p, pi, pi]
    lib.elpa_b200_autotune_save.restype = i64
    lib.elpa_b200_autotune_save.argtypes = [p, ctypes.c_char_p, sz]
    lib.elpa_b200_autotune_load.restype = p
    lib.elpa_b200_autotune_load.argtypes = [ctypes.c_char_p, pi]
    lib.elpa_b200_autotune_destroy.restype = None
    lib.elpa_b200_autotune_destroy.argtypes = [p]
    lib.elpa_b2f_count.restype = i64
    lib.elpa_b2f_count.argtypes = [i64, i64]
    lib.elpa_trans_ev_band_to_full.restype = i32
    lib.elpa_trans_ev_band_to_full.argtypes = [i64, i64, i64, p, i64, p, p, i64, p]
    lib.elpa_b200_autotune_setup_dtype.restype = p
    lib.elpa_b200_autotune_setup_dtype.argtypes = [i64, i64, i64, i32, i32, pi]
    lib.elpa_b200_autotune_run_dtype.restype = i32
    lib.elpa_b200_autotune_run_dtype.argtypes = [i64, i64, i64, i32, p, p, p, i64, p, i32, i32, p,
                                                 ctypes.POINTER(ctypes.c_double)]
    lib.elpa_b200_autotune_run.restype = i32
    lib.elpa_b200_autotune_run.argtypes = [i64, i64, i64, p, p, p, i64, p, i32, i32, p, ctypes.POINTER(ctypes.c_double)]
    return lib


_lib = _load()
LIBRARY_PATH = _SO


class Opts(ctypes.Structure):
    """elpa_b200_opts (include/elpa_b200.h)."""
    _fields_ = [("kernel", ctypes.c_int), ("depth_warps", ctypes.c_int), ("col_warps", ctypes.c_int),
                ("tiles_per_warp", ctypes.c_int), ("grid_ctas", ctypes.c_int),
                ("groups_per_step", ctypes.c_int), ("fused_k", ctypes.c_int)]


class ElpaB200Error(RuntimeError):
    def __init__(self, code, where=""):
        self.code = code
        super().__init__(f"{where}: {code} ({strerror(code)})")


def strerror(code):
    return _lib.elpa_b200_strerror(int(code)).decode()


def release_cache():
    """Return the library's cached workspace memory to the device (elpa_b200_release_cache)."""
    _check(_lib.elpa_b200_release_cache(), "elpa_b200_release_cache")


def set_workspace_cache(enable):
    """Keep (True, the default) or return at every synchronisation (False) the library's freed
    workspace memory (elpa_b200_set_workspace_cache; a documented deviation)."""
    _check(_lib.elpa_b200_set_workspace_cache(1 if enable else 0), "elpa_b200_set_workspace_cache")


def hh_count(n, nbw):
    return int(_lib.elpa_hh_count(int(n), int(nbw)))


def _opts_ptr(opts):
    if opts is None:
        return None, None
    if isinstance(opts, dict):
        opts = Opts(**opts)
    return opts, ctypes.byref(opts)


def _stream_handle(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(rc, where):
    if rc != OK:
        raise ElpaB200Error(rc, where)


def _dev_ptr(t, name, dtype=None):
    import torch
    if t is None:
        return None
    dtype = dtype or torch.float64
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
        raise TypeError(f"{name} must be a {str(dtype).replace('torch.', '')} CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _q_ldq(Q):
    if Q.dim() != 2 or Q.stride(1) != 1:
        raise ValueError("Q must be a (nev, ldq) tensor with unit stride along ldq")
    return Q.shape[0], (Q.stride(0) if Q.shape[0] > 1 else Q.shape[1])


def trans_ev_tridi_to_band(n, nbw, hh_v, hh_tau, Q, stream=None, opts=None):
    """Q <- H_0 H_1 ... H_{R-1} Q in place on the GPU (elpa_trans_ev_tridi_to_band[_ex]).
    Asynchronous on `stream` (default: torch's current stream).  float32 tensors go to the
    FP32 variant (elpa_trans_ev_tridi_to_band_f32, NEXT-3), complex128 tensors to the complex
    Hermitian variant (elpa_trans_ev_tridi_to_band_c64); all three must share the dtype."""
    import torch
    nev, ldq = _q_ldq(Q)
    o, op = _opts_ptr(opts)
    s = _stream_handle(stream, Q.device)
    if isinstance(Q, torch.Tensor) and Q.dtype == torch.complex128:
        z = torch.complex128
        rc = _lib.elpa_trans_ev_tridi_to_band_c64(int(n), int(nbw), int(nev), _dev_ptr(hh_v, "hh_v", z),
                                                  _dev_ptr(hh_tau, "hh_tau", z), _dev_ptr(Q, "Q", z), int(ldq), s,
                                                  op)
        _check(rc, "elpa_trans_ev_tridi_to_band_c64")
        return Q
    if isinstance(Q, torch.Tensor) and Q.dtype == torch.float32:
        f = torch.float32
        rc = _lib.elpa_trans_ev_tridi_to_band_f32(int(n), int(nbw), int(nev), _dev_ptr(hh_v, "hh_v", f),
                                                  _dev_ptr(hh_tau, "hh_tau", f), _dev_ptr(Q, "Q", f), int(ldq), s,
                                                  op)
        _check(rc, "elpa_trans_ev_tridi_to_band_f32")
        return Q
    args = (int(n), int(nbw), int(nev), _dev_ptr(hh_v, "hh_v"), _dev_ptr(hh_tau, "hh_tau"),
            _dev_ptr(Q, "Q"), int(ldq), s)
    rc = _lib.elpa_trans_ev_tridi_to_band(*args) if op is None else \
        _lib.elpa_trans_ev_tridi_to_band_ex(*args, op)
    _check(rc, "elpa_trans_ev_tridi_to_band")
    return Q


def trans_ev_tridi_to_band_host(n, nbw, hh_v, hh_tau, Q, stream=None, opts=None):
    """Host-buffer entry point (elpa_trans_ev_tridi_to_band_host): hh_v, hh_tau, Q are CPU
    float64 tensors (pinned for speed); Q is updated in place; synchronises `stream`."""
    import torch
    for t, nm in ((hh_v, "hh_v"), (hh_tau, "hh_tau"), (Q, "Q")):
        if t.is_cuda or t.dtype != torch.float64 or not (t.is_contiguous() or t is Q):
            raise TypeError(f"{nm} must be a contiguous float64 CPU tensor")
    # Q: (nev, ldq) contiguous, or an (nev, n) view with row stride ldq (a buffer that ends at
    # element (nev-1)*ldq + n, as the header allows)
    nev, ldq = _q_ldq(Q)
    o, op = _opts_ptr(opts)
    s = _stream_handle(stream, torch.device("cuda", torch.cuda.current_device()))
    rc = _lib.elpa_trans_ev_tridi_to_band_host(int(n), int(nbw), int(nev), ctypes.c_void_p(hh_v.data_ptr()),
                                              ctypes.c_void_p(hh_tau.data_ptr()), ctypes.c_void_p(Q.data_ptr()),
                                              int(ldq), s, op)
    _check(rc, "elpa_trans_ev_tridi_to_band_host")
    return Q


def workspace_bytes(n, nbw, opts=None):
    o, op = _opts_ptr(opts)
    return int(_lib.elpa_b200_workspace_bytes(int(n), int(nbw), op))


def prepare(n, nbw, hh_v, hh_tau, workspace, stream=None, opts=None):
    """Prepare the reflectors into `workspace` (a CUDA uint8 tensor of workspace_bytes())."""
    o, op = _opts_ptr(opts)
    s = _stream_handle(stream, hh_v.device)
    wptr = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None and workspace.numel() else None
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = _lib.elpa_b200_prepare(int(n), int(nbw), _dev_ptr(hh_v, "hh_v"), _dev_ptr(hh_tau, "hh_tau"),
                                wptr, nbytes, s, op)
    _check(rc, "elpa_b200_prepare")


def hh_offset(n, nbw, j):
    """off(j): generation index of sweep j's first reflector (R for j >= n - 2)."""
    return int(_lib.elpa_hh_offset(int(n), int(nbw), int(j)))


def prepare_sweeps(n, nbw, hh_v, hh_tau, workspace, sweep_lo, sweep_hi, stream=None, opts=None):
    """Chunked preparation (elpa_b200_prepare_sweeps): the groups complete for sweeps < sweep_hi
    not yet complete for sweeps < sweep_lo."""
    o, op = _opts_ptr(opts)
    s = _stream_handle(stream, hh_v.device)
    wptr = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None and workspace.numel() else None
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = _lib.elpa_b200_prepare_sweeps(int(n), int(nbw), _dev_ptr(hh_v, "hh_v"), _dev_ptr(hh_tau, "hh_tau"), wptr,
                                       nbytes, int(sweep_lo), int(sweep_hi), s, op)
    _check(rc, "elpa_b200_prepare_sweeps")


def apply_prepared(n, nbw, workspace, Q, hh_v=None, hh_tau=None, stream=None, opts=None):
    nev, ldq = _q_ldq(Q)
    o, op = _opts_ptr(opts)
    s = _stream_handle(stream, Q.device)
    wptr = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None and workspace.numel() else None
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = _lib.elpa_b200_apply_prepared(int(n), int(nbw), int(nev), _dev_ptr(hh_v, "hh_v"),
                                       _dev_ptr(hh_tau, "hh_tau"), wptr, nbytes, _dev_ptr(Q, "Q"),
                                       int(ldq), s, op)
    _check(rc, "elpa_b200_apply_prepared")
    return Q


def generalized_back_transform(n, L, Q, stream=None):
    """V = L^{-T} Vtilde in place (elpa_generalized_back_transform, NEXT-4; Eq. 7).  L: float64
    CUDA tensor (n, ldl) = row-major view of the column-major lower-triangular factor (row i =
    column i of L); Q: (nev, ldq) as for trans_ev_tridi_to_band."""
    nev, ldq = _q_ldq(Q)
    if L.dim() != 2 or L.stride(1) != 1:
        raise ValueError("L must be an (n, ldl) tensor with unit stride along ldl")
    ldl = L.stride(0) if L.shape[0] > 1 else L.shape[1]
    s = _stream_handle(stream, Q.device)
    rc = _lib.elpa_generalized_back_transform(int(n), int(nev), _dev_ptr(L, "L"), int(ldl), _dev_ptr(Q, "Q"),
                                              int(ldq), s)
    _check(rc, "elpa_generalized_back_transform")
    return Q


def describe_c64(n, nbw, nev, opts=None):
    """(launches, description) of the complex entry point's plan (elpa_b200_describe_c64)."""
    o, op = _opts_ptr(opts)
    buf = ctypes.create_string_buffer(512)
    rc = _lib.elpa_b200_describe_c64(int(n), int(nbw), int(nev), op, buf, 512)
    if rc < 0:
        raise ElpaB200Error(rc, "elpa_b200_describe_c64")
    return rc, buf.value.decode()


def describe_f32(n, nbw, nev, opts=None):
    """(launches, description) of the FP32 entry point's plan (elpa_b200_describe_f32)."""
    o, op = _opts_ptr(opts)
    buf = ctypes.create_string_buffer(512)
    rc = _lib.elpa_b200_describe_f32(int(n), int(nbw), int(nev), op, buf, 512)
    if rc < 0:
        raise ElpaB200Error(rc, "elpa_b200_describe_f32")
    return rc, buf.value.decode()


def describe(n, nbw, nev, opts=None):
    """(number of kernel launches per call, launch description string)."""
    o, op = _opts_ptr(opts)
    buf = ctypes.create_string_buffer(256)
    rc = _lib.elpa_b200_describe(int(n), int(nbw), int(nev), op, buf, 256)
    if rc < 0:
        raise ElpaB200Error(rc, "elpa_b200_describe")
    return rc, buf.value.decode()


def credited_flops(n, nbw, nev):
    """North-star flop credit: 4 * nbw * nev per reflector (BASELINE.json metric)."""
    return 4.0 * nbw * nev * hh_count(n, nbw)


AUTOTUNE_FAST, AUTOTUNE_MEDIUM = 1, 2
DTYPE_F64, DTYPE_F32, DTYPE_C64 = 0, 1, 2


def opts_dict(o):
    return {f: getattr(o, f) for f, _ in Opts._fields_}


class Autotuner:
    """ELPA-style autotuning of the back-transformation's blocking parameters:

        at = Autotuner(n, nbw, nev, AUTOTUNE_MEDIUM)
        while (opts := at.step()) is not None:
            ... run one trans_ev_tridi_to_band(..., opts=opts), time it ...
            at.report(ms)
        best_opts, best_ms = at.best()

    save() / Autotuner.load(state) snapshot and resume the loop."""

    def __init__(self, n=None, nbw=None, nev=None, level=AUTOTUNE_FAST, _handle=None, dtype=DTYPE_F64):
        if _handle is None:
            err = ctypes.c_int(0)
            _handle = _lib.elpa_b200_autotune_setup_dtype(int(n), int(nbw), int(nev), int(level), int(dtype),
                                                          ctypes.byref(err))
            if not _handle:
                raise ElpaB200Error(err.value, "elpa_b200_autotune_setup_dtype")
        self._h = ctypes.c_void_p(_handle)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.elpa_b200_autotune_destroy(self._h)
            self._h = None

    def step(self):
        o = Opts()
        rc = _lib.elpa_b200_autotune_step(self._h, ctypes.byref(o))
        if rc < 0:
            raise ElpaB200Error(rc, "elpa_b200_autotune_step")
        return opts_dict(o) if rc == 1 else None

    def report(self, ms):
        _check(_lib.elpa_b200_autotune_report(self._h, float(ms)), "elpa_b200_autotune_report")

    def best(self):
        o, ms = Opts(), ctypes.c_double(0)
        _check(_lib.elpa_b200_autotune_best(self._h, ctypes.byref(o), ctypes.byref(ms)), "elpa_b200_autotune_best")
        return opts_dict(o), ms.value

    def progress(self):
        a, b = ctypes.c_int(0), ctypes.c_int(0)
        _check(_lib.elpa_b200_autotune_progress(self._h, ctypes.byref(a), ctypes.byref(b)), "progress")
        return a.value, b.value

    def save(self):
        need = _lib.elpa_b200_autotune_save(self._h, None, 0)
        buf = ctypes.create_string_buffer(int(need))
        _lib.elpa_b200_autotune_save(self._h, buf, int(need))
        return buf.value.decode()

    @classmethod
    def load(cls, state):
        err = ctypes.c_int(0)
        h = _lib.elpa_b200_autotune_load(state.encode(), ctypes.byref(err))
        if not h:
            raise ElpaB200Error(err.value or ERR_ARG, "elpa_b200_autotune_load")
        return cls(_handle=h)


def autotune(n, nbw, hh_v, hh_tau, Q_scratch, level=AUTOTUNE_MEDIUM, reps=2, stream=None):
    """Run the autotuning loop on device buffers (elpa_b200_autotune_run[_dtype]); Q_scratch is
    overwritten.  The element type follows Q_scratch (float64, float32 or complex128).  Returns
    (best opts dict, best time in ms: the apply for float64, the whole call otherwise)."""
    import torch
    nev, ldq = _q_ldq(Q_scratch)
    o, ms = Opts(), ctypes.c_double(0)
    s = _stream_handle(stream, Q_scratch.device)
    dt = {torch.float64: DTYPE_F64, torch.float32: DTYPE_F32, torch.complex128: DTYPE_C64}.get(Q_scratch.dtype)
    if dt is None:
        raise TypeError("Q_scratch must be float64, float32 or complex128")
    tdt = Q_scratch.dtype
    rc = _lib.elpa_b200_autotune_run_dtype(int(n), int(nbw), int(nev), dt, _dev_ptr(hh_v, "hh_v", tdt),
                                           _dev_ptr(hh_tau, "hh_tau", tdt), _dev_ptr(Q_scratch, "Q", tdt), int(ldq), s,
                                           int(level), int(reps), ctypes.byref(o), ctypes.byref(ms))
    _check(rc, "elpa_b200_autotune_run_dtype")
    return opts_dict(o), ms.value


def b2f_count(n, nbw):
    """K = number of stage-1 reflectors of an n x n matrix reduced to half-bandwidth nbw."""
    return int(_lib.elpa_b2f_count(int(n), int(nbw)))


def trans_ev_band_to_full(n, nbw, hh1_v, hh1_tau, Q, stream=None):
    """NEXT-1: Q <- H_0 ... H_{K-1} Q with the stage-1 (full -> band) reflectors
    (elpa_trans_ev_band_to_full).  hh1_v: (K, ldv) float64 CUDA tensor (row j = reflector j's
    length-n column, the element at j + nbw treated as 1, earlier ones ignored); hh1_tau: (K,)."""
    nev, ldq = _q_ldq(Q)
    if hh1_v.dim() != 2 or hh1_v.stride(1) != 1:
        raise ValueError("hh1_v must be a (K, ldv) tensor with unit inner stride")
    ldv = hh1_v.stride(0) if hh1_v.shape[0] > 1 else max(hh1_v.shape[1], int(n))
    s = _stream_handle(stream, Q.device)
    rc = _lib.elpa_trans_ev_band_to_full(int(n), int(nbw), int(nev), _dev_ptr(hh1_v, "hh1_v"), int(ldv),
                                         _dev_ptr(hh1_tau, "hh1_tau"), _dev_ptr(Q, "Q"), int(ldq), s)
    _check(rc, "elpa_trans_ev_band_to_full")
    return Q
