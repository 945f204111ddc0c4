/*
 * elpa_b200.h — B200-native stage-2 eigenvector back-transformation of ELPA's two-stage
 * symmetric eigensolver (trans_ev_tridi_to_band), FP64, sm_100a only.
 *
 * What it computes (PAPER.md = arXiv 1811.01277 source; "P:L" = line L):
 *   The two-stage solver reduces a symmetric matrix to band form, then the band matrix B
 *   (half-bandwidth nbw) to tridiagonal T with Householder reflectors
 *   Q_i = I - beta_i v_i v_i^H that are "never constructed explicitly, but are always
 *   represented only by the Householder vector v_i" (Sec. 2 after Eq. 4;
 *   two-stage: P:141-144).  The eigenvectors Vhat of T (Eq. 5) must be
 *   back-transformed, Vtilde = Q^H Vhat (Eq. 6), and in the two-stage path
 *   "each eigenvector" is transformed twice.  This library performs the
 *   first of those two transforms — band <- tridiagonal — for nev eigenvectors:
 *
 *       Q  <-  H_0 H_1 ... H_{R-1} Q ,   H_r = I - tau_r v_r v_r^T   (H_{R-1} applied first)
 *
 *   Reflector r = (j, m) is the m-th reflector of chase sweep j (the sweep that
 *   eliminates column j), numbered in generation order (j ascending, then m ascending):
 *       first row   s = j + 1 + m*nbw        (0-based),
 *       length      L = min(nbw, n - s)      (it exists iff L >= 2),
 *       index       r(j,m) = off(j) + m,  off(j) = j + F(n-3) - F(n-3-j),
 *       F(x) = sum_{t=0}^{x} floor(t/nbw),  R = (n-2) + F(n-3)   (0 if n < 3 or nbw < 2).
 *   The reading of the chase, order and storage conventions is DESIGN.md §2 (R1-R12).
 *
 * Conventions shared by every entry point below
 *   hh_v   : nbw x R column-major (column r = reflector r's vector, contiguous, nbw doubles).
 *            Element 0 is treated as 1.0 (LAPACK v_0 = 1; SPEC S:196 — so buffers that keep
 *            tau in v_0 are accepted); elements >= L are never read.
 *   hh_tau : R doubles.  tau == 0 is the identity.
 *   Q      : n x nev column-major with leading dimension ldq (eigenvector c = column c).
 *            In: eigenvectors of T.  Out: eigenvectors of B (same eigenvalues).  Updated
 *            in place; rows [n, ldq) of every column are never written.
 *   Ownership: the caller owns every buffer.  The library keeps no problem state between calls.
 *            The one-shot entry points take temporary device workspace, stream-ordered on
 *            `stream`, from the library's own per-device memory pool, which keeps freed memory
 *            cached for the next call (elpa_b200_release_cache returns it to the device).
 *   Concurrency: calls on distinct streams with distinct buffers may run concurrently (the
 *            analogue of ELPA's multiple instances).  No host synchronisation
 *            happens inside the device-pointer entry points.
 *   Errors: integer codes (the analogue of ELPA's `int *error` out-parameter).
 *            Validation happens before any device work, in the order of the table in
 *            DESIGN.md §4; a kernel fault surfaces at the caller's next synchronisation.
 *            There is no CPU fallback and no slow path for misaligned Q.
 */
#ifndef ELPA_B200_H
#define ELPA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without including cuda_runtime.h (ABI: a CUstream handle, 0 = legacy default) */
typedef struct CUstream_st *elpa_b200_stream_t;

enum {
    ELPA_B200_OK = 0,
    ELPA_B200_ERR_ARG = -1,    /* n < 0 or n > 2^31 - 64, nbw < 1, nev < 0, nev > n, ldq < max(1,n),
                                  bad opts */
    ELPA_B200_ERR_NULL = -2,   /* a required pointer is NULL (R > 0 and nev > 0) */
    ELPA_B200_ERR_ALIGN = -3,  /* Q not 16-byte aligned, ldq odd (FP64) / not a multiple of 4 (FP32);
                                  workspace not 256-byte aligned */
    ELPA_B200_ERR_DEVICE = -4, /* current device is not compute capability 10.0 (B200, sm_100a) */
    ELPA_B200_ERR_CUDA = -5,   /* a CUDA runtime call or kernel launch failed */
    ELPA_B200_ERR_SPACE = -6   /* workspace smaller than elpa_b200_workspace_bytes() */
};

/* Kernel variants (elpa_b200_opts.kernel). */
enum {
    ELPA_B200_KERNEL_AUTO = 0,
    ELPA_B200_KERNEL_REFERENCE = 1, /* one thread per column, exact reverse generation order,
                                       no FMA contraction: bitwise equal to the CPU oracle */
    ELPA_B200_KERNEL_DMMA = 2,      /* k = 8 compact-WY groups on FP64 tensor cores (DMMA),
                                       depth-pipelined row windows; nbw % 8 == 0, nbw <= 128
                                       (AUTO picks it then, else REFERENCE) */
    ELPA_B200_KERNEL_DFMA = 3,      /* FP64 CUDA cores: a lane owns a column, k = fused_k
                                       reflectors applied in sequence to a register window of
                                       nbw + k rows (north_star item 3's design); nbw 8/16/32/64;
                                       the measured alternative to DMMA */
    ELPA_B200_KERNEL_FFMA2 = 4      /* FP32 entry point only: packed FP32 FMA (f32x2) kernel,
                                       same schedule; nbw % 8 == 0, nbw <= 128 */
};

/* Optional tuning knobs (the paper's "numerical blocking parameters of the
 * back-transformation").  Zero-initialise for automatic choices. */
typedef struct {
    int kernel;          /* ELPA_B200_KERNEL_* */
    int depth_warps;     /* D: chase depths pipelined per work item (1,2,4,8), 0 = auto */
    int col_warps;       /* CW: warps splitting a work item's column stripe, 0 = auto */
    int tiles_per_warp;  /* NCT: 8-column tiles per warp (1,2,4); an item has CW*NCT tiles */
    int grid_ctas;       /* persistent CTAs to launch, 0 = all co-resident (148 x occupancy) */
    int groups_per_step; /* K: reflector groups (of 8) per step, 0 = auto.  DMMA kernel: K = 1 runs
                            the per-group window (D, CW, NCT from the K = 1 menu); K >= 2 runs the
                            K-group register window (one depth per item, D = 1; nbw 32 or 64;
                            (D,CW,NCT,K) in (1,2,2,2) (1,4,2,2) (1,4,1,4) (1,4,1,2) (1,6,2,2)
                            (1,8,2,2) (1,3,2,2) (1,4,2,3) (1,8,1,2)), the automatic choice at
                            nbw = 64 (DESIGN.md §5.3 K2b, §6); other combinations: ERR_ARG */
    int fused_k;         /* DFMA kernel only: reflectors fused per group, k = 2, 4, 6 or 8 (0 = 8);
                            must be 0 for the other kernels */
} elpa_b200_opts;

/* Return the memory the library's per-device pool caches between calls (temporary workspaces)
 * to the device.  Call with no library work in flight on the current device.  OK or ERR_CUDA.
 * Deviation from the no-persistent-allocation rule of SURVEY §8(b), on by default: the pool keeps
 * freed workspace mapped so the next call does not re-map several GB (measured at C3: e2e
 * 18.8 -> 24.6 TFLOP/s).  elpa_b200_set_workspace_cache(0) switches the current
 * device's pool to release freed memory at every synchronisation (nothing outlives a call) and
 * trims it now; (1) restores caching.  OK or ERR_CUDA. */
int elpa_b200_release_cache(void);
int elpa_b200_set_workspace_cache(int enable);

/* R(n, nbw): number of reflectors the band->tridiagonal chase produces.
 * 0 if n < 3 or nbw == 1 (nbw = 1: the input is already tridiagonal);
 * -1 if n < 0 or nbw < 1. */
int64_t elpa_hh_count(int64_t n, int64_t nbw);

/* off(j): generation index of the first reflector of sweep j (the reflectors of sweeps < j are
 * rows [0, off(j)) of hh_v); R for j >= n - 2, 0 when R == 0; -1 on bad arguments. */
int64_t elpa_hh_offset(int64_t n, int64_t nbw, int64_t j);

/* One-shot device call: Q <- H_0 ... H_{R-1} Q, asynchronous on `stream`.
 * hh_v, hh_tau, Q are device pointers.  Returns ELPA_B200_OK or a negative code.
 * nev == 0 or R == 0 returns OK without touching memory. */
int elpa_trans_ev_tridi_to_band(int64_t n, int64_t nbw, int64_t nev,
                                const double *hh_v, const double *hh_tau,
                                double *Q, int64_t ldq, elpa_b200_stream_t stream);

/* Same, with tuning options (opts may be NULL = all automatic). */
int elpa_trans_ev_tridi_to_band_ex(int64_t n, int64_t nbw, int64_t nev,
                                   const double *hh_v, const double *hh_tau,
                                   double *Q, int64_t ldq, elpa_b200_stream_t stream,
                                   const elpa_b200_opts *opts);

/* Host-buffer call (end-to-end path): hh_v, hh_tau, Q are HOST pointers (pinned memory is
 * needed for copy/compute overlap).  Copies the reflectors to a temporary device workspace on
 * `stream` and prepares them, then streams Q through the GPU in ~6 column blocks (H2D, apply,
 * D2H on two internal copy streams, overlapped with the kernel), and synchronises before
 * returning.  The result is bitwise that of the device-pointer call. */
int elpa_trans_ev_tridi_to_band_host(int64_t n, int64_t nbw, int64_t nev,
                                     const double *hh_v, const double *hh_tau,
                                     double *Q, int64_t ldq, elpa_b200_stream_t stream,
                                     const elpa_b200_opts *opts);

/* Two-phase use (prepare the reflectors once, apply them to many eigenvector blocks):
 * elpa_b200_workspace_bytes  -> bytes of device workspace for the prepared reflectors
 *                               (0 when the chosen kernel needs none); -1 on bad args.
 * elpa_b200_prepare          -> re-lays hh_v/hh_tau into per-group tensor-core fragments
 *                               plus the k x k compact-WY factor of every group.
 * elpa_b200_apply_prepared   -> Q <- H_0 ... H_{R-1} Q from the prepared workspace (the
 *                               REFERENCE kernel reads hh_v/hh_tau directly; pass them). */
int64_t elpa_b200_workspace_bytes(int64_t n, int64_t nbw, const elpa_b200_opts *opts);
int elpa_b200_prepare(int64_t n, int64_t nbw, const double *hh_v, const double *hh_tau,
                      void *workspace, size_t workspace_bytes, elpa_b200_stream_t stream,
                      const elpa_b200_opts *opts);
/* Chunked preparation (the multi-GPU path prepares while the broadcast of later reflectors is
 * still in flight): prepares the reflector groups that are complete once the reflectors of every
 * sweep j < sweep_hi are in hh_v/hh_tau and that were not complete for sweeps j < sweep_lo
 * (sweep_lo = 0 on the first call).  A sequence of calls with sweep_lo = the previous sweep_hi,
 * the last with sweep_hi >= n - 2, prepares the workspace exactly as elpa_b200_prepare does.
 * Sweep j's reflectors are rows [off(j), off(j) + M_j) of hh_v: contiguous in generation order.
 * ERR_ARG also when sweep_lo < 0 or sweep_hi < sweep_lo. */
int elpa_b200_prepare_sweeps(int64_t n, int64_t nbw, const double *hh_v, const double *hh_tau,
                             void *workspace, size_t workspace_bytes, int64_t sweep_lo, int64_t sweep_hi,
                             elpa_b200_stream_t stream, const elpa_b200_opts *opts);
/* opts.kernel and n, nbw must be the ones the workspace was prepared with: a workspace this
 * process prepared for another kernel, n or nbw is rejected with ELPA_B200_ERR_ARG (the library
 * remembers the last 256 prepared workspace pointers; others are not checked). */
int elpa_b200_apply_prepared(int64_t n, int64_t nbw, int64_t nev,
                             const double *hh_v, const double *hh_tau,
                             const void *workspace, size_t workspace_bytes,
                             double *Q, int64_t ldq, elpa_b200_stream_t stream,
                             const elpa_b200_opts *opts);

/* Describe the launch the library would make for (n, nbw, nev, opts): writes
 * "kernel=... D=.. CW=.. NCT=.. K=.. items=.. grid_req=.. block=.. smem=.. ws=.." into buf.
 * Returns the number of kernel launches one elpa_trans_ev_tridi_to_band call makes, or a
 * negative code. */
int elpa_b200_describe(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts,
                       char *buf, size_t buflen);

/* ---------------------------------------------------------------------------------------
 * Autotuning of the back-transformation's blocking parameters.
 * Mirrors ELPA's autotuning API: set up with a level, step through candidates
 * (each used for one call whose time the caller reports), pick the best, snapshot/resume.
 *   FAST: the kernel variant only (DMMA, DFMA, and the reference kernel for
 *          small problems), each with its automatic shape;
 *   MEDIUM ("numerical blocking parameters of the back-transformation"):
 *          FAST plus every compiled DMMA shape (D, CW, NCT) for this nbw.
 * The object is host state only; it never touches the device.
 * ------------------------------------------------------------------------------------- */
typedef struct elpa_b200_autotune elpa_b200_autotune;
enum { ELPA_B200_AUTOTUNE_FAST = 1, ELPA_B200_AUTOTUNE_MEDIUM = 2 };

/* NULL on bad arguments (*error = ELPA_B200_ERR_ARG) */
elpa_b200_autotune *elpa_b200_autotune_setup(int64_t n, int64_t nbw, int64_t nev, int level, int *error);
/* 1 and the next candidate in *opts while candidates remain, 0 when all were tried, <0 error */
int elpa_b200_autotune_step(elpa_b200_autotune *at, elpa_b200_opts *opts);
/* time (ms, > 0) of the candidate the last _step returned */
int elpa_b200_autotune_report(elpa_b200_autotune *at, double ms);
/* best candidate reported so far (ELPA_B200_ERR_ARG if none) */
int elpa_b200_autotune_best(const elpa_b200_autotune *at, elpa_b200_opts *opts, double *ms);
/* number of candidates, and how many were reported */
int elpa_b200_autotune_progress(const elpa_b200_autotune *at, int *tried, int *total);
/* snapshot: writes a text state into buf; returns its length (incl. NUL) or the
 * size needed when buflen is too small; resume with _load */
int64_t elpa_b200_autotune_save(const elpa_b200_autotune *at, char *buf, size_t buflen);
elpa_b200_autotune *elpa_b200_autotune_load(const char *state, int *error);
void elpa_b200_autotune_destroy(elpa_b200_autotune *at);
/* The same tuning for the NEXT-3 variants (element type ELPA_B200_DTYPE_*).  FAST: the variant's
 * fast kernel with its automatic shape (and its reference kernel for small problems); MEDIUM
 * adds every compiled shape of the variant (FP32: D, CW, NC, K; complex: D, CW, complex tiles).
 * elpa_b200_autotune_setup == _setup_dtype(..., ELPA_B200_DTYPE_F64, ...).  Snapshots carry the
 * type (format v2; v1 snapshots load as FP64). */
enum { ELPA_B200_DTYPE_F64 = 0, ELPA_B200_DTYPE_F32 = 1, ELPA_B200_DTYPE_C64 = 2 };
elpa_b200_autotune *elpa_b200_autotune_setup_dtype(int64_t n, int64_t nbw, int64_t nev, int level, int dtype,
                                                  int *error);
/* Convenience: run the whole loop on device buffers.  Prepares the reflectors once per kernel
 * variant, times each candidate's apply on Q (which is overwritten: pass a scratch copy) with
 * CUDA events on `stream` (best of `reps`), returns the best options and time. */
int elpa_b200_autotune_run(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                           double *Q_scratch, int64_t ldq, elpa_b200_stream_t stream, int level, int reps,
                           elpa_b200_opts *best, double *best_ms);

/* The loop for any element type: hh_v, hh_tau, Q_scratch point to data of that type (complex:
 * interleaved doubles).  FP32 and complex candidates are timed as whole calls (prep + apply). */
int elpa_b200_autotune_run_dtype(int64_t n, int64_t nbw, int64_t nev, int dtype, const void *hh_v, const void *hh_tau,
                                 void *Q_scratch, int64_t ldq, elpa_b200_stream_t stream, int level, int reps,
                                 elpa_b200_opts *best, double *best_ms);

/* ---------------------------------------------------------------------------------------
 * NEXT-1: band -> full back-transformation (the second transform of every eigenvector in the
 * two-stage solver).  Stage-1 reflector j (j = 0 .. K-1) annihilated column j of the
 * full -> band reduction below row j + nbw; it acts on rows [j + nbw, n):
 *      Q <- H_0 H_1 ... H_{K-1} Q        (H_{K-1} applied first), K = n - nbw - 1.
 * hh1_v  : device, n x K column-major (ldv >= n); column j = reflector j; the element at row
 *          j + nbw is treated as 1.0 and rows above it are never read.
 * hh1_tau: device, K doubles (0 = identity).
 * Q      : device, n x nev column-major (ldq >= n), updated in place.
 * Blocked compact WY (panels of 256 reflectors, B_p = I - V_p T_p V_p^T), applied last panel
 * first as Q <- Q + U_p (V_p^T Q) with U_p = -V_p T_p; every product runs in the library's own
 * FP64 tensor-core (DMMA) contraction kernel — no BLAS.  Asynchronous on `stream`; temporary
 * workspace (about 2x the packed panels, n^2 doubles at nbw << n) from the library's pool.
 * Errors: ERR_ARG (n < 0 or n > 2^31 - 64, nbw < 1, nev < 0, nev > n, ldv or ldq < max(1, n)),
 * ERR_NULL, ERR_DEVICE, ERR_CUDA; K == 0 or nev == 0 is OK without memory access.
 * ------------------------------------------------------------------------------------- */
int64_t elpa_b2f_count(int64_t n, int64_t nbw);   /* K, or -1 on bad arguments */
int elpa_trans_ev_band_to_full(int64_t n, int64_t nbw, int64_t nev, const double *hh1_v, int64_t ldv,
                               const double *hh1_tau, double *Q, int64_t ldq, elpa_b200_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-4: generalized back-transformation.  For the generalized EVP A x = lambda B x with the
 * Cholesky factorisation B = L L^H and the standard problem of
 * Atilde = L^{-1} A L^{-H}, the last step of the solver maps its eigenvectors
 * back:  V = (L^{-1})^H Vtilde  (Eq. 7; real case: L^{-T}).
 * L : device, n x n lower triangular, column-major (ldl >= n); only the lower triangle
 *     (diagonal included) is read; its diagonal must be nonzero (not checked).
 * Q : device, n x nev column-major (ldq >= n): in Vtilde, out V (in place).
 * Blocked left-looking triangular solve: 128 x 128 diagonal blocks inverted by an own kernel,
 * the off-diagonal updates and the inverted-block products run in the library's own FP64
 * tensor-core (DMMA) contraction kernel — no BLAS.  Asynchronous on `stream`.
 * Errors: ERR_ARG (n < 0 or n > 2^31 - 64, nev < 0, nev > n, ldl or ldq < max(1, n)), ERR_NULL,
 * ERR_DEVICE, ERR_CUDA; n == 0 or nev == 0 is OK without memory access.
 * ------------------------------------------------------------------------------------- */
int elpa_generalized_back_transform(int64_t n, int64_t nev, const double *L, int64_t ldl, double *Q, int64_t ldq,
                                    elpa_b200_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: FP32 variant.  ELPA offers the whole solver in single precision, and
 * single precision in the eigen-steps is where the paper's 1.3-1.5x SCF gains come from
 * (P:663-692).  Same operation, reflector order, storage conventions, validation order and
 * error codes as elpa_trans_ev_tridi_to_band, on float data:
 *   hh_v   : device, nbw x R floats; hh_tau: device, R floats;
 *   Q      : device, n x nev floats, ldq % 4 == 0 and Q 16-byte aligned (else ERR_ALIGN).
 * opts (may be NULL): kernel AUTO (FFMA2 when nbw % 8 == 0 and nbw <= 128, else REFERENCE),
 *   ELPA_B200_KERNEL_FFMA2 or ELPA_B200_KERNEL_REFERENCE (one thread per column, explicitly
 *   rounded FP32, any nbw); depth_warps = D, col_warps = CW, tiles_per_warp = NC (32-column
 *   blocks per warp, 1 or 2), grid_ctas as for FP64; groups_per_step (K groups of 8 reflectors
 *   per step) 0 = auto, 1 or 2 where that shape is compiled (elpa_b200_describe_f32 says; MEDIUM
 *   autotuning enumerates them).
 * Accuracy: FP32 rounding, tolerance DESIGN.md R14.  Asynchronous on `stream`; the temporary
 * workspace comes from the library's pool, stream-ordered on `stream`.
 * ------------------------------------------------------------------------------------- */
int elpa_trans_ev_tridi_to_band_f32(int64_t n, int64_t nbw, int64_t nev, const float *hh_v, const float *hh_tau,
                                    float *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts);
/* As elpa_b200_describe, for the FP32 entry point. */
int elpa_b200_describe_f32(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts,
                           char *buf, size_t buflen);

/* ---------------------------------------------------------------------------------------
 * NEXT-3 (second half): complex Hermitian variant.  ELPA's complex solver chases a
 * Hermitian band matrix with complex reflectors H_r = I - tau_r v_r v_r^H (zlarfg
 * convention, R15).  Same geometry, order and error codes as the real entry:
 *      Q <- H_0 H_1 ... H_{R-1} Q,   per reflector  w = tau_r v_r^H q,  q -= w v_r.
 * Complex data are interleaved (re, im) doubles (C99 double complex / cuDoubleComplex layout):
 *   hh_v : device, nbw x R complex (column r = reflector r), element 0 treated as 1;
 *   hh_tau: device, R complex;  Q: device, n x nev complex, ldq >= n (complex elements),
 *   16-byte aligned (else ERR_ALIGN).
 * opts (may be NULL): kernel AUTO (DMMA when nbw % 8 == 0 and nbw <= 128, else REFERENCE),
 *   ELPA_B200_KERNEL_DMMA (complex compact-WY groups on FP64 tensor cores, 4 real DMMAs per
 *   complex product) or ELPA_B200_KERNEL_REFERENCE (one thread per column, bitwise the CPU
 *   oracle); depth_warps D, col_warps CW, tiles_per_warp = complex 8-column tiles per warp;
 *   groups_per_step 0 (auto), 1, or 2 with D = 1, NZ = 1, CW in {2, 4, 8} at nbw 32 or 64 (the
 *   K-group register-window kernel on complex tiles; the automatic choice below 8000 eigenvectors
 *   at nbw 32 and 64); other combinations: ERR_ARG.  Asynchronous on `stream`.
 * ------------------------------------------------------------------------------------- */
int elpa_trans_ev_tridi_to_band_c64(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                                    double *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts);
/* As elpa_b200_describe, for the complex entry point. */
int elpa_b200_describe_c64(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts,
                           char *buf, size_t buflen);

/* Static description of an error code. */
const char *elpa_b200_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* ELPA_B200_H */
