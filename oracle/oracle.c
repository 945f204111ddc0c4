/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for ELPA's stage-2 eigenvector
 * back-transformation (trans_ev_tridi_to_band) and the band->tridiagonal chase that
 * produces its reflectors.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_1811_01277_b200/csrc/).
 *
 * Citations (PAPER.md = /root/reference/PAPER.md, "P:L" = line L; SPEC.md "S:L"):
 *   - Householder reflector Q_i = I - beta_i v_i v_i^H, never formed        P:117-121 (Sec. 2, after Eq. 4)
 *   - one reflector per eliminated column, stored as (v, beta)
 *   - two-stage: band -> tridiagonal as a second step
 *   - back-transformation  Vtilde = Q^H Vhat  (Eq. 6)
 *   - each eigenvector transformed twice in the two-stage path
 *   - reflector convention v_0 = 1, LAPACK beta, sign opposite to leading
 *   - beta = 0 means identity (skipped column)
 *   - chase "single-sweep ... column elimination with reflector length <= b;
 *     schedule stored explicitly"
 * Readings where the paper is silent are listed in DESIGN.md §2 (R1..R12).
 *
 * Build (done by __graft_entry__.build() / oracle.ensure_built()):
 *   gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared -o oracle/liboracle.so oracle/oracle.c -lm
 * -ffp-contract=off: round-to-nearest products and sums, no FMA contraction (R10).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * Schedule: enumerate the chase's reflectors in generation order by plain loops
 * (sweep j ascending, then position m ascending).  Reflector (j, m) eliminates the
 * entries below row s = j+1+m*b of column (m==0 ? j : previous s); it acts on rows
 * [s, s+L), L = min(b, n-s); it exists iff L >= 2 (R2/R4).
 * Returns R; fills s_out/L_out if non-NULL.
 * ---------------------------------------------------------------------------------- */
int64_t oracle_schedule(int64_t n, int64_t b, int64_t *s_out, int64_t *L_out) {
    int64_t r = 0;
    if (n < 3 || b < 2) return 0;
    for (int64_t j = 0; j <= n - 3; j++) {
        for (int64_t s = j + 1; s <= n - 2; s += b) {
            int64_t L = (n - s < b) ? (n - s) : b;
            if (s_out) s_out[r] = s;
            if (L_out) L_out[r] = L;
            r++;
        }
    }
    return r;
}

/* ------------------------------------------------------------------------------------
 * Symmetric matrix in lower band storage with room for 3b sub-diagonals
 * (the chase's transient bulge reaches 2b-1; 3b is slack).  A(r,c), r>=c, at
 * w[c*ld + (r-c)].
 * ---------------------------------------------------------------------------------- */
typedef struct { int64_t n, ld; double *w; } symband;

static double sb_get(const symband *A, int64_t r, int64_t c) {
    if (r < c) { int64_t t = r; r = c; c = t; }
    if (r - c >= A->ld) return 0.0;
    return A->w[c * A->ld + (r - c)];
}

/* returns 0 on success, 1 if a nonzero value falls outside the storage */
static int sb_set(symband *A, int64_t r, int64_t c, double x) {
    if (r < c) { int64_t t = r; r = c; c = t; }
    if (r - c >= A->ld) return x != 0.0;
    A->w[c * A->ld + (r - c)] = x;
    return 0;
}

/* LAPACK dlarfg convention: for x of length L, find (v, tau, beta) with
 * (I - tau v v^T) x = beta e_0, v_0 = 1.  alpha = x0, sigma^2 = sum_{i>=1} x_i^2.
 * sigma == 0 -> tau = 0, v = e_0, beta = alpha (identity).  Otherwise
 * beta = -sign(alpha) sqrt(alpha^2 + sigma^2) (sign(0) = +1), tau = (beta - alpha)/beta,
 * v_i = x_i / (alpha - beta). */
static void plain_dlarfg(int64_t L, const double *x, double *v, double *tau, double *beta) {
    double alpha = x[0], sig2 = 0.0;
    for (int64_t i = 1; i < L; i++) sig2 += x[i] * x[i];
    v[0] = 1.0;
    if (sig2 == 0.0) {
        for (int64_t i = 1; i < L; i++) v[i] = 0.0;
        *tau = 0.0;
        *beta = alpha;
        return;
    }
    double nrm = sqrt(alpha * alpha + sig2);
    double bt = (alpha >= 0.0) ? -nrm : nrm;
    *tau = (bt - alpha) / bt;
    double scal = alpha - bt;
    for (int64_t i = 1; i < L; i++) v[i] = x[i] / scal;
    *beta = bt;
}

/* ------------------------------------------------------------------------------------
 * Band -> tridiagonal bulge chase recording every reflector (R1).
 *   band_in : (b+1) x n, band_in[d*n + c] = B(c+d, c)  (row-major (b+1, n) array)
 *   hh_v    : R x b  (reflector r's vector at hh_v[r*b .. r*b+b), zero-padded past L, v0=1)
 *   hh_tau  : R
 *   s_out, L_out : explicit schedule (R each)
 *   d (n), e (n-1): the resulting tridiagonal T
 * Each step applies A <- H A H literally: first H*A on rows [s, s+L) of a dense copy of
 * the window [s-2b, s+L+2b) x same, then (H*A)*H on its columns [s, s+L), and writes
 * the window back.  The eliminated entries are then set to exactly (beta, 0, ..., 0).
 * Returns R, or -1 if a nonzero value would leave the 3b storage (never expected).
 * ---------------------------------------------------------------------------------- */
int64_t oracle_chase(int64_t n, int64_t b, const double *band_in,
                     double *hh_v, double *hh_tau, int64_t *s_out, int64_t *L_out,
                     double *d, double *e) {
    symband A;
    A.n = n;
    A.ld = 3 * b + 1;
    A.w = (double *)calloc((size_t)(n * A.ld), sizeof(double));
    for (int64_t c = 0; c < n; c++)
        for (int64_t dd = 0; dd <= b && c + dd < n; dd++)
            A.w[c * A.ld + dd] = band_in[dd * n + c];

    int64_t wmax = 5 * b + 2;
    double *win = (double *)malloc(sizeof(double) * (size_t)(wmax * wmax));
    double *x = (double *)malloc(sizeof(double) * (size_t)(b + 1));
    double *v = (double *)malloc(sizeof(double) * (size_t)(b + 1));
    int64_t r = 0;
    int bad = 0;

    if (n >= 3 && b >= 2) {
        for (int64_t j = 0; j <= n - 3; j++) {
            int64_t col = j;
            for (int64_t s = j + 1; s <= n - 2; s += b) {
                int64_t L = (n - s < b) ? (n - s) : b;
                for (int64_t i = 0; i < L; i++) x[i] = sb_get(&A, s + i, col);
                double tau, beta;
                plain_dlarfg(L, x, v, &tau, &beta);

                if (tau != 0.0) {
                    int64_t k0 = s - 2 * b; if (k0 < 0) k0 = 0;
                    int64_t k1 = s + L + 2 * b; if (k1 > n) k1 = n;
                    int64_t K = k1 - k0;
                    int64_t o = s - k0; /* window offset of row/col s */
                    /* only rows [o,o+L) and cols [o,o+L) of the window are read or written.
                     * OpenMP splits each loop over independent rows/columns only: every element's
                     * arithmetic (and summation order) is the same for any thread count. */
#pragma omp parallel for schedule(static) if (K * L >= 4096)
                    for (int64_t i = 0; i < L; i++)
                        for (int64_t t = 0; t < K; t++) {
                            win[(o + i) * K + t] = sb_get(&A, s + i, k0 + t);
                            win[t * K + o + i] = sb_get(&A, k0 + t, s + i);
                        }
                    /* left: rows [o, o+L) <- H * rows */
#pragma omp parallel for schedule(static) if (K * L >= 4096)
                    for (int64_t cc = 0; cc < K; cc++) {
                        double p = 0.0;
                        for (int64_t i = 0; i < L; i++) p += v[i] * win[(o + i) * K + cc];
                        p *= tau;
                        for (int64_t i = 0; i < L; i++) win[(o + i) * K + cc] -= p * v[i];
                    }
                    /* right: cols [o, o+L) <- cols * H */
#pragma omp parallel for schedule(static) if (K * L >= 4096)
                    for (int64_t rr = 0; rr < K; rr++) {
                        double q = 0.0;
                        for (int64_t i = 0; i < L; i++) q += win[rr * K + o + i] * v[i];
                        q *= tau;
                        for (int64_t i = 0; i < L; i++) win[rr * K + o + i] -= q * v[i];
                    }
                    /* write back the lower triangle of the touched rows/cols */
#pragma omp parallel for schedule(static) reduction(| : bad) if (K * L >= 4096)
                    for (int64_t i = 0; i < L; i++)
                        for (int64_t t = 0; t < K; t++) {
                            if (t <= o + i) bad |= sb_set(&A, s + i, k0 + t, win[(o + i) * K + t]);
                            else            bad |= sb_set(&A, k0 + t, s + i, win[t * K + o + i]);
                        }
                }
                /* eliminated column: exactly (beta, 0, ..., 0) */
                bad |= sb_set(&A, s, col, beta);
                for (int64_t i = 1; i < L; i++) bad |= sb_set(&A, s + i, col, 0.0);

                for (int64_t i = 0; i < b; i++) hh_v[r * b + i] = (i < L) ? v[i] : 0.0;
                hh_tau[r] = tau;
                s_out[r] = s;
                L_out[r] = L;
                r++;
                col = s;
            }
        }
    }
    for (int64_t i = 0; i < n; i++) d[i] = sb_get(&A, i, i);
    for (int64_t i = 0; i + 1 < n; i++) e[i] = sb_get(&A, i + 1, i);
    free(win); free(x); free(v); free(A.w);
    return bad ? -1 : r;
}

/* ------------------------------------------------------------------------------------
 * Back-transformation, one reflector at a time (the plain definition, R3):
 *   Q_out = H_0 H_1 ... H_{R-1} Q,   H_r = I - tau_r v_r v_r^T on rows [s_r, s_r+L_r)
 * i.e. for r = R-1 down to 0, for every column c:
 *   w = tau_r * sum_{i=0}^{L_r-1} v_r[i] * Q[s_r+i, c]   (summed in increasing i)
 *   Q[s_r+i, c] -= w * v_r[i]
 * v_r[0] is taken as 1.0 and v_r[i >= L_r] is never read (the ABI's convention).
 *   hh_v : R x nbw (row r = reflector r), hh_tau : R, s_arr/L_arr : schedule
 *   Q    : nev x ldq (row c = column c of the column-major n x nev block)
 * OpenMP over columns only: every column's arithmetic is independent of the thread
 * count (bitwise deterministic).
 * ---------------------------------------------------------------------------------- */
void oracle_apply(int64_t n, int64_t nbw, int64_t nev, int64_t R,
                  const double *hh_v, const double *hh_tau,
                  const int64_t *s_arr, const int64_t *L_arr,
                  double *Q, int64_t ldq, int nthreads) {
    (void)n;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < nev; c++) {
        double *q = Q + c * ldq;
        for (int64_t r = R - 1; r >= 0; r--) {
            const double *v = hh_v + r * nbw;
            int64_t s = s_arr[r], L = L_arr[r];
            double sum = q[s];                      /* v[0] == 1 */
            for (int64_t i = 1; i < L; i++) sum += v[i] * q[s + i];
            double w = hh_tau[r] * sum;
            q[s] -= w;                              /* w * v[0] */
            for (int64_t i = 1; i < L; i++) q[s + i] -= w * v[i];
        }
    }
}

/* ====================================================================================
 * Stage 1 (NEXT-1): full -> band reduction and the band -> full back-transformation.
 * PAPER.md P:141-143 ("the matrix is reduced to a banded form ... BLAS level 3") and
 * P:144-146 (each eigenvector is transformed twice).  The oracle uses the unblocked form:
 * one reflector per column; ELPA's BLAS-3 panels regroup exactly these reflectors.
 * Reflector j (j = 0 .. n-b-2) annihilates A[j+b+1 : n, j]; it acts on rows [s, n) with
 * s = j + b, L = n - s >= 2.  V is n x K column-major (column j = reflector j, v[s] = 1,
 * zeros above s), K = n - b - 1 (0 if n < b + 2).
 * ==================================================================================== */
int64_t oracle_reduce_to_band(int64_t n, int64_t b, double *A, double *V, double *tau, int64_t *s_out) {
    int64_t K = (n >= b + 2) ? n - b - 1 : 0;
    double *x = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *v = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t j = 0; j < K; j++) {
        int64_t s = j + b, L = n - s;
        for (int64_t i = 0; i < L; i++) x[i] = A[j * n + s + i];
        double t, beta;
        plain_dlarfg(L, x, v, &t, &beta);
        if (t != 0.0) {
            /* left: A[s:, c] <- H A[s:, c] for all columns c */
            for (int64_t c = 0; c < n; c++) {
                double p = 0.0;
                for (int64_t i = 0; i < L; i++) p += v[i] * A[c * n + s + i];
                p *= t;
                for (int64_t i = 0; i < L; i++) A[c * n + s + i] -= p * v[i];
            }
            /* right: A[r, s:] <- A[r, s:] H for all rows r */
            for (int64_t r = 0; r < n; r++) {
                double q = 0.0;
                for (int64_t i = 0; i < L; i++) q += A[(s + i) * n + r] * v[i];
                q *= t;
                for (int64_t i = 0; i < L; i++) A[(s + i) * n + r] -= q * v[i];
            }
        }
        /* eliminated column/row: exactly (beta, 0, ..., 0) */
        A[j * n + s] = beta;
        A[s * n + j] = beta;
        for (int64_t i = 1; i < L; i++) {
            A[j * n + s + i] = 0.0;
            A[(s + i) * n + j] = 0.0;
        }
        for (int64_t i = 0; i < n; i++) V[j * n + i] = (i < s) ? 0.0 : v[i - s];
        tau[j] = t;
        s_out[j] = s;
    }
    free(x);
    free(v);
    return K;
}

/* Q_out = H_0 H_1 ... H_{K-1} Q (reflector K-1 applied first), H_r = I - tau_r v_r v_r^T on rows
 * [s_r, n): for r = K-1 .. 0, per column: w = tau_r * sum_{i>=s_r} v_r[i] Q[i] (v_r[s_r] = 1,
 * increasing i), Q[i] -= w v_r[i].  V: n x K column-major (ldv), Q: nev x ldq (row c = column c). */
void oracle_apply_full(int64_t n, int64_t K, const double *V, int64_t ldv, const double *tau, const int64_t *s_arr,
                       double *Q, int64_t ldq, int64_t nev, int nthreads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < nev; c++) {
        double *q = Q + c * ldq;
        for (int64_t r = K - 1; r >= 0; r--) {
            const double *v = V + r * ldv;
            int64_t s = s_arr[r];
            double sum = q[s];                          /* v[s] == 1 */
            for (int64_t i = s + 1; i < n; i++) sum += v[i] * q[i];
            double w = tau[r] * sum;
            q[s] -= w;
            for (int64_t i = s + 1; i < n; i++) q[i] -= w * v[i];
        }
    }
}

/* NEXT-4: generalized back-transformation V = (L^{-1})^H Vtilde (Eq. 7;
 * B = L L^H is the Cholesky factorisation of P:99-101; real case: L^{-T}).  Per column, plain
 * backward substitution with U = L^T:  for i = n-1 .. 0:
 *     v_i = (q_i - sum_{k = i+1}^{n-1} L[k][i] v_k) / L[i][i]      (k increasing)
 * L: n x n lower triangular, column-major with leading dimension ldl (column i contiguous);
 * Q: nev x ldq (row c = column c), overwritten with V. */
void oracle_gen_back(int64_t n, int64_t nev, const double *L, int64_t ldl, double *Q, int64_t ldq, int nthreads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < nev; c++) {
        double *q = Q + c * ldq;
        for (int64_t i = n - 1; i >= 0; i--) {
            const double *li = L + i * ldl;                 /* column i of L */
            double sum = 0.0;
            for (int64_t k = i + 1; k < n; k++) sum += li[k] * q[k];
            q[i] = (q[i] - sum) / li[i];
        }
    }
}

/* ====================================================================================
 * NEXT-3 (second half): the complex Hermitian case.  ELPA's complex solver
 * chases a Hermitian band matrix with complex reflectors Q_i = I - beta_i v_i v_i^H
 * (P:117-121 written for the complex case).  Same geometry as the real chase (R1,
 * R2): reflector (j, m) on rows [s, s+L), s = j+1+m*b, L = min(b, n-s) >= 2.  Convention
 * LAPACK zlarfg (R15): H^H (alpha; x) = (beta; 0) with beta REAL, H = I - tau v v^H,
 * v_0 = 1, tau complex; the chase applies A <- H^H A H; the back-transformation is
 *     Q_out = H_0 H_1 ... H_{R-1} Q,     per reflector  w = tau * sum_i conj(v_i) q_i,  q_i -= w v_i.
 * Complex numbers are C99 `double complex`; products and sums are the plain formulas
 * (a+bi)(c+di) = (ac-bd) + (ad+bc)i, -ffp-contract=off.
 * ==================================================================================== */
#include <complex.h>

typedef struct { int64_t n, ld; double complex *w; } hermband;

static double complex hb_get(const hermband *A, int64_t r, int64_t c) {
    if (r < c) {
        if (c - r >= A->ld) return 0.0;
        return conj(A->w[r * A->ld + (c - r)]);
    }
    if (r - c >= A->ld) return 0.0;
    return A->w[c * A->ld + (r - c)];
}

static int hb_set(hermband *A, int64_t r, int64_t c, double complex x) {
    if (r < c) { int64_t t = r; r = c; c = t; x = conj(x); }
    if (r - c >= A->ld) return x != 0.0;
    A->w[c * A->ld + (r - c)] = x;
    return 0;
}

/* zlarfg: alpha = x0, sigma^2 = sum_{i>=1} |x_i|^2.  sigma == 0 and Im(alpha) == 0 -> identity
 * (tau = 0, beta = alpha).  Otherwise beta = -sign(Re alpha) sqrt(|alpha|^2 + sigma^2)
 * (sign(0) = +1), tau = (beta - alpha) / beta, v_i = x_i / (alpha - beta). */
static void plain_zlarfg(int64_t L, const double complex *x, double complex *v, double complex *tau, double *beta) {
    double complex alpha = x[0];
    double sig2 = 0.0;
    for (int64_t i = 1; i < L; i++) sig2 += creal(x[i]) * creal(x[i]) + cimag(x[i]) * cimag(x[i]);
    v[0] = 1.0;
    if (sig2 == 0.0 && cimag(alpha) == 0.0) {
        for (int64_t i = 1; i < L; i++) v[i] = 0.0;
        *tau = 0.0;
        *beta = creal(alpha);
        return;
    }
    double nrm = sqrt(creal(alpha) * creal(alpha) + cimag(alpha) * cimag(alpha) + sig2);
    double bt = (creal(alpha) >= 0.0) ? -nrm : nrm;
    *tau = (bt - alpha) / bt;
    double complex scal = alpha - bt;
    for (int64_t i = 1; i < L; i++) v[i] = x[i] / scal;
    *beta = bt;
}

/* Hermitian band -> real-diagonal tridiagonal chase recording every reflector.
 *   band_in : (b+1) x n complex, band_in[dd*n + c] = B(c+dd, c) (the diagonal's imaginary part is ignored)
 *   hh_v    : R x b complex (v_0 = 1, zero past L), hh_tau : R complex
 *   d (n) real, e (n-1) complex: T(i+1, i) (real except possibly e[n-2], which no reflector touches)
 * Returns R, or -1 if a nonzero value would leave the 3b storage. */
int64_t oracle_chase_c(int64_t n, int64_t b, const double complex *band_in,
                       double complex *hh_v, double complex *hh_tau, int64_t *s_out, int64_t *L_out,
                       double *d, double complex *e) {
    hermband A;
    A.n = n;
    A.ld = 3 * b + 1;
    A.w = (double complex *)calloc((size_t)(n * A.ld), sizeof(double complex));
    for (int64_t c = 0; c < n; c++)
        for (int64_t dd = 0; dd <= b && c + dd < n; dd++)
            A.w[c * A.ld + dd] = dd == 0 ? creal(band_in[c]) : band_in[dd * n + c];
    int64_t wmax = 5 * b + 2;
    double complex *win = (double complex *)malloc(sizeof(double complex) * (size_t)(wmax * wmax));
    double complex *x = (double complex *)malloc(sizeof(double complex) * (size_t)(b + 1));
    double complex *v = (double complex *)malloc(sizeof(double complex) * (size_t)(b + 1));
    int64_t r = 0;
    int bad = 0;
    if (n >= 3 && b >= 2) {
        for (int64_t j = 0; j <= n - 3; j++) {
            int64_t col = j;
            for (int64_t s = j + 1; s <= n - 2; s += b) {
                int64_t L = (n - s < b) ? (n - s) : b;
                for (int64_t i = 0; i < L; i++) x[i] = hb_get(&A, s + i, col);
                double complex tau;
                double beta;
                plain_zlarfg(L, x, v, &tau, &beta);
                if (tau != 0.0) {
                    int64_t k0 = s - 2 * b; if (k0 < 0) k0 = 0;
                    int64_t k1 = s + L + 2 * b; if (k1 > n) k1 = n;
                    int64_t K = k1 - k0;
                    int64_t o = s - k0;
                    for (int64_t i = 0; i < L; i++)
                        for (int64_t t = 0; t < K; t++) {
                            win[(o + i) * K + t] = hb_get(&A, s + i, k0 + t);
                            win[t * K + o + i] = hb_get(&A, k0 + t, s + i);
                        }
                    /* left: rows [o, o+L) <- H^H rows = rows - conj(tau) v (v^H rows) */
                    for (int64_t cc = 0; cc < K; cc++) {
                        double complex p = 0.0;
                        for (int64_t i = 0; i < L; i++) p += conj(v[i]) * win[(o + i) * K + cc];
                        p *= conj(tau);
                        for (int64_t i = 0; i < L; i++) win[(o + i) * K + cc] -= p * v[i];
                    }
                    /* right: cols [o, o+L) <- cols H = cols - tau (cols v) v^H */
                    for (int64_t rr = 0; rr < K; rr++) {
                        double complex q = 0.0;
                        for (int64_t i = 0; i < L; i++) q += win[rr * K + o + i] * v[i];
                        q *= tau;
                        for (int64_t i = 0; i < L; i++) win[rr * K + o + i] -= q * conj(v[i]);
                    }
                    for (int64_t i = 0; i < L; i++)
                        for (int64_t t = 0; t < K; t++) {
                            if (t <= o + i) bad |= hb_set(&A, s + i, k0 + t, win[(o + i) * K + t]);
                            else            bad |= hb_set(&A, k0 + t, s + i, win[t * K + o + i]);
                        }
                    for (int64_t i = 0; i < L; i++)           /* Hermitian: real diagonal */
                        A.w[(s + i) * A.ld] = creal(A.w[(s + i) * A.ld]);
                }
                bad |= hb_set(&A, s, col, beta);
                for (int64_t i = 1; i < L; i++) bad |= hb_set(&A, s + i, col, 0.0);
                for (int64_t i = 0; i < b; i++) hh_v[r * b + i] = (i < L) ? v[i] : 0.0;
                hh_tau[r] = tau;
                s_out[r] = s;
                L_out[r] = L;
                r++;
                col = s;
            }
        }
    }
    for (int64_t i = 0; i < n; i++) d[i] = creal(hb_get(&A, i, i));
    for (int64_t i = 0; i + 1 < n; i++) e[i] = hb_get(&A, i + 1, i);
    free(win); free(x); free(v); free(A.w);
    return bad ? -1 : r;
}

/* Complex back-transformation, one reflector at a time in exact reverse generation order:
 * for r = R-1 .. 0, per column:  w = tau_r * sum_{i<L} conj(v_i) q[s+i]  (v_0 = 1, increasing i),
 * q[s+i] -= w * v_i.  hh_v: R x nbw complex; Q: nev x ldq complex (row c = column c). */
void oracle_apply_c(int64_t nbw, int64_t nev, int64_t R, const double complex *hh_v, const double complex *hh_tau,
                    const int64_t *s_arr, const int64_t *L_arr, double complex *Q, int64_t ldq, int nthreads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t c = 0; c < nev; c++) {
        double complex *q = Q + c * ldq;
        for (int64_t r = R - 1; r >= 0; r--) {
            const double complex *v = hh_v + r * nbw;
            int64_t s = s_arr[r], L = L_arr[r];
            double complex sum = q[s];
            for (int64_t i = 1; i < L; i++) sum += conj(v[i]) * q[s + i];
            double complex w = hh_tau[r] * sum;
            q[s] -= w;
            for (int64_t i = 1; i < L; i++) q[s + i] -= w * v[i];
        }
    }
}
