// geometry.cuh — closed-form reflector indexing of the band->tridiagonal chase
// (SURVEY.md §8 notation).  Shared by host and device code of the CUDA path.
//
// Reflector (j, m): sweep j in [0, n-3], depth m in [0, M_j), M_j = (n-3-j)/b + 1.
//   first row s = j + 1 + m*b, length L = min(b, n - s), exists iff s <= n-2.
//   generation index r(j,m) = off(j) + m,  off(j) = j + F(n-3) - F(n-3-j),
//   F(x) = sum_{t=0}^{x} floor(t/b) = b*q*(q-1)/2 + q*(x mod b + 1), q = floor(x/b), F(-1) = 0.
//   R = off(n-2) = (n-2) + F(n-3).   Depths: M = (n-3)/b + 1, J_m = n-3-m*b.
#pragma once
#include <stdint.h>

namespace elpa_b200 {

__host__ __device__ inline int64_t floor_sum(int64_t x, int64_t b) {
    if (x < 0) return 0;
    int64_t q = x / b;
    return b * q * (q - 1) / 2 + q * (x % b + 1);
}

__host__ __device__ inline int64_t hh_off(int64_t j, int64_t n, int64_t b) {
    return j + floor_sum(n - 3, b) - floor_sum(n - 3 - j, b);
}

__host__ __device__ inline int64_t hh_total(int64_t n, int64_t b) {
    if (n < 3 || b < 2) return 0;
    return (n - 2) + floor_sum(n - 3, b);
}

__host__ __device__ inline int64_t num_depths(int64_t n, int64_t b) {
    if (n < 3 || b < 2) return 0;
    return (n - 3) / b + 1;
}

// ---- k = 8 group geometry of the DMMA path (b % 8 == 0, b8 = b/8, lambda = b8 + 1) ----
// Group g of depth m holds sweeps j = 8g+6-a, a = 0..7 (a = 0 applied first).  Its row
// window is chunks [g + m*b8, g + m*b8 + lambda) (8 rows per chunk, 8*lambda = b + 8 rows):
// reflector a starts at window row 7-a.  G_m = ((n-2) >> 3) - m*b8 + 1 groups at depth m;
// blob(m, g) = base(m) + g with base(m) = m*G_0 - b8*m*(m-1)/2.
__host__ __device__ inline int64_t groups_at_depth(int64_t n, int64_t b8, int64_t m) {
    return ((n - 2) >> 3) - m * b8 + 1;
}
__host__ __device__ inline int64_t group_base(int64_t n, int64_t b8, int64_t m) {
    int64_t G0 = groups_at_depth(n, b8, 0);
    return m * G0 - b8 * m * (m - 1) / 2;
}
__host__ __device__ inline int64_t total_groups(int64_t n, int64_t b8, int64_t M) {
    return group_base(n, b8, M);
}
// doubles per prepared group.  DMMA layout (kind 0): dot B-fragments of U = -V T (lambda x 32
// lanes x 2), update B-fragments of V (same).  Complex layout (kind 2): B-fragments of Re U',
// Im U', Re V, Im V (4 x 64 lambda).
__host__ __device__ inline int64_t blob_doubles(int64_t lambda, int kind = 0) {
    return kind == 0 ? 128 * lambda : 256 * lambda;
}

}  // namespace elpa_b200
