// trunc2.cu — K6 recompression, blocked variant: one 256-thread CTA per problem,
// two CTAs resident per SM.  Same contract as k_truncate (truncate_lowrank,
// hmatrix.py:412-426: QR(U), QR(V^T), SVD of R_u R_v^T, keep s > tol * s_0) for
// U V^T with k <= 128 and m, n <= 512 -- every recompression of the H-LU and of
// the ACA leaves.  The unblocked k_truncate is latency bound (one CTA-wide
// barrier pair per Householder column, Q applied one reflector at a time, the
// Jacobi rotations accumulated); here:
//   1. blocked Householder QR of U and of Vt: panels of pw columns factored in
//      shared memory with ONE barrier per column (every warp regenerates the
//      reflector from the column itself), trailing columns updated with the
//      UT-transform block reflector  Q_p = I - Y S^{-1} Y^H,  S = triu(Y^H Y)
//      with unit diagonal (Y = reflectors scaled by sqrt(kappa));
//   2. core M = R_u R_v^T, then a column-pivoted QR of M stopped as soon as
//      the trailing Frobenius norm is <= DELTA * tol * (largest column norm)
//      (<= DELTA * tol * s_0): only directions far below the truncation
//      threshold are dropped, and the SVD works on k' ~ r + few columns;
//   3. one-sided Jacobi on R1^H (kk2 x k') WITHOUT accumulating rotations:
//      the columns converge to B = V_M Sigma, and the right singular vectors
//      of M are Vhat = P B / sigma;
//   4. U' = Q_u (M Vhat)  (= Q_u U_M Sigma),  Vt' = Q_v conj(Vhat), both Q's
//      applied with the stored block reflectors.
#include <cooperative_groups.h>

#include "hmatrix.h"
#include "lowrank.cuh"

#define T2NS t2s
#define T2_NT 256
#define T2_ELEMS 6144
#define T2_MINB 2
#include "trunc2_impl.cuh"
#undef T2NS
#undef T2_NT
#undef T2_ELEMS
#undef T2_MINB

#define T2NS t2b
#define T2_GRAM 1
#define T2_NT 512
#define T2_ELEMS 12800
#define T2_MINB 1
#include "trunc2_impl.cuh"
#undef T2NS
#undef T2_NT
#undef T2_ELEMS
#undef T2_MINB
#undef T2_GRAM

extern unsigned long long* g_trunc_prof;

// Gram-path recompression of factor-form problems; those whose device-side rank
// exceeds 64 are appended to defer (defer[0] = count, then indices into d_desc),
// unless mn_multi > 0: then ranks up to 256 with max(m, n) <= mn_multi take the
// multi-stage Gram path and only its failures are deferred
void launch_truncate_gram(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, double tol,
                          unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, zc* arena_out,
                          int* defer, const int* idx, int mn_multi, int csize) {
  if (nd == 0) return;
  t2b::launch_gram(arena, arena_out ? arena_out : arena, ranks, d_desc, nd, tol, overflow, scratch, s,
                   g_trunc_prof, defer, idx, mn_multi, csize);
}

// co-resident clusters of the Gram kernel per cluster size (cached per process; 0 = unknown)
int truncate_gram_max_clusters(int csize) {
  static int cache[9] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
  if (csize < 1 || csize > 8) return 0;
  if (cache[csize] < 0) cache[csize] = csize == 1 ? 148 : t2b::gram_max_clusters(csize);
  return cache[csize];
}

bool launch_truncate_blocked(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, double tol,
                             unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, int kc_max,
                             int mn_max, zc* arena_out, int* defer, const int* idx) {
  if (getenv("CBIE_TRUNC_UNBLOCKED")) return false;
  if (kc_max <= 0 || mn_max <= 0 || mn_max > t2b::MMAX) return false;
  if (!arena_out) arena_out = arena;
  if (nd == 0) return true;
  const int kc = std::min(kc_max, t2b::KMAX);
  // blocks up to 192 rows: 256 threads, 96 KB, two CTAs per SM; larger blocks:
  // 512 threads, 200 KB (wider panels, fewer trailing passes), one CTA per SM
  if (mn_max <= 192)
    t2s::launch_rpl<6>(arena, arena_out, ranks, d_desc, nd, kc, tol, overflow, scratch, s, g_trunc_prof, defer,
                       idx);
  else
    t2b::launch_rpl<12>(arena, arena_out, ranks, d_desc, nd, kc, tol, overflow, scratch, s, g_trunc_prof, defer,
                        idx);
  return true;
}

CBIE_FLOP_API(trunc2)
