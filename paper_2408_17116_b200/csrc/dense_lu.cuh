// dense_lu.cuh — blocked dense kernels for the diagonal leaves of the H-LU
// (zgetrf + zgecon at hmatrix.py:835-843, the zgetrs-style leaf solves of
// lsolve_dense / usolve_dense / rsolve_upper_dense, hmatrix.py:658-710).
//
// The unblocked kernels (k_getrf / k_trsm in hlu_kernels.cuh) take one
// CTA-wide barrier and one dependent L2 round trip per column: n = 192 costs
// ~4 ms per factorisation and ~0.5 ms per solve, all of it on the critical
// path of the H-LU (64 diagonal leaves at config 2).  Here every triangular
// dependency chain is cut into 32-wide diagonal blocks:
//   * the 32-step chain inside a diagonal block runs in registers of one warp
//     (lane = row, operands exchanged with shuffles, no barrier);
//   * the update of the rows below / above is a small GEMM done by the whole
//     CTA (independent loads, one barrier);
// so a triangular solve costs 2 barriers per 32 rows instead of one per row.
// The LU is right-looking with 32-column panels factored in shared memory,
// the row interchanges applied as one gathered permutation per panel, the
// U12 block solved in registers (thread per column) and the trailing update
// done as a shared-memory-panel GEMM.  rcond uses the same zlacn2 iteration
// as before on top of the blocked solves.
#pragma once
#include <cuda/barrier>

constexpr int LU_NT = 256;          // threads of the blocked LU / solve kernels
constexpr int LU_NW = LU_NT / 32;
constexpr int LU_NB = 32;           // panel width / triangular block
constexpr int LU_QC = 64;           // U12 columns staged per trailing-update chunk
constexpr int LU_NMAX = 384;        // largest leaf handled (panel n x 32 + U12 chunk in shared memory)

__device__ __forceinline__ zc zshfl(zc v, int src) {
  return zmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// element (i, j) of the triangular operator of a factored leaf A = P^T L U (col-major, ld n)
//   mode 0: L (unit lower)   1: U (upper)   2: U^H (lower)   3: L^H (unit upper)
__device__ __forceinline__ zc tri_el(const zc* __restrict__ A, int n, int mode, int i, int j) {
  return mode < 2 ? A[(int64_t)j * n + i] : zconj(A[(int64_t)i * n + j]);
}

// x <- T^{-1} x for one vector x (shared memory, n entries); all threads of the CTA
__device__ void blk_trsv(const zc* __restrict__ A, int n, int mode, zc* x) {
  const bool lower = (mode == 0 || mode == 2);
  const bool unit = (mode == 0 || mode == 3);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nbk = (n + LU_NB - 1) / LU_NB;
  for (int bb = 0; bb < nbk; ++bb) {
    const int b = lower ? bb : nbk - 1 - bb;
    const int j0 = b * LU_NB, bs = min(LU_NB, n - j0);
    if (w == 0) {
      zc t[LU_NB];
#pragma unroll
      for (int s = 0; s < LU_NB; ++s)
        t[s] = (s < bs && lane < bs) ? tri_el(A, n, mode, j0 + lane, j0 + s) : zmk(0.0, 0.0);
      zc xv = lane < bs ? x[j0 + lane] : zmk(0.0, 0.0);
      const zc dinv = (!unit && lane < bs) ? zdiv(zmk(1.0, 0.0), tri_el(A, n, mode, j0 + lane, j0 + lane))
                                           : zmk(1.0, 0.0);
      if (lower) {
#pragma unroll
        for (int s = 0; s < LU_NB; ++s) {
          if (s < bs) {
            if (!unit && lane == s) xv = zmul(xv, dinv);
            const zc xs = zshfl(xv, s);
            if (lane > s) xv = zsub(xv, zmul(t[s], xs));
          }
        }
      } else {
#pragma unroll
        for (int s = LU_NB - 1; s >= 0; --s) {
          if (s < bs) {
            if (!unit && lane == s) xv = zmul(xv, dinv);
            const zc xs = zshfl(xv, s);
            if (lane < s) xv = zsub(xv, zmul(t[s], xs));
          }
        }
      }
      if (lane < bs) x[j0 + lane] = xv;
    }
    __syncthreads();
    const int lo = lower ? j0 + bs : 0, hi = lower ? n : j0;
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      zc acc = x[i];
#pragma unroll
      for (int s = 0; s < LU_NB; ++s)
        if (s < bs) acc = zsub(acc, zmul(tri_el(A, n, mode, i, j0 + s), x[j0 + s]));
      x[i] = acc;
    }
    __syncthreads();
  }
}

// x <- A^{-1} x  (herm = false)  or  A^{-H} x  (herm = true), A = P^T L U
__device__ void blk_lu_solve(const zc* A, int n, const int* piv, zc* x, bool herm) {
  if (!herm) {
    if (threadIdx.x == 0)
      for (int k = 0; k < n; ++k)
        if (piv[k] != k) {
          const zc t = x[k];
          x[k] = x[piv[k]];
          x[piv[k]] = t;
        }
    __syncthreads();
    blk_trsv(A, n, 0, x);
    blk_trsv(A, n, 1, x);
  } else {
    blk_trsv(A, n, 2, x);
    blk_trsv(A, n, 3, x);
    if (threadIdx.x == 0)
      for (int k = n - 1; k >= 0; --k)
        if (piv[k] != k) {
          const zc t = x[k];
          x[k] = x[piv[k]];
          x[piv[k]] = t;
        }
    __syncthreads();
  }
}

__device__ __forceinline__ double lu_block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < LU_NW; ++i) t += red[i];
  return t;
}
// CTA argmax (first index among equal values); returns the index, all threads
template <int NWARP = LU_NW>
__device__ __forceinline__ int lu_block_argmax(double bv, int bi, double* sv, int* si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  // every warp reduces the NWARP partials by shuffles (a serial loop over them in every
  // thread was 13 % of k_getrf_blk's stall samples)
  static_assert(NWARP <= 32, "one lane per partial");
  const int l = threadIdx.x & 31;
  double B = l < NWARP ? sv[l] : -1.0;
  int I = l < NWARP ? si[l] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, B, o);
    const int oi = __shfl_xor_sync(0xffffffffu, I, o);
    if (ov > B || (ov == B && oi < I)) {
      B = ov;
      I = oi;
    }
  }
  return I;
}

// ---------------------------------------------------------------------------
// GETRF + rcond, one 512-thread CTA per diagonal leaf, n <= LU_NMAX
// dynamic shared memory: n * LU_NB complex (panel, later the estimator vector)
// ---------------------------------------------------------------------------
constexpr int GF_NT = 512;   // getrf threads (more loads in flight in the global-memory phases)
constexpr int GF_NW = GF_NT / 32;

__device__ __forceinline__ zc zshfl32(zc v, int src) {
  return zmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

__global__ void __launch_bounds__(GF_NT) k_getrf_blk(zc* __restrict__ ar, int* __restrict__ pivs,
                                                     const GetrfD* __restrict__ ds, double* anorm_out) {
  const GetrfD d = ds[blockIdx.x];
  const int n = d.n;
  zc* A = ar + d.A;
  int* piv = pivs + d.piv;
  if (threadIdx.x == 0) flop_add(8.0 * n * (double)n * n / 3.0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* P = reinterpret_cast<zc*>(smem_raw);   // panel, column c at P[c * n + i] (absolute rows)
  __shared__ double sv[GF_NW], red[GF_NW];
  __shared__ int si[GF_NW];
  __shared__ int spiv[LU_NB];
  __shared__ int trow[2 * LU_NB], tsrc[2 * LU_NB];
  __shared__ int ntouch;
  const int tid = threadIdx.x;
  // ||A||_1 of the unfactored block (np.linalg.norm(A, 1)), kept for the rcond kernel
  double anorm = 0.0;
  {
    const int lane = tid & 31, w = tid >> 5;
    double loc = 0.0;
    for (int j = w; j < n; j += GF_NW) {   // warp per column, coalesced
      double s = 0.0;
      for (int i = lane; i < n; i += 32) {
        const zc a = A[(int64_t)j * n + i];
        s += hypot(a.x, a.y);
      }
      loc = fmax(loc, warp_sum(s));
    }
    if (lane == 0) red[w] = loc;
    __syncthreads();
    for (int q = 0; q < GF_NW; ++q) anorm = fmax(anorm, red[q]);
    __syncthreads();
  }

  if (tid == 0) anorm_out[d.leaf] = anorm;
  bool zero_pivot = false;
  (void)zero_pivot;
  for (int j0 = 0; j0 < n; j0 += LU_NB) {
    const int jb = min(LU_NB, n - j0);
    for (int e = tid; e < jb * (n - j0); e += GF_NT) {
      const int c = e / (n - j0), i = j0 + e % (n - j0);
      P[c * n + i] = A[(int64_t)(j0 + c) * n + i];
    }
    __syncthreads();
    // --- panel factorisation (zgetf2 on rows j0.., columns j0..j0+jb) ---
    for (int c = 0; c < jb; ++c) {
      const int col = j0 + c;
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int i = col + tid; i < n; i += GF_NT) {
        const zc a = P[c * n + i];
        const double v = fabs(a.x) + fabs(a.y);
        if (v > bv) {
          bv = v;
          bi = i;
        }
      }
      const int pr = lu_block_argmax<GF_NW>(bv, bi, sv, si);
      if (tid == 0) {
        spiv[c] = pr;
        piv[col] = pr;
      }
      if (pr != col && tid < jb) {
        const zc t = P[tid * n + col];
        P[tid * n + col] = P[tid * n + pr];
        P[tid * n + pr] = t;
      }
      __syncthreads();
      const zc ajj = P[c * n + col];
      if (ajj.x == 0.0 && ajj.y == 0.0) {
        zero_pivot = true;
        if (tid == 0) anorm_out[d.leaf] = -1.0;   // exactly singular: rcond 0
        continue;
      }
      const zc rinv = zdiv(zmk(1.0, 0.0), ajj);
      for (int i = col + 1 + tid; i < n; i += GF_NT) P[c * n + i] = zmul(P[c * n + i], rinv);
      __syncthreads();
      // rank-1 update of the panel's remaining columns: one (row, column) item per thread
      // (independent read-modify-writes instead of a per-row chain over the columns)
      {
        const int rows = n - col - 1, cols = jb - c - 1;
        // e -> (e % rows, e / rows) through a float reciprocal: exact here (e + 0.5 is never
        // within rounding of a multiple of rows for e < 2^14), no integer division
        const float rrec = rows > 0 ? 1.0f / (float)rows : 0.0f;
        for (int e = tid; e < rows * cols; e += GF_NT) {
          const int q = (int)(((float)e + 0.5f) * rrec);
          const int i = col + 1 + e - q * rows, cc = c + 1 + q;
          P[cc * n + i] = zsub(P[cc * n + i], zmul(P[c * n + i], P[cc * n + col]));
        }
      }
      __syncthreads();
    }
    // --- write the panel back ---
    for (int e = tid; e < jb * (n - j0); e += GF_NT) {
      const int c = e / (n - j0), i = j0 + e % (n - j0);
      A[(int64_t)(j0 + c) * n + i] = P[c * n + i];
    }
    // --- net row permutation of this panel's interchanges (touched rows only) ---
    if (tid == 0) {
      int nt = 0;
      for (int c = 0; c < jb; ++c) {
        const int r[2] = {j0 + c, spiv[c]};
        for (int q = 0; q < 2; ++q) {
          int f = -1;
          for (int t = 0; t < nt; ++t)
            if (trow[t] == r[q]) f = t;
          if (f < 0) {
            trow[nt] = r[q];
            tsrc[nt] = r[q];
            ++nt;
          }
        }
        int a = -1, b = -1;   // swap the sources of rows j0+c and spiv[c]
        for (int t = 0; t < nt; ++t) {
          if (trow[t] == j0 + c) a = t;
          if (trow[t] == spiv[c]) b = t;
        }
        const int s = tsrc[a];
        tsrc[a] = tsrc[b];
        tsrc[b] = s;
      }
      ntouch = nt;
    }
    __syncthreads();
    {
      // columns outside the panel: row trow[t] <- old row tsrc[t]; a warp takes 4
      // columns at a time, lane t handles touched rows t and t + 32 (all reads of a
      // column land in registers before its writes)
      const int nt = ntouch, lane = tid & 31, w = tid >> 5;
      const int nq = n - jb;
      for (int q0 = 4 * w; q0 < nq; q0 += 4 * GF_NW) {
        zc v[4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          int q = q0 + a;
          q = q < j0 ? q : q + jb;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            if (q0 + a < nq && t < nt) v[a][h] = A[(int64_t)q * n + tsrc[t]];
          }
        }
        __syncwarp();
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          int q = q0 + a;
          q = q < j0 ? q : q + jb;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            if (q0 + a < nq && t < nt) A[(int64_t)q * n + trow[t]] = v[a][h];
          }
        }
      }
    }
    __syncthreads();
    const int j1 = j0 + jb;
    if (j1 >= n) break;
    // --- per chunk of LU_QC columns: U12 = L11^{-1} A12 (a warp per 4 columns, lanes =
    //     rows of the unit lower L11 from the panel, shuffle substitution), written to A
    //     and to shared memory; then A22 -= L21 U12 with 2 x 2 register tiles ---
    {
      zc* Us = P + (size_t)n * LU_NB;   // [LU_QC][LU_NB]
      const int m2 = n - j1;
      const int tr = (m2 + 1) / 2;
      const int lane = tid & 31, w = tid >> 5;
      for (int q0 = j1; q0 < n; q0 += LU_QC) {
        const int qc = min(LU_QC, n - q0);
        for (int c4 = 4 * w; c4 < qc; c4 += 4 * GF_NW) {
          zc x[4];
#pragma unroll
          for (int h = 0; h < 4; ++h)
            x[h] = (c4 + h < qc && lane < jb) ? A[(int64_t)(q0 + c4 + h) * n + j0 + lane] : zmk(0.0, 0.0);
#pragma unroll 4
          for (int c = 0; c < LU_NB; ++c) {
            if (c < jb) {
              const zc l = lane > c && lane < jb ? P[c * n + j0 + lane] : zmk(0.0, 0.0);
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const zc xc = zshfl32(x[h], c);
                x[h] = zsub(x[h], zmul(l, xc));
              }
            }
          }
#pragma unroll
          for (int h = 0; h < 4; ++h)
            if (c4 + h < qc && lane < jb) {
              A[(int64_t)(q0 + c4 + h) * n + j0 + lane] = x[h];
              Us[(c4 + h) * LU_NB + lane] = x[h];
            }
        }
        __syncthreads();
        const int tq = (qc + 1) / 2, ntile = tr * tq;
        for (int tix = tid; tix < ntile; tix += GF_NT) {
          const int i = j1 + 2 * (tix % tr), ql = 2 * (tix / tr);
          const bool i1 = i + 1 < n, q1 = ql + 1 < qc;
          zc a00 = zmk(0, 0), a01 = zmk(0, 0), a10 = zmk(0, 0), a11 = zmk(0, 0);
          const zc* u0 = Us + ql * LU_NB;
          const zc* u1 = Us + (q1 ? ql + 1 : ql) * LU_NB;
#pragma unroll 8
          for (int c = 0; c < LU_NB; ++c) {
            if (c < jb) {
              const zc l0 = P[c * n + i];
              const zc l1 = i1 ? P[c * n + i + 1] : zmk(0, 0);
              const zc b0 = u0[c], b1 = u1[c];
              zfma(a00, l0, b0);
              zfma(a01, l0, b1);
              zfma(a10, l1, b0);
              zfma(a11, l1, b1);
            }
          }
          zc* c0 = A + (int64_t)(q0 + ql) * n;
          c0[i] = zsub(c0[i], a00);
          if (i1) c0[i + 1] = zsub(c0[i + 1], a10);
          if (q1) {
            zc* c1 = c0 + n;
            c1[i] = zsub(c1[i], a01);
            if (i1) c1[i + 1] = zsub(c1[i + 1], a11);
          }
        }
        __syncthreads();
      }
    }
  }

}

// ---------------------------------------------------------------------------
// rcond of a factored diagonal leaf (zgecon): Hager/Higham 1-norm estimate of
// ||A^{-1}||_1 (zlacn2 structure) with the blocked solves.  Nothing in the
// factorisation consumes rcond (the reference raises SingularDiagonal, which we
// report after the factorisation), so it runs on a side stream off the
// critical path.  anorm[leaf] < 0 marks an exactly zero pivot.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(LU_NT) k_rcond_blk(const zc* __restrict__ ar, const int* __restrict__ pivs,
                                                     const GetrfD* __restrict__ ds, const double* anorm_in,
                                                     double* rcond_out, int* flag) {
  const GetrfD d = ds[blockIdx.x];
  const int n = d.n;
  const zc* A = ar + d.A;
  const int* piv = pivs + d.piv;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* x = reinterpret_cast<zc*>(smem_raw);   // n entries
  __shared__ double sv[LU_NW], red[LU_NW];
  __shared__ int si[LU_NW];
  const int tid = threadIdx.x;
  const double anorm = anorm_in[d.leaf];
  double rcond = 0.0;
  if (anorm > 0.0) {
    double est = 0.0;
    for (int i = tid; i < n; i += LU_NT) x[i] = zmk(1.0 / n, 0.0);
    __syncthreads();
    int jlast = -1;
    for (int it = 0; it < 5; ++it) {
      blk_lu_solve(A, n, piv, x, false);   // y = A^{-1} x
      double s = 0.0;
      for (int i = tid; i < n; i += LU_NT) s += hypot(x[i].x, x[i].y);
      s = lu_block_sum(s, red);
      if (it > 0 && s <= est) break;
      est = s;
      for (int i = tid; i < n; i += LU_NT) {   // xi = sign(y)
        const double a = hypot(x[i].x, x[i].y);
        x[i] = a > 0 ? zmk(x[i].x / a, x[i].y / a) : zmk(1.0, 0.0);
      }
      __syncthreads();
      blk_lu_solve(A, n, piv, x, true);    // z = A^{-H} xi
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int i = tid; i < n; i += LU_NT) {
        const double a = hypot(x[i].x, x[i].y);
        if (a > bv) {
          bv = a;
          bi = i;
        }
      }
      const int jm = lu_block_argmax(bv, bi, sv, si);
      if (jm == jlast) break;
      jlast = jm;
      __syncthreads();
      for (int i = tid; i < n; i += LU_NT) x[i] = zmk(i == jm ? 1.0 : 0.0, 0.0);
      __syncthreads();
    }
    // alternative estimate with x_i = (-1)^i (1 + i/(n-1))
    __syncthreads();
    for (int i = tid; i < n; i += LU_NT)
      x[i] = zmk((i % 2 ? -1.0 : 1.0) * (1.0 + (n > 1 ? (double)i / (n - 1) : 0.0)), 0.0);
    __syncthreads();
    blk_lu_solve(A, n, piv, x, false);
    double s = 0.0;
    for (int i = tid; i < n; i += LU_NT) s += hypot(x[i].x, x[i].y);
    s = lu_block_sum(s, red);
    est = fmax(est, 2.0 * s / (3.0 * n));
    rcond = est > 0.0 ? (1.0 / est) / anorm : 0.0;
  }
  if (tid == 0) {
    rcond_out[d.leaf] = rcond;
    if (!(rcond >= 1e-14)) atomicOr(flag, 1);
  }
}


// ---------------------------------------------------------------------------
// TRSM with a factored diagonal leaf (variants as k_trsm), blocked:
// one 512-thread CTA per (descriptor, 32-column chunk of Y), chunk in shared memory
// ---------------------------------------------------------------------------
// grid = tile list of the group (x: solve, y: 32-column chunk over its static width), as for
// k_gemm_mma: the widths of a group run from one rank to a whole 1536-column block
__global__ void __launch_bounds__(LU_NT, 2) k_trsm_blk(zc* __restrict__ ar, const int* __restrict__ ranks,
                                                    const int* __restrict__ pivs,
                                                    const TrsmD* __restrict__ ds, const uint2* __restrict__ tiles) {
  const uint2 tl = tiles[blockIdx.x];
  const TrsmD d = ds[tl.x];
  const int p = dimv(d.p, ranks), n = d.n;
  if (tl.y == 0 && threadIdx.x == 0) flop_add(4.0 * n * n * p);
  const int c0 = (int)tl.y * LU_NB;
  if (c0 >= p) return;
  const int nc = min(LU_NB, p - c0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* S = reinterpret_cast<zc*>(smem_raw);   // [nc][n]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (!d.Y.tr) {
    // untransposed right-hand side: every column of the chunk is one contiguous run of n
    // complex numbers -- staged by the bulk-copy engine (TMA, cp.async.bulk through
    // cuda::memcpy_async on a shared-memory barrier), one copy per column issued by one
    // thread, instead of a load / store round trip through every thread's registers
#pragma nv_diag_suppress static_var_with_dynamic_init
    __shared__ cuda::barrier<cuda::thread_scope_block> bar;
    if (tid == 0) {
      init(&bar, LU_NT);
      cuda::device::experimental::fence_proxy_async_shared_cta();
    }
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < nc; ++j)
        cuda::memcpy_async(S + (size_t)j * n, ar + d.Y.off + (int64_t)(c0 + j) * d.Y.ld,
                           cuda::aligned_size_t<16>((size_t)n * sizeof(zc)), bar);
    bar.arrive_and_wait();
  } else {
    for (int e = tid; e < n * nc; e += LU_NT) {
      const int i = e % n, j = e / n;
      S[j * n + i] = ar[vidx(d.Y, i, c0 + j)];
    }
    __syncthreads();
  }
  const zc* A = ar + d.T;
  // variant 0: P^T L  -> row swaps then mode 0;  1: U -> mode 1;  2: U^T (lower, no conj)
  if (d.variant == 0) {
    // pivots staged in shared memory first (one coalesced load): the swap chain below is
    // sequential, and a dependent global load per step made it the slowest part
    __shared__ int spv[LU_NMAX];
    for (int k2 = tid; k2 < n; k2 += LU_NT) spv[k2] = pivs[d.piv + k2];
    __syncthreads();
    if (tid < nc) {
      zc* s = S + tid * n;
      for (int k2 = 0; k2 < n; ++k2) {
        const int q = spv[k2];
        if (q != k2) {
          const zc t = s[k2];
          s[k2] = s[q];
          s[q] = t;
        }
      }
    }
    __syncthreads();
  }
  const bool lower = d.variant != 1;
  const bool unit = d.variant == 0;
  auto el = [&](int i, int j) -> zc {
    return d.variant == 2 ? A[(int64_t)i * n + j] : A[(int64_t)j * n + i];
  };
  const int nbk = (n + LU_NB - 1) / LU_NB;
  for (int bb = 0; bb < nbk; ++bb) {
    const int b = lower ? bb : nbk - 1 - bb;
    const int j0 = b * LU_NB, bs = min(LU_NB, n - j0);
    // diagonal block: warp w solves columns w, w + 16 (lane = row); warps without a
    // column skip the block load (one right-hand side: 1 of 16 warps works here)
    if (w < nc) {
      zc t[LU_NB];
#pragma unroll
      for (int s = 0; s < LU_NB; ++s) t[s] = (s < bs && lane < bs) ? el(j0 + lane, j0 + s) : zmk(0.0, 0.0);
      const zc dinv = (!unit && lane < bs) ? zdiv(zmk(1.0, 0.0), el(j0 + lane, j0 + lane)) : zmk(1.0, 0.0);
      for (int c = w; c < nc; c += LU_NW) {
        zc xv = lane < bs ? S[c * n + j0 + lane] : zmk(0.0, 0.0);
        if (lower) {
#pragma unroll
          for (int s = 0; s < LU_NB; ++s)
            if (s < bs) {
              if (!unit && lane == s) xv = zmul(xv, dinv);
              const zc xs = zshfl(xv, s);
              if (lane > s) xv = zsub(xv, zmul(t[s], xs));
            }
        } else {
#pragma unroll
          for (int s = LU_NB - 1; s >= 0; --s)
            if (s < bs) {
              if (lane == s) xv = zmul(xv, dinv);
              const zc xs = zshfl(xv, s);
              if (lane < s) xv = zsub(xv, zmul(t[s], xs));
            }
        }
        if (lane < bs) S[c * n + j0 + lane] = xv;
      }
    }
    __syncthreads();
    // remaining rows: S[c][i] -= sum_s T(i, j0 + s) S[c][j0 + s], 8 columns per work item
    const int lo = lower ? j0 + bs : 0, hi = lower ? n : j0;
    const int nr = hi - lo, ng = (nc + 7) / 8;
    for (int e = tid; e < nr * ng; e += LU_NT) {
      const int i = lo + e % nr, g = (e / nr) * 8;
      zc acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = (g + q < nc) ? S[(g + q) * n + i] : zmk(0.0, 0.0);
#pragma unroll 8
      for (int s = 0; s < LU_NB; ++s) {
        if (s < bs) {
          const zc tv = el(i, j0 + s);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (g + q < nc) acc[q] = zsub(acc[q], zmul(tv, S[(g + q) * n + j0 + s]));
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (g + q < nc) S[(g + q) * n + i] = acc[q];
    }
    __syncthreads();
  }
  for (int e = tid; e < n * nc; e += LU_NT) {
    const int i = e % n, j = e / n;
    ar[vidx(d.Y, i, c0 + j)] = S[j * n + i];
  }
}
