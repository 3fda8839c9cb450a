// lowrank.cuh — CTA-cooperative dense linear algebra on complex128 for the
// low-rank recompression (truncate_lowrank, hmatrix.py:412-426):
//   Householder QR (Hermitian reflectors, in place, column-major, any m x k)
//   application of Q to a block
//   one-sided (Hestenes) Jacobi SVD with round-robin parallel ordering
// All routines are called by every thread of the CTA; data may live in global
// or shared memory (generic addressing).
#pragma once
#include "common.cuh"

constexpr int LR_NT = 512;
constexpr int LR_NW = LR_NT / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ zc warp_sum(zc v) {
  return zmk(warp_sum(v.x), warp_sum(v.y));
}
// CTA-wide sum; red must hold LR_NW doubles; result broadcast to all threads
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < LR_NW; ++i) t += red[i];
  return t;
}

// Householder QR of A (m x k, ld) in place.  On exit the upper triangle
// (strictly above the diagonal) holds R, rdiag[j] = R[j][j], A[j:, j] holds the
// reflector u_j with H_j = I - kappa[j] u_j u_j^H (Hermitian, unitary), and
// A = H_0 H_1 ... H_{kk-1} [R; 0].  kk = min(m, k).
__device__ __forceinline__ void cta_qr(zc* A, int m, int k, int ld, zc* rdiag, double* kappa, double* red) {
  const int kk = min(m, k);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 0; j < kk; ++j) {
    zc* x = A + (int64_t)j * ld;
    double s = 0.0;
    for (int i = j + threadIdx.x; i < m; i += LR_NT) s += zabs2(x[i]);
    s = block_sum(s, red);
    const double nx = sqrt(s);
    const zc alpha = x[j];
    const double aa = sqrt(zabs2(alpha));
    const zc ph = aa > 0.0 ? zmk(alpha.x / aa, alpha.y / aa) : zmk(1.0, 0.0);
    double kap = 0.0;
    __syncthreads();   // everyone has read alpha before thread 0 overwrites it
    if (nx > 0.0) {
      kap = 1.0 / (nx * (nx + aa));
      if (threadIdx.x == 0) {
        x[j] = zscale(ph, aa + nx);      // u_0 = alpha - beta, beta = -ph * nx
        rdiag[j] = zscale(ph, -nx);
        kappa[j] = kap;
      }
    } else if (threadIdx.x == 0) {
      rdiag[j] = zmk(0.0, 0.0);
      kappa[j] = 0.0;
    }
    __syncthreads();
    if (kap != 0.0) {
      for (int c = j + 1 + w; c < k; c += LR_NW) {
        zc* y = A + (int64_t)c * ld;
        zc d = zmk(0.0, 0.0);
        for (int i = j + lane; i < m; i += 32) d = zadd(d, zcmul(x[i], y[i]));
        d = zscale(warp_sum(d), kap);
        for (int i = j + lane; i < m; i += 32) y[i] = zsub(y[i], zmul(d, x[i]));
      }
    }
    __syncthreads();
  }
}

// Z (m x ncol, ldz) := Q Z with Q = H_0 ... H_{kk-1} from cta_qr (reflectors in A).
__device__ __forceinline__ void cta_apply_q(const zc* A, int m, int kk, int ld, const double* kappa, zc* Z,
                            int ncol, int ldz) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = kk - 1; j >= 0; --j) {
    const double kap = kappa[j];
    if (kap != 0.0) {
      const zc* x = A + (int64_t)j * ld;
      for (int c = w; c < ncol; c += LR_NW) {
        zc* y = Z + (int64_t)c * ldz;
        zc d = zmk(0.0, 0.0);
        for (int i = j + lane; i < m; i += 32) d = zadd(d, zcmul(x[i], y[i]));
        d = zscale(warp_sum(d), kap);
        for (int i = j + lane; i < m; i += 32) y[i] = zsub(y[i], zmul(d, x[i]));
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi: M (p x q, ldm) <- M W with orthogonal columns, W (q x q,
// ldw) unitary (initialised here to I).  Returns the number of sweeps.
__device__ __forceinline__ int cta_jacobi(zc* M, int p, int q, int ldm, zc* W, int ldw, int* flag,
                                          double* red) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // columns below 1e-12 |M|_F are numerical noise for every truncation tolerance
  // used here (>= 1e-8); rotating them only chases rounding, so they are skipped
  double f2 = 0.0;
  for (int e = threadIdx.x; e < p * q; e += LR_NT) f2 += zabs2(M[(int64_t)(e / p) * ldm + e % p]);
  f2 = block_sum(f2, red);
  const double floor2 = 1e-24 * f2;
  for (int e = threadIdx.x; e < q * q; e += LR_NT) {
    int i = e % q, j = e / q;
    W[(int64_t)j * ldw + i] = zmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  if (q < 2) return 0;
  const int qe = q + (q & 1);
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < qe - 1; ++r) {
      for (int pi = w; pi < qe / 2; pi += LR_NW) {
        // circle method: position 0 fixed, others rotate
        const int pa = pi, pb = qe - 1 - pi;
        const int a = pa == 0 ? 0 : ((pa - 1 + r) % (qe - 1)) + 1;
        const int b = pb == 0 ? 0 : ((pb - 1 + r) % (qe - 1)) + 1;
        if (a >= q || b >= q) continue;
        zc* x = M + (int64_t)a * ldm;
        zc* y = M + (int64_t)b * ldm;
        double al = 0.0, be = 0.0;
        zc ga = zmk(0.0, 0.0);
        for (int i = lane; i < p; i += 32) {
          al += zabs2(x[i]);
          be += zabs2(y[i]);
          ga = zadd(ga, zcmul(x[i], y[i]));
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        const double g = sqrt(zabs2(ga));
        if (!(g > 1e-14 * sqrt(al * be)) || g == 0.0 || fmin(al, be) < floor2) continue;
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        const zc e = zmk(ga.x / g, ga.y / g);                  // e^{i phi}
        const zc se = zscale(e, sn), sec = zscale(zconj(e), sn);
        // x' = c x - s e^{-i phi} y ;  y' = s e^{i phi} x + c y
        for (int i = lane; i < p; i += 32) {
          const zc xi = x[i], yi = y[i];
          x[i] = zsub(zscale(xi, cs), zmul(sec, yi));
          y[i] = zadd(zmul(se, xi), zscale(yi, cs));
        }
        zc* wx = W + (int64_t)a * ldw;
        zc* wy = W + (int64_t)b * ldw;
        for (int i = lane; i < q; i += 32) {
          const zc xi = wx[i], yi = wy[i];
          wx[i] = zsub(zscale(xi, cs), zmul(sec, yi));
          wy[i] = zadd(zmul(se, xi), zscale(yi, cs));
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  return sweep;
}

// Hermitian two-sided Jacobi on the Gram matrix G = M^H M (q x q, in shared
// memory): G <- J^H G J until off-diagonal |g_pq| <= 1e-15 sqrt(g_pp g_qq),
// W <- W J (W q x q, shared, initialised to I).  Rounds use the parallel
// round-robin ordering; each round = rotation parameters (one thread per
// pair), column update, row update.  Returns sweeps.
__device__ __forceinline__ int cta_herm_jacobi(zc* G, zc* W, int q, double* cs_c, zc* cs_s,
                                               int* pa, int* pb, int* flag) {
  for (int e = threadIdx.x; e < q * q; e += LR_NT) {
    const int i = e % q, j = e / q;
    W[j * q + i] = zmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  if (q < 2) return 0;
  const int qe = q + (q & 1), np = qe / 2;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < qe - 1; ++r) {
      // (1) rotation parameters
      for (int pi = threadIdx.x; pi < np; pi += LR_NT) {
        const int xa = pi, xb = qe - 1 - pi;
        int a = xa == 0 ? 0 : ((xa - 1 + r) % (qe - 1)) + 1;
        int b = xb == 0 ? 0 : ((xb - 1 + r) % (qe - 1)) + 1;
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        pa[pi] = a;
        pb[pi] = b;
        cs_c[pi] = -1.0;   // inactive
        cs_s[pi] = zmk(0.0, 0.0);
        if (b >= q) continue;
        const double ga = G[a * q + a].x, gb = G[b * q + b].x;
        const zc g = G[b * q + a];   // G[a][b] (column-major: col b, row a)
        const double ag = sqrt(zabs2(g));
        if (!(ag > 1e-15 * sqrt(fabs(ga * gb))) || ag == 0.0) continue;
        const double zeta = (gb - ga) / (2.0 * ag);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        cs_c[pi] = c;
        // s e^{-i phi} with e^{i phi} = g / |g|
        cs_s[pi] = zmk(c * t * g.x / ag, -c * t * g.y / ag);
        *flag = 1;
      }
      __syncthreads();
      // (2) columns: G J and W J.  J = [[c, s], [-s e^{-i phi}, c e^{-i phi}]]
      //     col a' = c col a - s e^{-i phi} col b ;  col b' = s col a + c e^{-i phi} col b
      for (int e = threadIdx.x; e < np * q * 2; e += LR_NT) {
        const int which = e / (np * q);        // 0: G, 1: W
        const int pi = (e / q) % np, i = e % q;
        const double c = cs_c[pi];
        if (c < 0.0) continue;
        const zc se = cs_s[pi];                 // s e^{-i phi}
        const double s = sqrt(zabs2(se));
        const zc eph = s > 0 ? zmk(se.x / s, se.y / s) : zmk(1.0, 0.0);   // e^{-i phi}
        zc* X = which ? W : G;
        const int a = pa[pi], b = pb[pi];
        const zc xa = X[a * q + i], xb = X[b * q + i];
        X[a * q + i] = zsub(zscale(xa, c), zmul(se, xb));
        X[b * q + i] = zadd(zscale(xa, s), zmul(zscale(eph, c), xb));
      }
      __syncthreads();
      // (3) rows: J^H G.  row a' = c row a - s e^{+i phi} row b ; row b' = s row a + c e^{+i phi} row b
      for (int e = threadIdx.x; e < np * q; e += LR_NT) {
        const int pi = e / q, j = e % q;
        const double c = cs_c[pi];
        if (c < 0.0) continue;
        const zc se = zconj(cs_s[pi]);          // s e^{+i phi}
        const double s = sqrt(zabs2(se));
        const zc eph = s > 0 ? zmk(se.x / s, se.y / s) : zmk(1.0, 0.0);
        const int a = pa[pi], b = pb[pi];
        const zc ya = G[j * q + a], yb = G[j * q + b];
        G[j * q + a] = zsub(zscale(ya, c), zmul(se, yb));
        G[j * q + b] = zadd(zscale(ya, s), zmul(zscale(eph, c), yb));
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  return sweep;
}

// CTA-tiled small GEMM: C (rows x l, col-major ldc) = op(A) (rows x kk) * B (kk x l, ldb),
// l <= 64.  op: 0 A (col-major, lda), 1 A^T, 2 A^H, 3 conj(A).  Staging tiles of
// 64 rows x 32 k of op(A) and 32 x l of B in shared memory (sm >= 2*32*65 zc).
constexpr int TG_R = 64, TG_K = 32;
__device__ __forceinline__ void cta_gemm_tiled64(zc* C, int ldc, const zc* A, int lda, int mode,
                                                 const zc* B, int ldb, int rows, int kk, int l,
                                                 zc* sm);
// any l: column blocks of 64
__device__ __forceinline__ void cta_gemm_tiled(zc* C, int ldc, const zc* A, int lda, int mode,
                                               const zc* B, int ldb, int rows, int kk, int l,
                                               zc* sm) {
  for (int c0 = 0; c0 < l; c0 += 64)
    cta_gemm_tiled64(C + (int64_t)c0 * ldc, ldc, A, lda, mode, B + (int64_t)c0 * ldb, ldb, rows, kk,
                     min(64, l - c0), sm);
}
__device__ __forceinline__ void cta_gemm_tiled64(zc* C, int ldc, const zc* A, int lda, int mode,
                                                 const zc* B, int ldb, int rows, int kk, int l,
                                                 zc* sm) {
  zc* As = sm;                       // [TG_K][TG_R + 1]
  zc* Bs = sm + TG_K * (TG_R + 1);   // [TG_K][64 + 1]
  const int tr = threadIdx.x % TG_R, tg = threadIdx.x / TG_R;   // 8 column groups
  constexpr int NG = LR_NT / TG_R;
  for (int r0 = 0; r0 < rows; r0 += TG_R) {
    zc acc[64 / NG];
#pragma unroll
    for (int q = 0; q < 64 / NG; ++q) acc[q] = zmk(0.0, 0.0);
    for (int k0 = 0; k0 < kk; k0 += TG_K) {
      __syncthreads();
      for (int e = threadIdx.x; e < TG_K * TG_R; e += LR_NT) {
        int i, a;
        if (mode == 1 || mode == 2) {   // contiguous along k for a fixed row
          a = e % TG_K;
          i = e / TG_K;
        } else {
          i = e % TG_R;
          a = e / TG_R;
        }
        const int gi = r0 + i, ga = k0 + a;
        zc v = zmk(0.0, 0.0);
        if (gi < rows && ga < kk) {
          if (mode == 0) v = A[(int64_t)ga * lda + gi];
          else if (mode == 1) v = A[(int64_t)gi * lda + ga];
          else if (mode == 2) v = zconj(A[(int64_t)gi * lda + ga]);
          else v = zconj(A[(int64_t)ga * lda + gi]);
        }
        As[a * (TG_R + 1) + i] = v;
      }
      for (int e = threadIdx.x; e < TG_K * l; e += LR_NT) {
        const int a = e % TG_K, c = e / TG_K;
        Bs[a * 65 + c] = (k0 + a < kk) ? B[(int64_t)c * ldb + k0 + a] : zmk(0.0, 0.0);
      }
      __syncthreads();
      const int kmax = min(TG_K, kk - k0);
      for (int a = 0; a < kmax; ++a) {
        const zc av = As[a * (TG_R + 1) + tr];
#pragma unroll
        for (int q = 0; q < 64 / NG; ++q) {
          const int c = tg + NG * q;
          if (c < l) zfma(acc[q], av, Bs[a * 65 + c]);
        }
      }
    }
    if (r0 + tr < rows)
#pragma unroll
      for (int q = 0; q < 64 / NG; ++q) {
        const int c = tg + NG * q;
        if (c < l) C[(int64_t)c * ldc + r0 + tr] = acc[q];
      }
  }
  __syncthreads();
}

__device__ __forceinline__ double hw_sum(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One-sided Jacobi with one HALF-warp per column pair (32 pairs in flight per
// round with 512 threads); same rotation and skip rules as cta_jacobi.
__device__ __forceinline__ int cta_jacobi_hw(zc* M, int p, int q, int ldm, zc* W, int ldw, int* flag,
                                             double* red) {
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
  constexpr int NHW = LR_NT / 16;
  double f2 = 0.0;
  for (int e = threadIdx.x; e < p * q; e += LR_NT) f2 += zabs2(M[(int64_t)(e / p) * ldm + e % p]);
  f2 = block_sum(f2, red);
  const double floor2 = 1e-24 * f2;
  for (int e = threadIdx.x; e < q * q; e += LR_NT) {
    int i = e % q, j = e / q;
    W[(int64_t)j * ldw + i] = zmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  if (q < 2) return 0;
  const int qe = q + (q & 1);
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < qe - 1; ++r) {
      // warp-uniform trip count: both half-warps of a warp shuffle together
      for (int base = 0; base < qe / 2; base += NHW) {
        const int pi = base + hw;
        const int pa = pi, pb = qe - 1 - pi;
        const int a = pa == 0 ? 0 : ((pa - 1 + r) % (qe - 1)) + 1;
        const int b = pb == 0 ? 0 : ((pb - 1 + r) % (qe - 1)) + 1;
        const bool valid = pi < qe / 2 && a < q && b < q;
        zc* x = M + (int64_t)(valid ? a : 0) * ldm;
        zc* y = M + (int64_t)(valid ? b : 0) * ldm;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        if (valid)
          for (int i = hl; i < p; i += 16) {
            const zc xi = x[i], yi = y[i];
            al += zabs2(xi);
            be += zabs2(yi);
            gr += xi.x * yi.x + xi.y * yi.y;
            gi += xi.x * yi.y - xi.y * yi.x;
          }
        al = hw_sum(al);
        be = hw_sum(be);
        gr = hw_sum(gr);
        gi = hw_sum(gi);
        if (!valid) continue;
        const double g = sqrt(gr * gr + gi * gi);
        if (!(g > 1e-14 * sqrt(al * be)) || g == 0.0 || fmin(al, be) < floor2) continue;
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        const double ig = 1.0 / g;
        const zc se = zmk(gr * ig * sn, gi * ig * sn), sec = zmk(gr * ig * sn, -gi * ig * sn);
        for (int i = hl; i < p; i += 16) {
          const zc xi = x[i], yi = y[i];
          x[i] = zsub(zscale(xi, cs), zmul(sec, yi));
          y[i] = zadd(zmul(se, xi), zscale(yi, cs));
        }
        zc* wx = W + (int64_t)a * ldw;
        zc* wy = W + (int64_t)b * ldw;
        for (int i = hl; i < q; i += 16) {
          const zc xi = wx[i], yi = wy[i];
          wx[i] = zsub(zscale(xi, cs), zmul(sec, yi));
          wy[i] = zadd(zmul(se, xi), zscale(yi, cs));
        }
        if (hl == 0) *flag = 1;
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  return sweep;
}

// ---------------------------------------------------------------------------
// Split-CTA variants: the two halves of the CTA (threads [0, NT/2) and
// [NT/2, NT)) work on independent problems, synchronising with named barriers
// (bar.sync id, NT/2) instead of __syncthreads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void half_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(LR_NT / 2) : "memory");
}
__device__ __forceinline__ double half_sum(double v, double* red, int id) {
  constexpr int NWH = LR_NW / 2;
  v = warp_sum(v);
  const int w = (threadIdx.x >> 5) % NWH, l = threadIdx.x & 31;
  half_bar(id);
  if (l == 0) red[w] = v;
  half_bar(id);
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < NWH; ++i) t += red[i];
  return t;
}
// cta_qr for one half of the CTA; id = 1 + half index, red has LR_NW/2 doubles
__device__ __forceinline__ void half_qr(zc* A, int m, int k, int ld, zc* rdiag, double* kappa,
                                        double* red, int id) {
  constexpr int NTH = LR_NT / 2, NWH = LR_NW / 2;
  const int tid = threadIdx.x % NTH;
  const int kk = min(m, k);
  const int w = tid >> 5, lane = tid & 31;
  for (int j = 0; j < kk; ++j) {
    zc* x = A + (int64_t)j * ld;
    double s = 0.0;
    for (int i = j + tid; i < m; i += NTH) s += zabs2(x[i]);
    s = half_sum(s, red, id);
    const double nx = sqrt(s);
    const zc alpha = x[j];
    const double aa = sqrt(zabs2(alpha));
    const zc ph = aa > 0.0 ? zmk(alpha.x / aa, alpha.y / aa) : zmk(1.0, 0.0);
    double kap = 0.0;
    half_bar(id);
    if (nx > 0.0) {
      kap = 1.0 / (nx * (nx + aa));
      if (tid == 0) {
        x[j] = zscale(ph, aa + nx);
        rdiag[j] = zscale(ph, -nx);
        kappa[j] = kap;
      }
    } else if (tid == 0) {
      rdiag[j] = zmk(0.0, 0.0);
      kappa[j] = 0.0;
    }
    half_bar(id);
    if (kap != 0.0) {
      for (int c = j + 1 + w; c < k; c += NWH) {
        zc* y = A + (int64_t)c * ld;
        zc d = zmk(0.0, 0.0);
        for (int i = j + lane; i < m; i += 32) d = zadd(d, zcmul(x[i], y[i]));
        d = zscale(warp_sum(d), kap);
        for (int i = j + lane; i < m; i += 32) y[i] = zsub(y[i], zmul(d, x[i]));
      }
    }
    half_bar(id);
  }
}
__device__ __forceinline__ void half_apply_q(const zc* A, int m, int kk, int ld, const double* kappa,
                                             zc* Z, int ncol, int ldz, int id) {
  constexpr int NTH = LR_NT / 2, NWH = LR_NW / 2;
  const int tid = threadIdx.x % NTH;
  const int w = tid >> 5, lane = tid & 31;
  for (int j = kk - 1; j >= 0; --j) {
    const double kap = kappa[j];
    if (kap != 0.0) {
      const zc* x = A + (int64_t)j * ld;
      for (int c = w; c < ncol; c += NWH) {
        zc* y = Z + (int64_t)c * ldz;
        zc d = zmk(0.0, 0.0);
        for (int i = j + lane; i < m; i += 32) d = zadd(d, zcmul(x[i], y[i]));
        d = zscale(warp_sum(d), kap);
        for (int i = j + lane; i < m; i += 32) y[i] = zsub(y[i], zmul(d, x[i]));
      }
    }
    half_bar(id);
  }
}
