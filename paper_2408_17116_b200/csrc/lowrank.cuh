// lowrank.cuh — CTA-cooperative dense linear algebra on complex128 for the
// low-rank recompression (truncate_lowrank, hmatrix.py:412-426):
//   Householder QR (Hermitian reflectors, in place, column-major, any m x k)
//   application of Q to a block
//   one-sided (Hestenes) Jacobi SVD with round-robin parallel ordering
// All routines are called by every thread of the CTA; data may live in global
// or shared memory (generic addressing).
#pragma once
#include "common.cuh"

constexpr int LR_NT = 256;
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
__device__ __forceinline__ int cta_jacobi(zc* M, int p, int q, int ldm, zc* W, int ldw, int* flag) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < q * q; e += LR_NT) {
    int i = e % q, j = e / q;
    W[(int64_t)j * ldw + i] = zmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  if (q < 2) return 0;
  const int qe = q + (q & 1);
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
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
        if (!(g > 1e-15 * sqrt(al * be)) || g == 0.0) continue;
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
