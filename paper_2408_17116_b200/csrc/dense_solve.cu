// dense_solve.cu — the dense path solve_dense (solver.py:178-203) on the device:
// assemble_dense (assembly.py:438-460) straight into HBM, LU with partial pivoting
// (scipy.linalg.lu_factor -> zgetrf, solver.py:186) and lu_solve (zgetrs), residual
// |A x - b| / |b| from the kept matrix.
//
// Right-looking blocked LU, panels of NB = 32 columns, column-major:
//   k_panel    one CTA factors the tall panel A[j0:N, j0:j0+NB] in global memory (pivot =
//              first index of max |re| + |im| like izamax, row swap inside the panel,
//              scaling by the reciprocal pivot, rank-1 update of the panel's columns);
//   k_swap     the panel's interchanges applied to every column outside the panel;
//   k_trsm_u   U12 = L11^{-1} A12 (unit lower, 32 x 32 in shared memory);
//   k_update   A22 -= A21 U12: 64 x 64 output tiles, 4 x 4 per thread, operands staged
//              in shared memory (a rank-32 ZGEMM update).
// The solve applies the interchanges and then L and U by 32-row blocks (diagonal block
// solved in shared memory, the rest of the vector updated by a blocked GEMV).
#include <cmath>
#include <vector>

#include "context.h"

CBIE_FLOP_API(dense)

namespace {

constexpr int NB = 32;
constexpr int PT = 1024;   // panel threads

__device__ __forceinline__ double cabs1(zc z) { return fabs(z.x) + fabs(z.y); }

__global__ void __launch_bounds__(PT) k_panel(zc* __restrict__ A, int64_t N, int j0, int jb, int* __restrict__ piv,
                                             int* __restrict__ info) {
  __shared__ double bv[PT / 32];
  __shared__ int bi[PT / 32];
  __shared__ int sp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int jj = 0; jj < jb; ++jj) {
    const int64_t j = j0 + jj;
    zc* col = A + j * N;
    // pivot: first index of the largest |re| + |im| in rows j..N-1
    double best = -1.0;
    int64_t bix = N;
    for (int64_t i = j + threadIdx.x; i < N; i += PT) {
      const double v = cabs1(col[i]);
      if (v > best) {
        best = v;
        bix = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, (long long)bix, o);
      if (ob > best || (ob == best && oi < bix)) {
        best = ob;
        bix = oi;
      }
    }
    if (lane == 0) {
      bv[w] = best;
      bi[w] = (int)bix;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int ix = (int)N;
      for (int q = 0; q < PT / 32; ++q)
        if (bv[q] > b || (bv[q] == b && bi[q] < ix)) {
          b = bv[q];
          ix = bi[q];
        }
      sp = ix;
      piv[j] = ix;
      if (!(b > 0.0) && *info == 0) *info = (int)j + 1;   // exactly singular (zgetrf INFO > 0)
    }
    __syncthreads();
    const int64_t p = sp;
    // interchange rows j and p inside the panel
    if (p != j)
      for (int c = threadIdx.x; c < jb; c += PT) {
        zc* cc = A + (int64_t)(j0 + c) * N;
        const zc t = cc[j];
        cc[j] = cc[p];
        cc[p] = t;
      }
    __syncthreads();
    const zc d = col[j];
    const double dn = d.x * d.x + d.y * d.y;
    if (dn > 0.0) {
      const zc inv = zmk(d.x / dn, -d.y / dn);
      for (int64_t i = j + 1 + threadIdx.x; i < N; i += PT) col[i] = zmul(col[i], inv);
    }
    __syncthreads();
    // rank-1 update of the panel's remaining columns
    const int rest = jb - jj - 1;
    if (rest > 0) {
      const int64_t rows = N - j - 1;
      for (int64_t e = threadIdx.x; e < rows * rest; e += PT) {
        const int64_t i = j + 1 + e % rows;
        const int c = jj + 1 + (int)(e / rows);
        zc* cc = A + (int64_t)(j0 + c) * N;
        cc[i] = zsub(cc[i], zmul(col[i], cc[j]));
      }
    }
    __syncthreads();
  }
}

// interchanges of rows j0..j0+jb-1 applied to the columns outside [j0, j0 + jb)
__global__ void k_swap(zc* __restrict__ A, int64_t N, int j0, int jb, const int* __restrict__ piv) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N || (c >= j0 && c < j0 + jb)) return;
  zc* cc = A + c * N;
  for (int jj = 0; jj < jb; ++jj) {
    const int64_t j = j0 + jj, p = piv[j];
    if (p != j) {
      const zc t = cc[j];
      cc[j] = cc[p];
      cc[p] = t;
    }
  }
}

// U12 = L11^{-1} A12, one thread per column c >= j0 + jb
__global__ void k_trsm_u(zc* __restrict__ A, int64_t N, int j0, int jb) {
  __shared__ zc L[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, k = e / jb;
    L[i][k] = A[(int64_t)(j0 + k) * N + j0 + i];
  }
  __syncthreads();
  const int64_t c = j0 + jb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  zc* cc = A + c * N + j0;
  zc x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) x[i] = i < jb ? cc[i] : zmk(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < NB; ++k)
#pragma unroll
    for (int i = k + 1; i < NB; ++i)
      if (i < jb) x[i] = zsub(x[i], zmul(L[i][k], x[k]));
#pragma unroll
  for (int i = 0; i < NB; ++i)
    if (i < jb) cc[i] = x[i];
}

// A22 -= A21 U12 over rows / columns [r0, N); 64 x 64 tiles, 256 threads, 4 x 4 each
__global__ void __launch_bounds__(256) k_update(zc* __restrict__ A, int64_t N, int j0, int jb) {
  __shared__ zc sa[NB / 2][64 + 1];   // A21 tile, k-major (two halves of the panel)
  __shared__ zc sb[NB / 2][64 + 1];   // U12 tile
  const int64_t r0 = j0 + jb;
  const int64_t i0 = r0 + (int64_t)blockIdx.x * 64, c0 = r0 + (int64_t)blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double ar[4][4] = {}, ai[4][4] = {};
  for (int h = 0; h < NB; h += NB / 2) {
    __syncthreads();
    for (int e = threadIdx.x; e < (NB / 2) * 64; e += 256) {
      const int k = e / 64, t = e % 64;
      const int64_t i = i0 + t, c = c0 + t;
      sa[k][t] = (h + k < jb && i < N) ? A[(int64_t)(j0 + h + k) * N + i] : zmk(0.0, 0.0);
      sb[k][t] = (h + k < jb && c < N) ? A[c * N + j0 + h + k] : zmk(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < NB / 2; ++k) {
      zc a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sa[k][tx + 16 * q];
        b[q] = sb[k][ty + 16 * q];
      }
#pragma unroll
      for (int qa = 0; qa < 4; ++qa)
#pragma unroll
        for (int qb = 0; qb < 4; ++qb) {
          ar[qa][qb] = fma(a[qa].x, b[qb].x, fma(-a[qa].y, b[qb].y, ar[qa][qb]));
          ai[qa][qb] = fma(a[qa].x, b[qb].y, fma(a[qa].y, b[qb].x, ai[qa][qb]));
        }
    }
  }
#pragma unroll
  for (int qb = 0; qb < 4; ++qb) {
    const int64_t c = c0 + ty + 16 * qb;
    if (c >= N) continue;
#pragma unroll
    for (int qa = 0; qa < 4; ++qa) {
      const int64_t i = i0 + tx + 16 * qa;
      if (i >= N) continue;
      zc& v = A[c * N + i];
      v = zmk(v.x - ar[qa][qb], v.y - ai[qa][qb]);
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    const double rem = (double)(N - r0);
    flop_add(8.0 * rem * rem * jb);
  }
}

// row-major (fill) -> column-major (factor), 32 x 32 tiles
__global__ void k_transpose(const zc* __restrict__ in, zc* __restrict__ out, int64_t N) {
  __shared__ zc t[32][33];
  const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = by + k, c = bx + threadIdx.x;
    if (r < N && c < N) t[k][threadIdx.x] = in[r * N + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = bx + k, r = by + threadIdx.x;
    if (r < N && c < N) out[c * N + r] = t[threadIdx.x][k];
  }
}

// X (N x nrhs, column-major): the interchanges in order
__global__ void k_apply_piv(zc* __restrict__ X, int64_t N, int nrhs, const int* __restrict__ piv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  zc* x = X + (int64_t)r * N;
  for (int64_t j = 0; j < N; ++j) {
    const int64_t p = piv[j];
    if (p != j) {
      const zc t = x[j];
      x[j] = x[p];
      x[p] = t;
    }
  }
}

// block b of 32 rows: solve with the diagonal block (lower unit: upper == 0; upper: 1),
// one thread per right-hand side
__global__ void k_diag_solve(const zc* __restrict__ A, zc* __restrict__ X, int64_t N, int nrhs, int j0, int jb,
                             int upper) {
  __shared__ zc D[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, k = e / jb;
    D[i][k] = A[(int64_t)(j0 + k) * N + j0 + i];
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  zc* x = X + (int64_t)r * N + j0;
  zc v[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) v[i] = i < jb ? x[i] : zmk(0.0, 0.0);
  if (!upper) {
#pragma unroll
    for (int k = 0; k < NB; ++k)
#pragma unroll
      for (int i = k + 1; i < NB; ++i)
        if (i < jb) v[i] = zsub(v[i], zmul(D[i][k], v[k]));
  } else {
    for (int k = jb - 1; k >= 0; --k) {
      const zc d = D[k][k];
      const double dn = d.x * d.x + d.y * d.y;
      v[k] = zmul(v[k], zmk(d.x / dn, -d.y / dn));
      for (int i = 0; i < k; ++i) v[i] = zsub(v[i], zmul(D[i][k], v[k]));
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i)
    if (i < jb) x[i] = v[i];
}

// rows [lo, hi) of X -= A[lo:hi, j0:j0+jb] X[j0:j0+jb]
__global__ void k_block_gemv(const zc* __restrict__ A, zc* __restrict__ X, int64_t N, int nrhs, int j0, int jb,
                             int64_t lo, int64_t hi) {
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (i >= hi) return;
  zc* x = X + (int64_t)r * N;
  zc acc = zmk(0.0, 0.0);
  for (int k = 0; k < jb; ++k) acc = zadd(acc, zmul(A[(int64_t)(j0 + k) * N + i], x[j0 + k]));
  x[i] = zsub(x[i], acc);
}

// r = A x - b (A row-major), per rhs: sums of |r|^2 and |b|^2 (fixed-order block sums)
__global__ void k_residual(const zc* __restrict__ A, const zc* __restrict__ X, const zc* __restrict__ B, int64_t N,
                           int nrhs, double* __restrict__ part) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ double s1[256], s2[256];
  double a = 0.0, bb = 0.0;
  if (i < N)
    for (int r = 0; r < nrhs; ++r) {
      const zc* x = X + (int64_t)r * N;
      zc acc = zmk(0.0, 0.0);
      const zc* row = A + i * N;
      for (int64_t j = 0; j < N; ++j) acc = zadd(acc, zmul(row[j], x[j]));
      const zc bi = B[(int64_t)r * N + i];
      const zc d = zsub(acc, bi);
      a += d.x * d.x + d.y * d.y;
      bb += bi.x * bi.x + bi.y * bi.y;
    }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = bb;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1[0];
    part[2 * blockIdx.x + 1] = s2[0];
  }
}

}  // namespace

extern "C" int cbie_dense_solve(cbie_ctx* c, int64_t cap, const cbie_c128* b, int nrhs, cbie_c128* x,
                                double* residual, cbie_c128* lu_out, int32_t* piv_out) {
  try {
    cudaSetDevice(c->device);
    c->require(c->has_class, "classify first");
    const int64_t N = c->N;
    if (N > cap) throw cbie_error(CBIE_ECAP_EXCEEDED, "N exceeds dense cap");
    if (nrhs < 1) throw cbie_error(CBIE_EINVALID, "nrhs >= 1");
    cudaStream_t s = c->stream;
    EvTimer tm;
    tm.start(s);
    DBuf<zc> A, L, X, B;
    DBuf<int> piv, info;
    DBuf<double> part;
    A.alloc((size_t)(N * N));
    L.alloc((size_t)(N * N));
    piv.alloc((size_t)N);
    info.alloc(1);
    CK(cudaMemsetAsync(info.p, 0, sizeof(int), s));
    ctx_fill_dense_device(c, A.p);
    const double fill_ms = tm.stop_ms(s);
    tm.start(s);
    {
      const unsigned g = (unsigned)((N + 31) / 32);
      k_transpose<<<dim3(g, g), dim3(32, 8), 0, s>>>(A.p, L.p, N);
      CKL();
    }
    dense_flops_reset();
    for (int j0 = 0; j0 < N; j0 += NB) {
      const int jb = (int)std::min<int64_t>(NB, N - j0);
      k_panel<<<1, PT, 0, s>>>(L.p, N, j0, jb, piv.p, info.p);
      k_swap<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(L.p, N, j0, jb, piv.p);
      const int64_t rest = N - j0 - jb;
      if (rest > 0) {
        k_trsm_u<<<(unsigned)((rest + 127) / 128), 128, 0, s>>>(L.p, N, j0, jb);
        const unsigned t = (unsigned)((rest + 63) / 64);
        k_update<<<dim3(t, t), 256, 0, s>>>(L.p, N, j0, jb);
      }
      CKL();
    }
    const double lu_ms = tm.stop_ms(s);
    int hinfo = 0;
    CK(cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (hinfo) throw cbie_error(CBIE_ESINGULAR_DIAGONAL, "exactly singular U(" + std::to_string(hinfo) + ")");
    // right-hand sides: row-major host (N x nrhs) -> column-major device
    std::vector<zc> hb((size_t)N * nrhs);
    const zc* bb = reinterpret_cast<const zc*>(b);
    for (int64_t i = 0; i < N; ++i)
      for (int r = 0; r < nrhs; ++r) hb[(size_t)r * N + i] = bb[(size_t)i * nrhs + r];
    X.alloc(hb.size());
    B.alloc(hb.size());
    CK(cudaMemcpyAsync(B.p, hb.data(), sizeof(zc) * hb.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(X.p, B.p, sizeof(zc) * hb.size(), cudaMemcpyDeviceToDevice, s));
    tm.start(s);
    const unsigned rb = (unsigned)((nrhs + 31) / 32);
    k_apply_piv<<<rb, 32, 0, s>>>(X.p, N, nrhs, piv.p);
    for (int j0 = 0; j0 < N; j0 += NB) {   // L y = P b
      const int jb = (int)std::min<int64_t>(NB, N - j0);
      k_diag_solve<<<rb, 32, 0, s>>>(L.p, X.p, N, nrhs, j0, jb, 0);
      if (j0 + jb < N)
        k_block_gemv<<<dim3((unsigned)((N - j0 - jb + 255) / 256), (unsigned)nrhs), 256, 0, s>>>(L.p, X.p, N, nrhs, j0,
                                                                                                jb, j0 + jb, N);
    }
    for (int64_t j0 = ((N - 1) / NB) * NB; j0 >= 0; j0 -= NB) {   // U x = y
      const int jb = (int)std::min<int64_t>(NB, N - j0);
      k_diag_solve<<<rb, 32, 0, s>>>(L.p, X.p, N, nrhs, (int)j0, jb, 1);
      if (j0 > 0)
        k_block_gemv<<<dim3((unsigned)((j0 + 255) / 256), (unsigned)nrhs), 256, 0, s>>>(L.p, X.p, N, nrhs, (int)j0,
                                                                                       jb, 0, j0);
    }
    CKL();
    const double solve_ms = tm.stop_ms(s);
    // residual |A x - b| / |b| with the unfactored matrix (solver.py:197-198)
    const unsigned nbk = (unsigned)((N + 255) / 256);
    part.alloc(2 * (size_t)nbk);
    k_residual<<<nbk, 256, 0, s>>>(A.p, X.p, B.p, N, nrhs, part.p);
    CKL();
    std::vector<double> hp(2 * (size_t)nbk);
    CK(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hb.data(), X.p, sizeof(zc) * hb.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double rr = 0.0, bn = 0.0;
    for (unsigned q = 0; q < nbk; ++q) {
      rr += hp[2 * q];
      bn += hp[2 * q + 1];
    }
    if (residual) *residual = bn > 0.0 ? std::sqrt(rr / bn) : 0.0;
    zc* xo = reinterpret_cast<zc*>(x);
    for (int64_t i = 0; i < N; ++i)
      for (int r = 0; r < nrhs; ++r) xo[(size_t)i * nrhs + r] = hb[(size_t)r * N + i];
    if (lu_out) {   // row-major, scipy's (lu, piv) layout: piv 0-based interchanges
      std::vector<zc> cm((size_t)(N * N));
      CK(cudaMemcpy(cm.data(), L.p, sizeof(zc) * cm.size(), cudaMemcpyDeviceToHost));
      zc* o = reinterpret_cast<zc*>(lu_out);
      for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < N; ++j) o[i * N + j] = cm[j * N + i];
    }
    if (piv_out) CK(cudaMemcpy(piv_out, piv.p, sizeof(int) * N, cudaMemcpyDeviceToHost));
    c->stat["dense_fill_ms"] = fill_ms;
    c->stat["dense_lu_ms"] = lu_ms;
    c->stat["dense_solve_ms"] = solve_ms;
    c->stat["dense_lu_update_flops"] = dense_flops_read();
  } catch (const cbie_error& e) {
    c->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}
