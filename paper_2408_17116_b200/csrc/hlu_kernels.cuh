// hlu_kernels.cuh — batched device kernels of the H-LU executor.
//
// Every kernel takes an array of descriptors (one per independent task of a
// schedule level) and reads dynamic dimensions (low-rank ranks) from the
// device-resident rank array, so the host never synchronises on ranks.
// Matrices are "views" into one complex128 arena: element (i, j) of a view is
// arena[off + (tr ? i*ld + j : j*ld + i)].
#pragma once
#include "lowrank.cuh"

struct View {
  int64_t off;
  int ld;
  int tr;
};
struct DimR {     // actual = slot >= 0 ? ranks[slot] : v
  int v;
  int slot;
};
__device__ __forceinline__ int dimv(DimR d, const int* ranks) { return d.slot >= 0 ? ranks[d.slot] : d.v; }
__device__ __forceinline__ int64_t vidx(const View& v, int i, int j) {
  return v.off + (v.tr ? (int64_t)i * v.ld + j : (int64_t)j * v.ld + i);
}

// ---------------------------------------------------------------------------
// GEMM: C = alpha A B + beta C      (A m x k, B k x n, C m x n; any views)
// ---------------------------------------------------------------------------
struct GemmD {
  View A, B, C;
  DimR m, n, k;
  zc alpha, beta;
};

constexpr int GT = 32;   // output tile
constexpr int GK = 16;   // k chunk

__global__ void __launch_bounds__(256) k_gemm(zc* __restrict__ ar, const int* __restrict__ ranks,
                                              const GemmD* __restrict__ ds) {
  const GemmD d = ds[blockIdx.z];
  const int m = dimv(d.m, ranks), n = dimv(d.n, ranks), k = dimv(d.k, ranks);
  const int i0 = blockIdx.x * GT, j0 = blockIdx.y * GT;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) flop_add(8.0 * m * n * k);
  if (i0 >= m || j0 >= n) return;
  __shared__ zc sA[GK][GT + 1];
  __shared__ zc sB[GK][GT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;   // 16 x 16 threads, 2x2 outputs each
  zc acc[2][2] = {{zmk(0, 0), zmk(0, 0)}, {zmk(0, 0), zmk(0, 0)}};
  for (int k0 = 0; k0 < k; k0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += 256) {
      const int kk = e / GT, ii = e % GT;
      const int gi = i0 + ii, gk = k0 + kk;
      sA[kk][ii] = (gi < m && gk < k) ? ar[vidx(d.A, gi, gk)] : zmk(0, 0);
      const int gj = j0 + ii;
      sB[kk][ii] = (gj < n && gk < k) ? ar[vidx(d.B, gk, gj)] : zmk(0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      const zc a0 = sA[kk][ty], a1 = sA[kk][ty + 16];
      const zc b0 = sB[kk][tx], b1 = sB[kk][tx + 16];
      zfma(acc[0][0], a0, b0);
      zfma(acc[0][1], a0, b1);
      zfma(acc[1][0], a1, b0);
      zfma(acc[1][1], a1, b1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
      if (gi < m && gj < n) {
        const int64_t o = vidx(d.C, gi, gj);
        zc v = zmul(d.alpha, acc[a][b]);
        if (d.beta.x != 0.0 || d.beta.y != 0.0) v = zadd(v, zmul(d.beta, ar[o]));
        ar[o] = v;
      }
    }
}

// 64 x 64 output tiles, 4 x 4 complex outputs per thread (8 shared loads per 16
// complex FMAs instead of 4 per 4): groups whose blocks are >= 128 on both sides
constexpr int GT64 = 64;
__global__ void __launch_bounds__(256) k_gemm64(zc* __restrict__ ar, const int* __restrict__ ranks,
                                                const GemmD* __restrict__ ds) {
  const GemmD d = ds[blockIdx.z];
  const int m = dimv(d.m, ranks), n = dimv(d.n, ranks), k = dimv(d.k, ranks);
  const int i0 = blockIdx.x * GT64, j0 = blockIdx.y * GT64;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) flop_add(8.0 * m * n * k);
  if (i0 >= m || j0 >= n) return;
  __shared__ zc sA[GK][GT64 + 1];
  __shared__ zc sB[GK][GT64 + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;   // outputs (ty + 16 a, tx + 16 b)
  zc acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = zmk(0, 0);
  for (int k0 = 0; k0 < k; k0 += GK) {
    for (int e = threadIdx.x; e < GK * GT64; e += 256) {
      const int kk = e / GT64, ii = e % GT64;
      const int gi = i0 + ii, gk = k0 + kk;
      sA[kk][ii] = (gi < m && gk < k) ? ar[vidx(d.A, gi, gk)] : zmk(0, 0);
      const int gj = j0 + ii;
      sB[kk][ii] = (gj < n && gk < k) ? ar[vidx(d.B, gk, gj)] : zmk(0, 0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GK; ++kk) {
      zc a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sA[kk][ty + 16 * q];
        b[q] = sB[kk][tx + 16 * q];
      }
#pragma unroll
      for (int qa = 0; qa < 4; ++qa)
#pragma unroll
        for (int qb = 0; qb < 4; ++qb) zfma(acc[qa][qb], a[qa], b[qb]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
      if (gi < m && gj < n) {
        const int64_t o = vidx(d.C, gi, gj);
        zc v = zmul(d.alpha, acc[a][b]);
        if (d.beta.x != 0.0 || d.beta.y != 0.0) v = zadd(v, zmul(d.beta, ar[o]));
        ar[o] = v;
      }
    }
}

// FP64 tensor-core GEMM (mma.sync.m8n8k4.f64, common.cuh zdmma): one 64 x BN output tile
// per CTA, 8 warps as 4 x 2, each warp a 16 x BN/2 sub-tile of 2 x BN/16 m8n8 blocks.
// K runs in chunks of 16 through a double-buffered shared staging filled by cp.async (one
// 16-byte complex per copy, so any view -- transposed or not, any ld -- stages the same
// way; out-of-range elements are zero-filled by the copy).  The staging is k-major with a
// row stride = 2 (mod 8) complex: the 8 lanes of a quarter-warp (4 k x 2 rows) then hit 8
// distinct 16-byte bank groups, so every fragment load is conflict-free.
constexpr int GM_BM = 64, GM_BK = 16;
__device__ __forceinline__ void gm_cp16(void* sdst, const void* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 16 : 0) : "memory");
}
constexpr size_t gm_smem_bytes(int bn) { return (size_t)2 * GM_BK * (GM_BM + 2 + bn + 2) * sizeof(zc); }
// The grid is a TILE LIST built with the plan (x: product of the group, y: tile row |
// tile column << 16, over the products' static sizes): a group mixes products from 100 x 76
// to 192 x 1536, and a (max rows, max columns, products) grid launched ~10 x more CTAs than
// there are tiles, every one of them fetching its descriptor before leaving.
template <int BN>
__global__ void __launch_bounds__(256, 2) k_gemm_mma(zc* __restrict__ ar, const int* __restrict__ ranks,
                                                     const GemmD* __restrict__ ds, const uint2* __restrict__ tiles) {
  constexpr int LDA = GM_BM + 2, LDB = BN + 2;
  constexpr int NB = BN / 16;   // m8n8 column blocks per warp
  const uint2 tl = tiles[blockIdx.x];
  const GemmD d = ds[tl.x];
  const int m = dimv(d.m, ranks), n = dimv(d.n, ranks), k = dimv(d.k, ranks);
  const int i0 = (int)(tl.y & 0xffffu) * GM_BM, j0 = (int)(tl.y >> 16) * BN;
  if (tl.y == 0 && threadIdx.x == 0) flop_add(8.0 * m * n * k);
  if (i0 >= m || j0 >= n) return;
  extern __shared__ __align__(16) unsigned char gm_smem[];
  zc(*sA)[GM_BK * LDA] = reinterpret_cast<zc(*)[GM_BK * LDA]>(gm_smem);
  zc(*sB)[GM_BK * LDB] = reinterpret_cast<zc(*)[GM_BK * LDB]>(gm_smem + 2 * GM_BK * LDA * sizeof(zc));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wm = w & 3, wn = w >> 2;
  const int fr = lane & 3, fc = lane >> 2;
  double acc[2][NB][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[a][b][0] = acc[a][b][1] = acc[a][b][2] = acc[a][b][3] = 0.0;
  const zc* __restrict__ Ag = ar + d.A.off;
  const zc* __restrict__ Bg = ar + d.B.off;
  const int lda = d.A.ld, ldb = d.B.ld, atr = d.A.tr, btr = d.B.tr;
  const int nch = (k + GM_BK - 1) / GM_BK;
  auto issue = [&](int c) {
    if (c < nch) {
      const int k0 = c * GM_BK;
      zc* a_s = sA[c & 1];
      zc* b_s = sB[c & 1];
      // the index that is contiguous in global memory runs fastest over the threads
      for (int e = threadIdx.x; e < GM_BK * GM_BM; e += 256) {
        const int kk = atr ? e % GM_BK : e / GM_BM, ii = atr ? e / GM_BK : e % GM_BM;
        const int gi = i0 + ii, gk = k0 + kk;
        const bool ok = gi < m && gk < k;
        gm_cp16(a_s + kk * LDA + ii, ok ? Ag + (atr ? (int64_t)gi * lda + gk : (int64_t)gk * lda + gi) : Ag, ok);
      }
      for (int e = threadIdx.x; e < GM_BK * BN; e += 256) {
        const int kk = btr ? e / BN : e % GM_BK, jj = btr ? e % BN : e / GM_BK;
        const int gj = j0 + jj, gk = k0 + kk;
        const bool ok = gj < n && gk < k;
        gm_cp16(b_s + kk * LDB + jj, ok ? Bg + (btr ? (int64_t)gk * ldb + gj : (int64_t)gj * ldb + gk) : Bg, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  for (int c = 0; c < nch; ++c) {
    issue(c + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const zc* a_s = sA[c & 1] + wm * 16 + fc;
    const zc* b_s = sB[c & 1] + wn * (BN / 2) + fc;
#pragma unroll
    for (int ks = 0; ks < GM_BK / 4; ++ks) {
      zc a[2], b[NB];
#pragma unroll
      for (int q = 0; q < 2; ++q) a[q] = a_s[(ks * 4 + fr) * LDA + q * 8];
#pragma unroll
      for (int q = 0; q < NB; ++q) b[q] = b_s[(ks * 4 + fr) * LDB + q * 8];
#pragma unroll
      for (int qa = 0; qa < 2; ++qa)
#pragma unroll
        for (int qb = 0; qb < NB; ++qb) zdmma(acc[qa][qb], a[qa], b[qb]);
    }
    __syncthreads();   // buffer c & 1 is refilled by the next iteration's issue
  }
  const bool has_beta = d.beta.x != 0.0 || d.beta.y != 0.0;
#pragma unroll
  for (int qa = 0; qa < 2; ++qa)
#pragma unroll
    for (int qb = 0; qb < NB; ++qb)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int gi = i0 + wm * 16 + qa * 8 + fc, gj = j0 + wn * (BN / 2) + qb * 8 + 2 * fr + j;
        if (gi < m && gj < n) {
          const int64_t o = vidx(d.C, gi, gj);
          zc v = zmul(d.alpha, zmk(acc[qa][qb][j], acc[qa][qb][2 + j]));
          if (has_beta) v = zadd(v, zmul(d.beta, ar[o]));
          ar[o] = v;
        }
      }
}

// matrix x vector (n == 1, the triangular solves with one right-hand side): a CTA takes 32
// rows, its 8 warps split the inner dimension (lanes = rows: coalesced over a column-major
// A), partial sums reduced through shared memory in a fixed order
constexpr int GV_NT = 256, GV_ROWS = 32;
__global__ void __launch_bounds__(GV_NT) k_gemv(zc* __restrict__ ar, const int* __restrict__ ranks,
                                                const GemmD* __restrict__ ds) {
  const GemmD d = ds[blockIdx.y];
  const int m = dimv(d.m, ranks), n = dimv(d.n, ranks), k = dimv(d.k, ranks);
  if (blockIdx.x == 0 && threadIdx.x == 0) flop_add(8.0 * m * n * k);
  const int r0 = blockIdx.x * GV_ROWS;
  if (r0 >= m || n < 1) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = r0 + lane;
  __shared__ zc part[GV_NT / 32][GV_ROWS];
  zc acc = zmk(0, 0);
  if (i < m)
    for (int kk = w; kk < k; kk += GV_NT / 32) zfma(acc, ar[vidx(d.A, i, kk)], ar[vidx(d.B, kk, 0)]);
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && i < m) {
    zc sum = part[0][lane];
    for (int q = 1; q < GV_NT / 32; ++q) sum = zadd(sum, part[q][lane]);
    const int64_t o = vidx(d.C, i, 0);
    zc v = zmul(d.alpha, sum);
    if (d.beta.x != 0.0 || d.beta.y != 0.0) v = zadd(v, zmul(d.beta, ar[o]));
    ar[o] = v;
  }
}

// ---------------------------------------------------------------------------
// EW: Y = a X + b Y  (X optional)
// ---------------------------------------------------------------------------
struct EwD {
  View X, Y;
  DimR m, n;
  zc a, b;
  int hasX;
};
__global__ void k_ew(zc* __restrict__ ar, const int* __restrict__ ranks, const EwD* __restrict__ ds) {
  const EwD d = ds[blockIdx.y];
  const int m = dimv(d.m, ranks), n = dimv(d.n, ranks);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const int64_t oy = vidx(d.Y, i, j);
    zc v = (d.b.x != 0.0 || d.b.y != 0.0) ? zmul(d.b, ar[oy]) : zmk(0, 0);
    if (d.hasX) v = zadd(v, zmul(d.a, ar[vidx(d.X, i, j)]));
    ar[oy] = v;
  }
}

// ---------------------------------------------------------------------------
// CONCAT: dst (rows x cap, col-major, ld rows) <- [piece_0 | piece_1 | ...]
// each piece placed at rows [roff, roff + prow) and zero elsewhere, scaled;
// ranks[out_slot] <- total columns
// ---------------------------------------------------------------------------
struct Piece {
  View src;
  int prow, roff;
  DimR cols;
  zc scale;
};
constexpr int MAX_PIECES = 16;
struct ConcatD {   // the pieces live in one pool shared by all concatenations of a plan
  int64_t dst;
  int rows, out_slot, np;
  int p0;          // first piece in the pool
};
__global__ void k_concat(zc* __restrict__ ar, int* __restrict__ ranks, const ConcatD* __restrict__ ds,
                         const Piece* __restrict__ pool) {
  // descriptor and column offsets staged once per CTA in shared memory (a per-thread
  // copy of the 800-byte descriptor, indexed by piece, went to local memory)
  __shared__ Piece sp[MAX_PIECES];
  __shared__ int c0[MAX_PIECES + 1];
  __shared__ int64_t sdst;
  __shared__ int srows, snp, sslot;
  const ConcatD* dp = ds + blockIdx.y;
  if (threadIdx.x == 0) {
    snp = dp->np;
    srows = dp->rows;
    sdst = dp->dst;
    sslot = dp->out_slot;
  }
  __syncthreads();
  const int np = snp, rows = srows;
  for (int q = threadIdx.x; q < np; q += blockDim.x) sp[q] = pool[dp->p0 + q];
  __syncthreads();
  if (threadIdx.x == 0) {
    c0[0] = 0;
    for (int q = 0; q < np; ++q) c0[q + 1] = c0[q] + dimv(sp[q].cols, ranks);
  }
  __syncthreads();
  const int tot = c0[np];
  // one column per (CTA, warp-group) pass: rows contiguous in the destination
  for (int j = blockIdx.x; j < tot; j += gridDim.x) {
    int q = 0;
    while (j >= c0[q + 1]) ++q;
    const Piece& P = sp[q];
    const int jj = j - c0[q];
    zc* dst = ar + sdst + (int64_t)j * rows;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      zc v = zmk(0, 0);
      if (i >= P.roff && i < P.roff + P.prow) v = zmul(P.scale, ar[vidx(P.src, i - P.roff, jj)]);
      dst[i] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ranks[sslot] = tot;
}

// ---------------------------------------------------------------------------
// TRSM (left): Y <- op(T)^{-1} Y for a factored dense diagonal leaf T (n x n)
//   variant 0: T = P^T L U, solve L (unit lower) after applying the row swaps
//   variant 1: U (upper, non-unit)
//   variant 2: U^T (lower, non-unit)         [right solves X U^{-1} = (U^{-T} X^T)^T]
// One CTA per (descriptor, 32-column chunk); the chunk lives in shared memory.
// ---------------------------------------------------------------------------
struct TrsmD {
  int64_t T;
  int64_t piv;     // offset into the pivot array (variant 0)
  int n, variant;
  View Y;
  DimR p;
};
constexpr int TS_COLS = 32;
__global__ void __launch_bounds__(256) k_trsm(zc* __restrict__ ar, const int* __restrict__ ranks,
                                              const int* __restrict__ pivs,
                                              const TrsmD* __restrict__ ds) {
  const TrsmD d = ds[blockIdx.y];
  const int p = dimv(d.p, ranks), n = d.n;
  if (blockIdx.x == 0 && threadIdx.x == 0) flop_add(4.0 * n * n * p);
  const int c0 = blockIdx.x * TS_COLS;
  if (c0 >= p) return;
  const int nc = min(TS_COLS, p - c0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* S = reinterpret_cast<zc*>(smem_raw);   // [nc][n]
  for (int e = threadIdx.x; e < n * nc; e += blockDim.x) {
    const int i = e % n, j = e / n;
    S[j * n + i] = ar[vidx(d.Y, i, c0 + j)];
  }
  __syncthreads();
  const zc* T = ar + d.T;
  if (d.variant == 0) {
    if (threadIdx.x < nc) {   // row swaps, sequential per column (zgetrs / _apply_piv order)
      zc* s = S + threadIdx.x * n;
      const int* pv = pivs + d.piv;
      for (int k2 = 0; k2 < n; ++k2) {
        const int q = pv[k2];
        if (q != k2) {
          zc tmp = s[k2];
          s[k2] = s[q];
          s[q] = tmp;
        }
      }
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {   // forward, unit diagonal
      for (int e = threadIdx.x; e < (n - j - 1) * nc; e += blockDim.x) {
        const int i = j + 1 + e % (n - j - 1), c = e / (n - j - 1);
        S[c * n + i] = zsub(S[c * n + i], zmul(T[(int64_t)j * n + i], S[c * n + j]));
      }
      __syncthreads();
    }
  } else if (d.variant == 1) {
    for (int j = n - 1; j >= 0; --j) {   // backward with U
      const zc djj = T[(int64_t)j * n + j];
      if (threadIdx.x < nc) S[threadIdx.x * n + j] = zdiv(S[threadIdx.x * n + j], djj);
      __syncthreads();
      for (int e = threadIdx.x; e < j * nc; e += blockDim.x) {
        const int i = e % j, c = e / j;
        S[c * n + i] = zsub(S[c * n + i], zmul(T[(int64_t)j * n + i], S[c * n + j]));
      }
      __syncthreads();
    }
  } else {
    for (int j = 0; j < n; ++j) {        // forward with U^T: (U^T)[i][j] = U[j][i]
      const zc djj = T[(int64_t)j * n + j];
      if (threadIdx.x < nc) S[threadIdx.x * n + j] = zdiv(S[threadIdx.x * n + j], djj);
      __syncthreads();
      for (int e = threadIdx.x; e < (n - j - 1) * nc; e += blockDim.x) {
        const int i = j + 1 + e % (n - j - 1), c = e / (n - j - 1);
        S[c * n + i] = zsub(S[c * n + i], zmul(T[(int64_t)i * n + j], S[c * n + j]));
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < n * nc; e += blockDim.x) {
    const int i = e % n, j = e / n;
    ar[vidx(d.Y, i, c0 + j)] = S[j * n + i];
  }
}

// ---------------------------------------------------------------------------
// GETRF + rcond: unblocked right-looking LU with partial pivoting (zgetf2:
// pivot = first max of |Re|+|Im|), then a Hager/Higham 1-norm estimate of
// ||A^{-1}||_1 (zlacn2) by one warp; rcond < 1e-14 -> SingularDiagonal
// (hmatrix.py:835-843).  One CTA per diagonal leaf.
// ---------------------------------------------------------------------------
struct GetrfD {
  int64_t A;
  int64_t piv;
  int n;
  int leaf;
};

__device__ void warp_lu_solve(const zc* A, int n, const int* piv, zc* x, bool herm) {
  // x <- A^{-1} x  or  A^{-H} x  with A = P^T L U, one warp, x in shared memory
  const int lane = threadIdx.x & 31;
  if (!herm) {
    if (lane == 0)
      for (int k = 0; k < n; ++k)
        if (piv[k] != k) {
          zc t = x[k];
          x[k] = x[piv[k]];
          x[piv[k]] = t;
        }
    __syncwarp();
    for (int i = 0; i < n; ++i) {   // L y = x
      zc s = zmk(0, 0);
      for (int j = lane; j < i; j += 32) s = zadd(s, zmul(A[(int64_t)j * n + i], x[j]));
      s = warp_sum(s);
      if (lane == 0) x[i] = zsub(x[i], s);
      __syncwarp();
    }
    for (int i = n - 1; i >= 0; --i) {   // U z = y
      zc s = zmk(0, 0);
      for (int j = i + 1 + lane; j < n; j += 32) s = zadd(s, zmul(A[(int64_t)j * n + i], x[j]));
      s = warp_sum(s);
      if (lane == 0) x[i] = zdiv(zsub(x[i], s), A[(int64_t)i * n + i]);
      __syncwarp();
    }
  } else {
    for (int i = 0; i < n; ++i) {   // U^H y = x
      zc s = zmk(0, 0);
      for (int j = lane; j < i; j += 32) s = zadd(s, zcmul(A[(int64_t)i * n + j], x[j]));
      s = warp_sum(s);
      if (lane == 0) x[i] = zdiv(zsub(x[i], s), zconj(A[(int64_t)i * n + i]));
      __syncwarp();
    }
    for (int i = n - 1; i >= 0; --i) {   // L^H z = y
      zc s = zmk(0, 0);
      for (int j = i + 1 + lane; j < n; j += 32) s = zadd(s, zcmul(A[(int64_t)i * n + j], x[j]));
      s = warp_sum(s);
      if (lane == 0) x[i] = zsub(x[i], s);
      __syncwarp();
    }
    if (lane == 0)
      for (int k = n - 1; k >= 0; --k)
        if (piv[k] != k) {
          zc t = x[k];
          x[k] = x[piv[k]];
          x[piv[k]] = t;
        }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) k_getrf(zc* __restrict__ ar, int* __restrict__ pivs,
                                               const GetrfD* __restrict__ ds, double* rcond_out,
                                               int* flag) {
  const GetrfD d = ds[blockIdx.x];
  const int n = d.n;
  zc* A = ar + d.A;
  int* piv = pivs + d.piv;
  if (threadIdx.x == 0) flop_add(8.0 * n * (double)n * n / 3.0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* x = reinterpret_cast<zc*>(smem_raw);   // [n] estimator vector
  __shared__ double red[LR_NW];
  __shared__ double s_v[LR_NW];
  __shared__ int s_i[LR_NW];
  __shared__ int s_piv;
  // ||A||_1 of the unfactored block (np.linalg.norm(A, 1))
  double anorm = 0.0;
  {
    double loc = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) {
        const zc a = A[(int64_t)j * n + i];
        s += hypot(a.x, a.y);
      }
      loc = fmax(loc, s);
    }
    for (int o = 16; o > 0; o >>= 1) loc = fmax(loc, __shfl_xor_sync(0xffffffffu, loc, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = loc;
    __syncthreads();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) anorm = fmax(anorm, red[w]);
    __syncthreads();
  }
  bool zero_pivot = false;
  for (int j = 0; j < n; ++j) {
    // pivot: first index of max |Re|+|Im| in column j, rows j..n-1
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
      const zc a = A[(int64_t)j * n + i];
      const double v = fabs(a.x) + fabs(a.y);
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      s_v[threadIdx.x >> 5] = bv;
      s_i[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double B = s_v[0];
      int I = s_i[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (s_v[w] > B || (s_v[w] == B && s_i[w] < I)) {
          B = s_v[w];
          I = s_i[w];
        }
      s_piv = I;
      piv[j] = I;
    }
    __syncthreads();
    const int pr = s_piv;
    if (pr != j)
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        zc t = A[(int64_t)c * n + j];
        A[(int64_t)c * n + j] = A[(int64_t)c * n + pr];
        A[(int64_t)c * n + pr] = t;
      }
    __syncthreads();
    const zc ajj = A[(int64_t)j * n + j];
    if (ajj.x == 0.0 && ajj.y == 0.0) {
      zero_pivot = true;
      continue;
    }
    const zc rinv = zdiv(zmk(1.0, 0.0), ajj);
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
      A[(int64_t)j * n + i] = zmul(A[(int64_t)j * n + i], rinv);
    __syncthreads();
    const int rem = n - j - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int i = j + 1 + e % rem, c = j + 1 + e / rem;
      A[(int64_t)c * n + i] = zsub(A[(int64_t)c * n + i], zmul(A[(int64_t)j * n + i], A[(int64_t)c * n + j]));
    }
    __syncthreads();
  }
  // rcond via the 1-norm estimator (zlacn2 structure), warp 0 only
  double rcond = 0.0;
  if (!zero_pivot && anorm > 0.0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double est = 0.0;
    for (int i = lane; i < n; i += 32) x[i] = zmk(1.0 / n, 0.0);
    __syncwarp();
    int jlast = -1;
    for (int it = 0; it < 5; ++it) {
      warp_lu_solve(A, n, piv, x, false);   // y = A^{-1} x
      double s = 0.0;
      for (int i = lane; i < n; i += 32) s += hypot(x[i].x, x[i].y);
      s = warp_sum(s);
      if (it > 0 && s <= est) break;
      est = s;
      for (int i = lane; i < n; i += 32) {   // xi = sign(y)
        const double a = hypot(x[i].x, x[i].y);
        x[i] = a > 0 ? zmk(x[i].x / a, x[i].y / a) : zmk(1.0, 0.0);
      }
      __syncwarp();
      warp_lu_solve(A, n, piv, x, true);    // z = A^{-H} xi
      double bv = -1.0;
      int bi = 0;
      for (int i = lane; i < n; i += 32) {
        const double a = hypot(x[i].x, x[i].y);
        if (a > bv) {
          bv = a;
          bi = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (bi == jlast) break;
      jlast = bi;
      for (int i = lane; i < n; i += 32) x[i] = zmk(i == bi ? 1.0 : 0.0, 0.0);
      __syncwarp();
    }
    // alternative estimate with x_i = (-1)^i (1 + i/(n-1))
    for (int i = lane; i < n; i += 32)
      x[i] = zmk((i % 2 ? -1.0 : 1.0) * (1.0 + (n > 1 ? (double)i / (n - 1) : 0.0)), 0.0);
    __syncwarp();
    warp_lu_solve(A, n, piv, x, false);
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += hypot(x[i].x, x[i].y);
    s = warp_sum(s);
    est = fmax(est, 2.0 * s / (3.0 * n));
    rcond = est > 0.0 ? (1.0 / est) / anorm : 0.0;
  }
  if (threadIdx.x == 0) {
    rcond_out[d.leaf] = rcond;
    if (!(rcond >= 1e-14)) atomicOr(flag, 1);
  }
}
#include "dense_lu.cuh"
