// lowrank.cu — K6: batched low-rank recompression, one CTA per problem.
//
// truncate_lowrank (hmatrix.py:412-426): QR(U), QR(V^T), SVD(R_u R_v^T), keep
// singular values s > tol * s_0 (at least 1), U' = Q_u W_r s_r, V' = Z_r Q_v^T.
// With in_v < 0 the input is a dense m x n block P and V = I (the full-SVD
// truncation of add_dense / _overwrite_block, hmatrix.py:605-609, 776-783).
// Ranks are device-resident: k is read from ranks[k_slot], r is written to
// ranks[out_slot]; the host never synchronises on them.
#include "hmatrix.h"
#include "lowrank.cuh"

namespace {

constexpr int SMEM_J = 64;   // cores up to 64 x 64 run the Jacobi SVD in shared memory
__device__ int prof_onesided_flag_dev = 0;

constexpr int KEXACT = 64;    // cores up to this size run in shared memory
constexpr int KRAND = 128;    // concatenated ranks above this use the randomized path
constexpr int RLMAX = 192;    // largest sketch (cores above SMEM_J run in global scratch)
constexpr int RL0 = 48;       // initial sketch size (accepts ranks <= 32 in one attempt)

__device__ __forceinline__ double hash_u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return (double)h * (2.0 / 4294967296.0) - 1.0;
}

// C (rows x l, col-major ldc) = op(A) * B where op selects how A (given col-major
// with leading dimension lda) is read: mode 0: C = A B (A rows x kk); mode 1:
// C = A^T B (A kk x rows); mode 2: C = A^H B; mode 3: C = conj(A) B.
__device__ __forceinline__ void cta_gemm_small(zc* C, int ldc, const zc* A, int lda, const zc* B,
                                               int ldb, int rows, int kk, int l, int mode) {
  for (int64_t e = threadIdx.x; e < (int64_t)rows * l; e += LR_NT) {
    const int i = (int)(e % rows), c = (int)(e / rows);
    zc s = zmk(0.0, 0.0);
    const zc* b = B + (int64_t)c * ldb;
    if (mode == 0) {
      for (int a = 0; a < kk; ++a) zfma(s, A[(int64_t)a * lda + i], b[a]);
    } else if (mode == 1) {
      const zc* ai = A + (int64_t)i * lda;
      for (int a = 0; a < kk; ++a) zfma(s, ai[a], b[a]);
    } else if (mode == 2) {
      const zc* ai = A + (int64_t)i * lda;
      for (int a = 0; a < kk; ++a) zfma(s, zconj(ai[a]), b[a]);
    } else {
      for (int a = 0; a < kk; ++a) zfma(s, zconj(A[(int64_t)a * lda + i]), b[a]);
    }
    C[e] = s;
  }
  __syncthreads();
}

// Randomized recompression of A = U V (U m x k, V = Vt^T), k > KEXACT:
// adaptive range finder with one power iteration, exact SVD of the l x l core.
// Accepts when the sketch shows >= 4 singular values below tol * s0, else
// doubles l (<= SMEM_J).  Returns false if l would exceed SMEM_J.
__device__ bool rand_truncate(const TruncDesc& d, zc* arena, zc* aout, int* ranks, int k, zc* sc,
                              int64_t scper, double tol, zc* rdv, double* kapv, double* sig,
                              int* order, zc* Ms, zc* Ws, double* red, int* flag,
                              unsigned long long* overflow, zc* gsm) {
  const int m = d.m, n = d.n;
  const zc* U = arena + d.in_u;
  const zc* Vt = arena + d.in_v;
  const int lmax = min(RLMAX, min(min(m, n), k));
  // first sketch sized from k: a concatenation [U1 U2] typically keeps ~k/2
  int l = min(lmax, max(RL0, ((k * 5 / 8 + 16 + 15) / 16) * 16));
  zc* Y = sc;                         // m x RLMAX (becomes Q's reflectors)
  zc* Z = Y + (int64_t)m * RLMAX;     // n x RLMAX (becomes Bt, then its reflectors)
  zc* T = Z + (int64_t)n * RLMAX;     // k x RLMAX
  zc* Om = T + (int64_t)k * RLMAX;    // n x RLMAX (Omega)
  zc* Mg = Om + (int64_t)(n + m) * RLMAX;   // RLMAX^2 core (global, for l > SMEM_J)
  zc* Wg = Mg + (int64_t)RLMAX * RLMAX;
  (void)scper;
  for (int attempt = 0;; ++attempt) {
    for (int64_t e = threadIdx.x; e < (int64_t)n * l; e += LR_NT)
      Om[e] = zmk(hash_u((uint32_t)(e % n), (uint32_t)(e / n), 2 * attempt),
                  hash_u((uint32_t)(e % n), (uint32_t)(e / n), 2 * attempt + 1));
    __syncthreads();
    cta_gemm_tiled(T, k, Vt, d.ldv, 1, Om, n, k, n, l, gsm);   // T = Vt^T Om      (k x l)
    cta_gemm_tiled(Y, m, U, d.ldu, 0, T, k, m, k, l, gsm);     // Y = U T          (m x l)
    // no power iteration: without re-orthonormalisation (A A^H)^q A Omega loses the
    // singular directions below eps^(1/(2q+1)) s0, which the truncation needs; a
    // 16-column oversampling margin is used instead
    for (int q = 0; q < 0; ++q) {
      cta_gemm_small(T, k, U, d.ldu, Y, m, k, m, l, 2);   // T = U^H Y        (k x l)
      cta_gemm_small(Z, n, Vt, d.ldv, T, k, n, k, l, 3);  // Z = conj(Vt) T   (n x l)
      cta_gemm_small(T, k, Vt, d.ldv, Z, n, k, n, l, 1);  // T = Vt^T Z       (k x l)
      cta_gemm_small(Y, m, U, d.ldu, T, k, m, k, l, 0);   // Y = U T          (m x l)
    }
    cta_qr(Y, m, l, m, rdv, kapv, red);
    // explicit Q (m x l) into Om (reuse, needs m <= n? use Z's region? ) -> stage in Om2
    zc* Q = Om + (int64_t)n * RLMAX;   // m x l (explicit Q)
    for (int64_t e = threadIdx.x; e < (int64_t)m * l; e += LR_NT) {
      const int i = (int)(e % m), c = (int)(e / m);
      Q[e] = zmk(i == c ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    cta_apply_q(Y, m, l, m, kapv, Q, l, m);
    // T = U^H Q (k x l);  Bt = Vt T (n x l)  [B = Q^H U V, Bt = B^T = Vt (U^T conj Q) = Vt conj(T)]
    cta_gemm_tiled(T, k, U, d.ldu, 2, Q, m, k, m, l, gsm);
    for (int64_t e = threadIdx.x; e < (int64_t)k * l; e += LR_NT) T[e] = zconj(T[e]);
    __syncthreads();
    cta_gemm_tiled(Z, n, Vt, d.ldv, 0, T, k, n, k, l, gsm);    // Z = Bt (n x l)
    // exact SVD of B = R2^T Q2^T:  QR(Bt) = Q2 R2, core M = R2^T (l x l)
    cta_qr(Z, n, l, n, rdv, kapv, red);
    zc* Mj = l <= SMEM_J ? Ms : Mg;
    zc* Wj = l <= SMEM_J ? Ws : Wg;
    for (int e = threadIdx.x; e < l * l; e += LR_NT) {
      const int a = e % l, b = e / l;   // M[a][b] = R2[b][a]
      Mj[e] = a == b ? rdv[a] : (a > b ? Z[(int64_t)a * n + b] : zmk(0.0, 0.0));
    }
    __syncthreads();
    cta_jacobi_hw(Mj, l, l, l, Wj, l, flag, red);
    for (int c = threadIdx.x; c < l; c += LR_NT) {
      double sq = 0.0;
      for (int i = 0; i < l; ++i) sq += zabs2(Mj[c * l + i]);
      sig[c] = sqrt(sq);
    }    __syncthreads();
    for (int c = threadIdx.x; c < l; c += LR_NT) {
      int pos = 0;
      for (int o = 0; o < l; ++o)
        if (sig[o] > sig[c] || (sig[o] == sig[c] && o < c)) ++pos;
      order[pos] = c;
    }
    __syncthreads();
    const double s0 = sig[order[0]];
    int r = 0;
    if (s0 > 0.0) {
      for (int c = 0; c < l; ++c)
        if (sig[c] > tol * s0) ++r;
      r = max(r, 1);
    }
    if (!(r <= l - 16) && l < min(min(m, n), k)) {   // sketch too small: grow or give up
      if (l >= lmax) return false;
      l = min(2 * l, lmax);
      __syncthreads();
      continue;
    }
    if (r > d.cap) {
      if (threadIdx.x == 0) atomicAdd(overflow, 1ull);
      r = d.cap;
    }
    // U' = Q (M W)[:, order[:r]]   (m x r)
    zc* Uo = aout + d.out_u;
    zc* Vo = aout + d.out_v;
    for (int64_t e = threadIdx.x; e < (int64_t)m * r; e += LR_NT) {
      const int i = (int)(e % m), c = (int)(e / m);
      const zc* mc = Mj + order[c] * l;
      zc s = zmk(0.0, 0.0);
      for (int a = 0; a < l; ++a) zfma(s, Q[(int64_t)a * m + i], mc[a]);
      Uo[e] = s;
    }
    // Vt' = Q2 [conj(W[:, order[:r]]); 0]
    for (int64_t e = threadIdx.x; e < (int64_t)n * r; e += LR_NT) {
      const int j = (int)(e % n), c = (int)(e / n);
      Vo[e] = j < l ? zconj(Wj[order[c] * l + j]) : zmk(0.0, 0.0);
    }
    __syncthreads();
    cta_apply_q(Z, n, l, n, kapv, Vo, r, n);
    if (threadIdx.x == 0) ranks[d.out_slot] = r;
    return true;
  }
}

__device__ void trunc_task(const TruncDesc d, zc* arena, zc* aout, int* ranks, zc* scratch,
                           int64_t scratch_per, int KS, double tol, unsigned long long* overflow,
                           unsigned long long* prof, unsigned char* smem_raw) {
  long long tc0 = clock64();
  __shared__ double red[LR_NW];
  __shared__ int flag;
  // per-CTA vectors (reflector scalars, singular values, order) live at the end of
  // the CTA's global scratch slot so the shared memory stays free for the cores
  zc* rd1 = scratch + (int64_t)blockIdx.x * scratch_per + (scratch_per - 4 * (int64_t)KS);
  zc* rd2 = rd1 + KS;
  double* kap1 = reinterpret_cast<double*>(rd2 + KS);
  double* kap2 = kap1 + KS;
  double* sig = kap2 + KS;
  int* order = reinterpret_cast<int*>(sig + KS);
  unsigned char* smem_base = smem_raw;

  const int m = d.m, n = d.n;
  if (d.skip_slot >= 0 && ranks[d.skip_slot] == 0) return;
  const int k = d.k_slot >= 0 ? ranks[d.k_slot] : d.k;
  const bool ident = d.in_v < 0;
  if (k <= 0 || m == 0 || n == 0) {
    if (threadIdx.x == 0) ranks[d.out_slot] = 0;
    return;
  }
  if (threadIdx.x == 0) flop_add(flops_trunc(m, n, k, ident));
  if (!ident && k > KRAND && min(m, n) > 2 * RL0) {
    zc* Ms = reinterpret_cast<zc*>(smem_base);
    zc* Ws = Ms + SMEM_J * SMEM_J;
    zc* sc = scratch + (int64_t)blockIdx.x * scratch_per;
    const long long tr0 = clock64();
    const bool ok = rand_truncate(d, arena, aout, ranks, k, sc, scratch_per, tol, rd1, kap1, sig, order, Ms,
                                  Ws, red, &flag, overflow, Ws + SMEM_J * SMEM_J);
    if (prof && threadIdx.x == 0) {
      atomicAdd(prof + (ok ? 6 : 8), 1ull);
      atomicAdd(prof + (ok ? 7 : 9), (unsigned long long)(clock64() - tr0));
    }
    if (ok) return;
    __syncthreads();
  }
  zc* U = arena + d.in_u;
  zc* Vt = ident ? nullptr : arena + d.in_v;
  const int kk1 = min(m, k);
  const int kk2 = ident ? n : min(n, k);
  zc* M = scratch + (int64_t)blockIdx.x * scratch_per;   // kk1 x kk2, ld kk1
  zc* W = M + (int64_t)kk1 * kk2;                         // kk2 x kk2

  const int ldu = d.ldu, ldv = d.ldv;
  if (ident) {
    cta_qr(U, m, k, ldu, rd1, kap1, red);
  } else {
    // the two QRs are independent: one per CTA half, named barriers 1 and 2
    __shared__ double red2[LR_NW];
    const int half = threadIdx.x / (LR_NT / 2);
    if (half == 0) half_qr(U, m, k, ldu, rd1, kap1, red2, 1);
    else half_qr(Vt, n, k, ldv, rd2, kap2, red2 + LR_NW / 2, 2);
    __syncthreads();
  }
  long long tc1 = clock64();
  // M = R1 R2^T (R2 = I for the dense mode)
  for (int e = threadIdx.x; e < kk1 * kk2; e += LR_NT) {
    const int a = e % kk1, b = e / kk1;
    zc s = zmk(0.0, 0.0);
    if (ident) {
      s = b == a ? rd1[a] : (b > a ? U[(int64_t)b * ldu + a] : zmk(0.0, 0.0));
    } else {
      for (int c = max(a, b); c < k; ++c) {
        const zc r1 = c == a ? rd1[a] : U[(int64_t)c * ldu + a];
        const zc r2 = c == b ? rd2[b] : Vt[(int64_t)c * ldv + b];
        s = zadd(s, zmul(r1, r2));
      }
    }
    M[(int64_t)b * kk1 + a] = s;
  }
  __syncthreads();
  long long tc2 = clock64();
  int sweeps = 0;
  bool precond = false;
  zc* Ms = nullptr;
  zc* Bs = nullptr;
  zc* Js = nullptr;
  double* kapM = nullptr;
  if (kk1 >= kk2 && !ident) {
    // QR-preconditioned one-sided Jacobi (M = Q_M R, Jacobi on R^H): a few sweeps
    // instead of ~11.  Cores up to 64 x 64 live in shared memory, larger ones in
    // the CTA's global scratch slot (after M and W).
    precond = true;
    const bool small = kk1 <= SMEM_J && kk2 <= SMEM_J;
    if (small) {
      Ms = reinterpret_cast<zc*>(smem_base);
      Bs = Ms + SMEM_J * SMEM_J;
      Js = Bs + SMEM_J * SMEM_J;
    } else {
      Ms = W + (int64_t)KS * KS;
      Bs = Ms + (int64_t)KS * KS;
      Js = Bs + (int64_t)KS * KS;
    }
    zc* rdQ = reinterpret_cast<zc*>(Js + (small ? SMEM_J * SMEM_J : (int64_t)KS * KS));
    double* kpQ = reinterpret_cast<double*>(rdQ + KS);
    if (small) {   // the small-core scalars stay in shared memory
      rdQ = reinterpret_cast<zc*>(Js + SMEM_J * SMEM_J);
      kpQ = reinterpret_cast<double*>(rdQ + SMEM_J);
    }
    kapM = kpQ;
    for (int e = threadIdx.x; e < kk1 * kk2; e += LR_NT) Ms[e] = M[e];
    __syncthreads();
    cta_qr(Ms, kk1, kk2, kk1, rdQ, kapM, red);
    // A = R^H (kk2 x kk2): A[i][j] = conj(R[j][i]), R upper (diag rdQ, strict upper in Ms)
    for (int e = threadIdx.x; e < kk2 * kk2; e += LR_NT) {
      const int i = e % kk2, j = e / kk2;
      zc v = zmk(0.0, 0.0);
      if (i == j) v = zconj(rdQ[i]);
      else if (i > j) v = zconj(Ms[i * kk1 + j]);
      Bs[j * kk2 + i] = v;
    }
    __syncthreads();
    sweeps = cta_jacobi_hw(Bs, kk2, kk2, kk2, Js, kk2, &flag, red);
    for (int c = threadIdx.x; c < kk2; c += LR_NT) {
      double sq = 0.0;
      for (int i = 0; i < kk2; ++i) sq += zabs2(Bs[c * kk2 + i]);
      sig[c] = sqrt(sq);
    }
    __syncthreads();
  } else if (kk1 <= SMEM_J && kk2 <= SMEM_J) {
    // one-sided Jacobi with M and W resident in shared memory
    zc* Mss = reinterpret_cast<zc*>(smem_base);
    zc* Wss = Mss + SMEM_J * SMEM_J;
    for (int e = threadIdx.x; e < kk1 * kk2; e += LR_NT) Mss[e] = M[e];
    __syncthreads();
    sweeps = cta_jacobi_hw(Mss, kk1, kk2, kk1, Wss, kk2, &flag, red);
    for (int c = threadIdx.x; c < kk2; c += LR_NT) {
      double sq = 0.0;
      for (int i = 0; i < kk1; ++i) sq += zabs2(Mss[c * kk1 + i]);
      sig[c] = sqrt(sq);
    }
    for (int e = threadIdx.x; e < kk1 * kk2; e += LR_NT) M[e] = Mss[e];
    for (int e = threadIdx.x; e < kk2 * kk2; e += LR_NT) W[e] = Wss[e];
    __syncthreads();
  } else {
    sweeps = cta_jacobi(M, kk1, kk2, kk1, W, kk2, &flag, red);
    // singular values and descending order (stable)
    for (int c = threadIdx.x; c < kk2; c += LR_NT) {
      double s = 0.0;
      for (int i = 0; i < kk1; ++i) s += zabs2(M[(int64_t)c * kk1 + i]);
      sig[c] = sqrt(s);
    }
    __syncthreads();
  }
  long long tc3 = clock64();
  for (int c = threadIdx.x; c < kk2; c += LR_NT) {
    int pos = 0;
    for (int o = 0; o < kk2; ++o)
      if (sig[o] > sig[c] || (sig[o] == sig[c] && o < c)) ++pos;
    order[pos] = c;
  }
  __syncthreads();
  const double s0 = sig[order[0]];
  int r = 0;
  if (s0 > 0.0) {
    for (int c = 0; c < kk2; ++c)
      if (sig[c] > tol * s0) ++r;
    r = max(r, 1);
  }
  if (r > d.cap) {
    if (threadIdx.x == 0) atomicAdd(overflow, 1ull);
    r = d.cap;
  }
  zc* Uo = aout + d.out_u;
  zc* Vo = aout + d.out_v;
  if (precond) {
    // U' = Q1 Q_M [J_r Sigma_r; 0],  Vt' = Q2 [conj(B_r) / sigma; 0]
    for (int e = threadIdx.x; e < m * r; e += LR_NT) {
      const int i = e % m, l = e / m;
      Uo[(int64_t)l * m + i] = i < kk2 ? zscale(Js[order[l] * kk2 + i], sig[order[l]]) : zmk(0.0, 0.0);
    }
    for (int e = threadIdx.x; e < n * r; e += LR_NT) {
      const int j = e % n, l = e / n;
      Vo[(int64_t)l * n + j] =
          j < kk2 ? zscale(zconj(Bs[order[l] * kk2 + j]), 1.0 / sig[order[l]]) : zmk(0.0, 0.0);
    }
    __syncthreads();
    cta_apply_q(Ms, kk1, kk2, kk1, kapM, Uo, r, m);   // Q_M on the top kk1 rows
  } else {
    // U' = Q1 [ (M W)[:, order[:r]] ; 0 ]
    for (int e = threadIdx.x; e < m * r; e += LR_NT) {
      const int i = e % m, l = e / m;
      Uo[(int64_t)l * m + i] = i < kk1 ? M[(int64_t)order[l] * kk1 + i] : zmk(0.0, 0.0);
    }
    // Vt' = Q2 [ conj(W[:, order[:r]]) ; 0 ]
    for (int e = threadIdx.x; e < n * r; e += LR_NT) {
      const int j = e % n, l = e / n;
      Vo[(int64_t)l * n + j] = j < kk2 ? zconj(W[(int64_t)order[l] * kk2 + j]) : zmk(0.0, 0.0);
    }
  }
  __syncthreads();
  if (ident) {
    cta_apply_q(U, m, kk1, ldu, kap1, Uo, r, m);
  } else {
    const int half = threadIdx.x / (LR_NT / 2);
    if (half == 0) half_apply_q(U, m, kk1, ldu, kap1, Uo, r, m, 1);
    else half_apply_q(Vt, n, kk2, ldv, kap2, Vo, r, n, 2);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ranks[d.out_slot] = r;
    if (prof) {
      long long tc4 = clock64();
      atomicAdd(prof + 0, (unsigned long long)(tc1 - tc0));
      atomicAdd(prof + 1, (unsigned long long)(tc2 - tc1));
      atomicAdd(prof + 2, (unsigned long long)(tc3 - tc2));
      atomicAdd(prof + 3, (unsigned long long)(tc4 - tc3));
      atomicAdd(prof + 4, 1ull);
      atomicAdd(prof + 5, (unsigned long long)sweeps);
      const bool sm = kk1 <= SMEM_J && kk2 <= SMEM_J;
      atomicAdd(prof + (sm ? 10 : 12), 1ull);
      atomicAdd(prof + (sm ? 11 : 13), (unsigned long long)(tc4 - tc0));
    }
  }
}

// idx == nullptr: CTA b handles descs[b].  Deferred mode (problems the blocked
// kernel could not take): idx[0] = count, idx[1 + i] = descriptor index; the
// CTAs stride over the list.
__global__ void __launch_bounds__(LR_NT) k_truncate(zc* arena, zc* aout, int* ranks,
                                                    const TruncDesc* __restrict__ descs,
                                                    zc* scratch, int64_t scratch_per, int KS,
                                                    double tol, unsigned long long* overflow,
                                                    unsigned long long* prof, const int* idx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (!idx) {
    trunc_task(descs[blockIdx.x], arena, aout, ranks, scratch, scratch_per, KS, tol, overflow, prof, smem_raw);
    return;
  }
  const int cnt = idx[0];
  for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
    trunc_task(descs[idx[1 + i]], arena, aout, ranks, scratch, scratch_per, KS, tol, overflow, prof, smem_raw);
    __syncthreads();
  }
}

}  // namespace

unsigned long long* g_trunc_prof = nullptr;
bool g_ws_tight = false;   // debug cycle counters (CBIE_PROFILE)

void trunc_prof_enable(bool on, int onesided) {
  if (on && !g_trunc_prof) {
    cudaMalloc(&g_trunc_prof, 32 * sizeof(unsigned long long));
    cudaMemset(g_trunc_prof, 0, 32 * sizeof(unsigned long long));
  }
  cudaMemcpyToSymbol(prof_onesided_flag_dev, &onesided, sizeof(int));
}
void trunc_prof_read(unsigned long long* h) {
  if (g_trunc_prof) cudaMemcpy(h, g_trunc_prof, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}

// unblocked kernel over a device-side list of problems (list[0] = count): strided grid
static void launch_unblocked_list(zc* arena, zc* arena_out, int* ranks, const TruncDesc* d_desc, int nd,
                                  int kmax, int64_t per, double tol, unsigned long long* overflow,
                                  TruncWork& work, cudaStream_t s, const int* list) {
  DBuf<zc>& dscratch = work.dscratch;
  // one CTA per SM (grid-stride over the list) unless the scratch would exceed 4 GB
  const int64_t cap_mem = std::max<int64_t>(ws_tight() ? 1 : 74, (int64_t)ws_cap(4) / std::max<int64_t>(per * (int64_t)sizeof(zc), 1));
  const int grid = (int)std::min<int64_t>(nd, std::min<int64_t>(148, cap_mem));
  if (dscratch.n < (size_t)grid * per) dscratch.alloc((size_t)grid * per);
  const size_t smem = std::max((size_t)SMEM_J * SMEM_J * 3 * sizeof(zc) + SMEM_J * (sizeof(zc) + sizeof(double)),
                               (size_t)SMEM_J * SMEM_J * 2 * sizeof(zc) +
                                   (size_t)TG_K * (TG_R + 1 + 65) * sizeof(zc));
  CK(cudaFuncSetAttribute(k_truncate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_truncate<<<grid, LR_NT, smem, s>>>(arena, arena_out, ranks, d_desc, dscratch.p, per, kmax, tol, overflow,
                                       g_trunc_prof, list);
  CKL();
}

namespace {
// split problems by device-side rank: k <= kg (and no-ops) -> la (Gram kernel), the rest -> lb
// (i >= nsmall: Gram problems of the large blocks -> lg, when lg != nullptr)
// One CTA: the Gram lists (la, lg) come out ordered by estimated cost, heaviest first
// (counting sort over RB cost buckets), so the long problems of a launch start first and
// the short ones fill the SMs behind them; with arrival order a multi-stage 1536-row
// problem could start in the last wave and the whole group waited for it.
constexpr int RB = 16;
__global__ void __launch_bounds__(256) k_route(const int* __restrict__ ranks, const TruncDesc* __restrict__ ds, int nd,
                                               int kg, int* la, int* lb, int* lg, int nsmall,
                                               unsigned long long* overflow) {
  __shared__ int cnt[2][RB], pos[2][RB];
  for (int e = threadIdx.x; e < 2 * RB; e += blockDim.x) (&cnt[0][0])[e] = 0;
  __syncthreads();
  auto classify = [&](int i, int& list, int& bucket) {
    const TruncDesc& d = ds[i];
    const int k = trunc_k(d, ranks);
    const bool skip = d.skip_slot >= 0 && ranks[d.skip_slot] == 0;
    if (skip || k <= kg) {
      list = (lg && i >= nsmall) ? 1 : 0;
      // ~ stages x (k x k work + row streams): k = 64, m + n = 3072 -> 128
      const int cost = skip ? 0 : ((k + 15) / 16) * ((d.m + d.n) / 128 + 8);
      bucket = RB - 1 - min(RB - 1, cost / 16);
    } else {
      list = d.in_u2 >= 0 ? 3 : 2;
      bucket = 0;
    }
  };
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    int l, b;
    classify(i, l, b);
    if (l < 2) atomicAdd(&cnt[l][b], 1);
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    int acc = 0;
    for (int b = 0; b < RB; ++b) {
      pos[threadIdx.x][b] = acc;
      acc += cnt[threadIdx.x][b];
    }
    int* l = threadIdx.x == 0 ? la : lg;
    if (l) l[0] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    int l, b;
    classify(i, l, b);
    if (l < 2) {
      int* dst = l == 0 ? la : lg;
      dst[1 + atomicAdd(&pos[l][b], 1)] = i;
    } else if (l == 3) {
      // two-source inputs exist only for the Gram path: counted as a clipped truncation, the
      // factorisation is redone with materialised concatenations (cbie_hlu_factor)
      atomicAdd(overflow, 1ull);
    } else {
      lb[1 + atomicAdd(lb, 1)] = i;
    }
  }
}
}  // namespace

// Householder kernels over a device-side list (count in list[0]): blocked kernel for
// k <= 128 and max(m, n) <= 384 (its own hand-offs), unblocked for the rest
static void householder_list(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, int kmax, double tol,
                             unsigned long long* overflow, TruncWork& w, cudaStream_t st, int kc_max, int mn_max,
                             const int* list, zc* aout) {
  bool done = false;
  if (mn_max <= 384) {
    int* dfr = nullptr;
    if (kc_max > 128) {
      if (w.defer.n < (size_t)nd + 1) w.defer.alloc(std::max<size_t>(nd + 1, 4096));
      dfr = w.defer.p;
      CK(cudaMemsetAsync(dfr, 0, sizeof(int), st));
    }
    launch_truncate_blocked(arena, ranks, d_desc, nd, tol, overflow, w.scratch, st, kc_max, mn_max, aout, dfr,
                            list);
    if (!dfr) done = true;
    else list = dfr;
  }
  if (!done) {
    kmax = std::max(std::max(kmax, 1), RLMAX);
    const int64_t per = std::max<int64_t>((int64_t)kmax * kmax * 5 + 2 * (int64_t)kmax,
                                          (int64_t)RLMAX * (4 * (int64_t)mn_max + kc_max + 1) +
                                              2 * (int64_t)RLMAX * RLMAX) +
                        4 * (int64_t)kmax;
    launch_unblocked_list(arena, aout, ranks, d_desc, nd, kmax, per, tol, overflow, w, st, list);
  }
}

// Gram kernel for ranks <= 64 and, multi-stage, up to 256 (its failures then go to
// the Householder kernels on the same stream); larger ranks to the Householder
// kernels on the second stream, concurrently.
void launch_truncate_routed(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, int kmax, double tol,
                            unsigned long long* overflow, TruncWork& work, cudaStream_t s, int kc_max,
                            int mn_max, TruncWork* work2, cudaStream_t s2, zc* arena_out, const TruncBig* big) {
  if (nd == 0) return;
  zc* aout = arena_out ? arena_out : arena;
  const bool multi = getenv("CBIE_NO_MULTISTAGE") == nullptr;
  const int kg = multi ? 256 : 64;
  // large blocks in their own cluster launch on s3, concurrently with the small ones
  const bool split = big && big->s3 && big->work3 && big->nsmall >= 0 && big->nsmall < nd && big->cbig > 1 &&
                     getenv("CBIE_NO_CLUSTER") == nullptr;
  cudaEvent_t f3 = nullptr, j3 = nullptr;
  if (split) {
    CK(cudaEventCreateWithFlags(&f3, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&j3, cudaEventDisableTiming));
  }
  if (kc_max <= 64) {   // no capacity can exceed the single-stage Gram path
    if (!split) {
      launch_truncate_gram(arena, ranks, d_desc, nd, tol, overflow, work.scratch, s, aout, nullptr);
      return;
    }
    CK(cudaEventRecord(f3, s));
    CK(cudaStreamWaitEvent(big->s3, f3, 0));
    launch_truncate_gram(arena, ranks, d_desc + big->nsmall, nd - big->nsmall, tol, overflow, big->work3->scratch,
                         big->s3, aout, nullptr, nullptr, 0, big->cbig);
    launch_truncate_gram(arena, ranks, d_desc, big->nsmall, tol, overflow, work.scratch, s, aout, nullptr);
    CK(cudaEventRecord(j3, big->s3));
    CK(cudaStreamWaitEvent(s, j3, 0));
    cudaEventDestroy(f3);
    cudaEventDestroy(j3);
    return;
  }
  TruncWork& wb = work2 ? *work2 : work;
  cudaStream_t sb = work2 && s2 ? s2 : s;
  // lists: la (Gram), lb (Householder, stream sb), lf (Gram failures, stream s), lg (Gram,
  // large blocks, stream s3)
  if (work.gdefer.n < 4 * (size_t)nd + 4) work.gdefer.alloc(std::max<size_t>(4 * nd + 4, 4 * 4096));
  int* la = work.gdefer.p;
  int* lf = la + nd + 1;
  int* lb = lf + nd + 1;
  int* lg = lb + nd + 1;
  CK(cudaMemsetAsync(la, 0, sizeof(int) * (2 * nd + 2), s));   // counts of la and lf (and la's payload)
  CK(cudaMemsetAsync(lb, 0, sizeof(int), s));
  CK(cudaMemsetAsync(lg, 0, sizeof(int), s));
  // multi-stage on: the (rare) problems beyond its 256 columns join the Gram failures'
  // list and run with them after the Gram launches -- one Householder pass per group
  // instead of two mostly empty ones
  k_route<<<1, 256, 0, s>>>(ranks, d_desc, nd, kg, la, multi ? lf : lb,
                                                          split ? lg : nullptr, split ? big->nsmall : nd, overflow);
  CKL();
  cudaEvent_t fork = nullptr, join = nullptr;
  const bool two = sb != s && kc_max > kg && !multi;
  if (two) {
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    CK(cudaEventRecord(fork, s));
    CK(cudaStreamWaitEvent(sb, fork, 0));
  }
  if (split) {
    CK(cudaEventRecord(f3, s));
    CK(cudaStreamWaitEvent(big->s3, f3, 0));
    launch_truncate_gram(arena, ranks, d_desc, nd - big->nsmall, tol, overflow, big->work3->scratch, big->s3, aout,
                         multi ? lf : nullptr, lg, multi ? mn_max : 0, big->cbig);
  }
  if (kc_max > kg && !multi)
    householder_list(arena, ranks, d_desc, nd, kmax, tol, overflow, two ? wb : work, two ? sb : s, kc_max, mn_max,
                     lb, aout);
  launch_truncate_gram(arena, ranks, d_desc, split ? big->nsmall : nd, tol, overflow, work.scratch, s, aout,
                       multi ? lf : nullptr, la, multi ? (split ? big->mn_small : mn_max) : 0);
  if (two) {
    CK(cudaEventRecord(join, sb));
    CK(cudaStreamWaitEvent(s, join, 0));
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
  }
  if (split) {
    CK(cudaEventRecord(j3, big->s3));
    CK(cudaStreamWaitEvent(s, j3, 0));
    cudaEventDestroy(f3);
    cudaEventDestroy(j3);
  }
  // multi-stage failures (kept rank filled the Gram capacity), after the joins so that
  // they reuse the Householder workspaces of the second stream
  if (multi) householder_list(arena, ranks, d_desc, nd, kmax, tol, overflow, wb, s, kc_max, mn_max, lf, aout);
}

void launch_truncate(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, int kmax, double tol,
                     unsigned long long* overflow, TruncWork& work, cudaStream_t s, int kc_max,
                     int mn_max, zc* arena_out, int flags) {
  DBuf<zc>& scratch = work.scratch;
  if (!arena_out) arena_out = arena;
  if (nd == 0) return;
  DBuf<int>& defer = work.defer;   // deferred-problem list of the blocked kernel
  int* dfr = nullptr;
  if (flags & TRUNC_NO_DENSE) {
    if (kc_max > 128) {
      if (defer.n < (size_t)nd + 1) defer.alloc(std::max<size_t>(nd + 1, 4096));
      CK(cudaMemsetAsync(defer.p, 0, sizeof(int), s));
      dfr = defer.p;
    }
    if (launch_truncate_blocked(arena, ranks, d_desc, nd, tol, overflow, scratch, s, kc_max, mn_max,
                                arena_out, dfr)) {
      if (!dfr) return;
    } else {
      dfr = nullptr;
    }
  }
  kmax = std::max(std::max(kmax, 1), RLMAX);
  const int64_t per = std::max<int64_t>((int64_t)kmax * kmax * 5 + 2 * (int64_t)kmax,
                                        (int64_t)RLMAX * (4 * (int64_t)mn_max + kc_max + 1) +
                                            2 * (int64_t)RLMAX * RLMAX) +
                      4 * (int64_t)kmax;
  // waves keep the Jacobi scratch bounded (<= 1 GiB); the buffer is reused across calls
  if (dfr) {   // the blocked kernel's leftovers: a strided grid over the deferred list
    launch_unblocked_list(arena, arena_out, ranks, d_desc, nd, kmax, per, tol, overflow, work, s, dfr);
    return;
  }
  const int wave = (int)std::max<int64_t>(1, (int64_t)ws_cap(1) / (per * (int64_t)sizeof(zc)));
  const size_t need = (size_t)std::min(wave, nd) * per;
  if (scratch.n < need) scratch.alloc(need);
  // exact path: Ms, Bs, Js (3 x 64^2) + rdM/kapM; randomized path: Ms, Ws + GEMM tiles
  const size_t smem = std::max((size_t)SMEM_J * SMEM_J * 3 * sizeof(zc) + SMEM_J * (sizeof(zc) + sizeof(double)),
                               (size_t)SMEM_J * SMEM_J * 2 * sizeof(zc) +
                                   (size_t)TG_K * (TG_R + 1 + 65) * sizeof(zc));
  if (smem > 232448 - 2048) throw cbie_error(CBIE_EINVALID, "truncation dimension too large");
  CK(cudaFuncSetAttribute(k_truncate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int b0 = 0; b0 < nd; b0 += wave) {
    int nb = std::min(wave, nd - b0);
    k_truncate<<<nb, LR_NT, smem, s>>>(arena, arena_out, ranks, d_desc + b0, scratch.p, per, kmax, tol,
                                       overflow, g_trunc_prof, nullptr);
    CKL();
  }
}

extern "C" int cbie_lowrank_truncate(cbie_ctx* c, const cbie_c128* U, int m, int k,
                                     const cbie_c128* V, int n, double tol, int* r,
                                     cbie_c128* Uo, cbie_c128* Vo) {
  try {
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const bool dense = V == nullptr;
    if (dense) k = n;
    if (m <= 0 || n <= 0 || k <= 0) throw cbie_error(CBIE_EINVALID, "empty factors");
    const int cap = std::min(std::min(m, n), k);
    // arena: U col-major m x k | Vt col-major n x k | Uo m x cap | Vto n x cap
    std::vector<zc> h((size_t)(m + n) * k + (size_t)(m + n) * cap);
    const zc* hu = reinterpret_cast<const zc*>(U);
    for (int i = 0; i < m; ++i)
      for (int l = 0; l < k; ++l) h[(size_t)l * m + i] = hu[(size_t)i * k + l];
    if (!dense) {
      const zc* hv = reinterpret_cast<const zc*>(V);
      for (int l = 0; l < k; ++l)
        for (int j = 0; j < n; ++j) h[(size_t)m * k + (size_t)l * n + j] = hv[(size_t)l * n + j];
    }
    DBuf<zc> ar;
    ar.upload(h, s);
    DBuf<int> ranks;
    std::vector<int> r0(2, 0);
    ranks.upload(r0, s);
    TruncDesc d;
    d.in_u = 0;
    d.in_v = dense ? -1 : (int64_t)m * k;
    d.ldu = m;
    d.ldv = n;
    d.skip_slot = -1;
    d.out_u = (int64_t)(m + n) * k;
    d.out_v = d.out_u + (int64_t)m * cap;
    d.m = m;
    d.n = n;
    d.k = k;
    d.k_slot = -1;
    d.cap = cap;
    d.out_slot = 0;
    DBuf<TruncDesc> dd;
    dd.upload(&d, 1, s);
    DBuf<unsigned long long> ovf;
    ovf.alloc(1);
    CK(cudaMemsetAsync(ovf.p, 0, 8, s));
    TruncWork work;
    const int kmax = dense ? std::max(m, n) : std::min(k, std::max(m, n));
    // same routing as the H-LU executor (hlu.cu make_plan): factor form at tol >= 1e-5
    // takes the Gram path (ranks <= 64) and its hand-offs
    if (!dense && tol >= 1e-5 && getenv("CBIE_NO_GRAM") == nullptr)
      launch_truncate_routed(ar.p, ranks.p, dd.p, 1, kmax, tol, ovf.p, work, s, k, std::max(m, n));
    else
      launch_truncate(ar.p, ranks.p, dd.p, 1, kmax, tol, ovf.p, work, s, k, std::max(m, n), nullptr,
                      dense ? 0 : TRUNC_NO_DENSE);
    int rr = 0;
    CK(cudaMemcpyAsync(&rr, ranks.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    std::vector<zc> out((size_t)(m + n) * cap);
    CK(cudaMemcpyAsync(out.data(), ar.p + d.out_u, sizeof(zc) * out.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *r = rr;
    zc* uo = reinterpret_cast<zc*>(Uo);
    zc* vo = reinterpret_cast<zc*>(Vo);
    for (int i = 0; i < m; ++i)
      for (int l = 0; l < rr; ++l) uo[(size_t)i * rr + l] = out[(size_t)l * m + i];
    for (int l = 0; l < rr; ++l)
      for (int j = 0; j < n; ++j) vo[(size_t)l * n + j] = out[(size_t)m * cap + (size_t)l * n + j];
  } catch (const cbie_error& e) {
    c->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}

// ---------------------------------------------------------------------------
// Dense -> low rank by an adaptive randomized range finder (one CTA per task).
// P (m x n, col-major, ld) ~= Q B, Q (m x l) orthonormal, B = Q^H P, with one
// power iteration; l doubles until the Frobenius residual
// sqrt(|P|_F^2 - |B|_F^2) <= tol * s0_lb (s0_lb = largest row norm of B, a
// lower bound of s_0).  Replaces the full SVD of dense updates landing in
// low-rank targets (hmatrix.py:605-609); the result (U = Q, Vt = B^T, rank l)
// is truncated exactly by the following add_lowrank recompression.
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ double hash_unit(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return (double)h * (2.0 / 4294967296.0) - 1.0;
}

// The three range-finder products of the first attempt for ALL tasks of a launch,
// 32 x 32 output tiles over the whole GPU (the per-task kernel below then starts from
// Y; a task has ~1 CTA otherwise, ~20 tasks per launch on 148 SMs):
//   mode 0: Y = P Omega,  mode 1: Z = P^H Y,  mode 2: Y = P Z
// (Omega from the same hash as the per-task kernel; tasks on the exact path skip.)
__global__ void __launch_bounds__(256) k_dlr_range(const zc* __restrict__ arena, const DenseLRDesc* __restrict__ ds,
                                                   zc* scratch, int64_t scratch_per, int mode) {
  const DenseLRDesc d = ds[blockIdx.z];
  const int m = d.m, n = d.n, ld = d.ld;
  const int full = min(m, n);
  int l = min(d.l0, full);
  const bool exact = 2 * l > full;
  if (exact) l = full;
  if (exact && l == n) return;
  const zc* P = arena + d.p;
  zc* Y = scratch + (int64_t)blockIdx.z * scratch_per;
  zc* Z = Y + (int64_t)m * d.cap;
  const int rows = mode == 1 ? n : m, inner = mode == 1 ? m : n;
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (i0 >= rows || j0 >= l) return;
  __shared__ zc sA[16][33];
  __shared__ zc sB[16][33];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  zc acc[2][2] = {{zmk(0, 0), zmk(0, 0)}, {zmk(0, 0), zmk(0, 0)}};
  for (int k0 = 0; k0 < inner; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 32; e += 256) {
      const int kk = e / 32, ii = e % 32;
      const int gi = i0 + ii, gk = k0 + kk, gj = j0 + ii;
      zc a = zmk(0, 0), b = zmk(0, 0);
      if (gi < rows && gk < inner) a = mode == 1 ? zconj(P[(int64_t)gi * ld + gk]) : P[(int64_t)gk * ld + gi];
      if (gj < l && gk < inner) {
        if (mode == 0) b = zmk(hash_unit((uint32_t)gk, (uint32_t)gj, 0), hash_unit((uint32_t)gk, (uint32_t)gj, 1));
        else if (mode == 1) b = Y[(int64_t)gj * m + gk];
        else b = Z[(int64_t)gj * n + gk];
      }
      sA[kk][ii] = a;
      sB[kk][ii] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const zc a0 = sA[kk][ty], a1 = sA[kk][ty + 16];
      const zc b0 = sB[kk][tx], b1 = sB[kk][tx + 16];
      zfma(acc[0][0], a0, b0);
      zfma(acc[0][1], a0, b1);
      zfma(acc[1][0], a1, b0);
      zfma(acc[1][1], a1, b1);
    }
    __syncthreads();
  }
  zc* C = mode == 1 ? Z : Y;
  const int ldc = mode == 1 ? n : m;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
      if (gi < rows && gj < l) C[(int64_t)gj * ldc + gi] = acc[a][b];
    }
}

__global__ void __launch_bounds__(LR_NT) k_dense_lr(zc* arena, int* ranks,
                                                    const DenseLRDesc* __restrict__ ds,
                                                    zc* scratch, int64_t scratch_per, int pre) {
  const DenseLRDesc d = ds[blockIdx.x];
  const int m = d.m, n = d.n, ld = d.ld;
  const zc* P = arena + d.p;
  zc* U = arena + d.out_u;   // m x cap
  zc* Vt = arena + d.out_v;  // n x cap
  zc* Y = scratch + (int64_t)blockIdx.x * scratch_per;   // m x cap
  zc* Z = Y + (int64_t)m * d.cap;                          // n x cap
  __shared__ double red[LR_NW];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* rd = reinterpret_cast<zc*>(smem_raw);
  double* kap = reinterpret_cast<double*>(rd + d.cap);
  zc* gsm = reinterpret_cast<zc*>((reinterpret_cast<uintptr_t>(kap + d.cap) + 15) & ~uintptr_t(15));
  double pf2 = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)m * n; e += LR_NT)
    pf2 += zabs2(P[(e / m) * ld + e % m]);
  pf2 = block_sum(pf2, red);
  if (pf2 == 0.0) {
    if (threadIdx.x == 0) ranks[d.out_slot] = 0;
    return;
  }
  const int full = min(m, n);
  int l = min(d.l0, full);
  for (int attempt = 0;; ++attempt) {
    const bool exact = 2 * l > full;
    if (exact) l = full;
    if (exact && l == n) {
      for (int64_t e = threadIdx.x; e < (int64_t)m * l; e += LR_NT)
        Y[e] = P[(e / m) * ld + e % m];
    } else if (pre && attempt == 0) {
      // Y = P (P^H (P Omega)) already in scratch (k_dlr_range)
    } else {
      zc* Om = Z;   // Omega (n x l) staged in the Z region, then Z reused below
      for (int64_t e = threadIdx.x; e < (int64_t)n * l; e += LR_NT)
        Om[e] = zmk(hash_unit((uint32_t)(e % n), (uint32_t)(e / n), 2 * attempt),
                    hash_unit((uint32_t)(e % n), (uint32_t)(e / n), 2 * attempt + 1));
      __syncthreads();
      cta_gemm_tiled(Y, m, P, ld, 0, Om, n, m, n, l, gsm);   // Y = P Omega
      cta_gemm_tiled(Z, n, P, ld, 2, Y, m, n, m, l, gsm);    // Z = P^H Y
      cta_gemm_tiled(Y, m, P, ld, 0, Z, n, m, n, l, gsm);    // Y = P Z
    }
    __syncthreads();
    if (threadIdx.x == 0)   // range finder GEMMs, QR + Q formation, B = Q^H P
      flop_add((exact && l == n ? 0.0 : 24.0 * m * (double)n * l) + flops_qr(m, min(m, l)) +
               8.0 * m * (double)n * min(m, l));
    cta_qr(Y, m, l, m, rd, kap, red);
    const int lq = min(m, l);
    // Q = H_0..H_{lq-1} [I; 0] into U
    for (int64_t e = threadIdx.x; e < (int64_t)m * lq; e += LR_NT) {
      const int i = (int)(e % m), c = (int)(e / m);
      U[e] = zmk(i == c ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    cta_apply_q(Y, m, lq, m, kap, U, lq, m);
    // Vt = P^T conj(Q)  (B = Q^H P, Vt = B^T):  Vt = conj(P^H Q)
    cta_gemm_tiled(Vt, n, P, ld, 2, U, m, n, m, lq, gsm);
    double bf2 = 0.0;
    for (int64_t e = threadIdx.x; e < (int64_t)n * lq; e += LR_NT) {
      const zc v = zconj(Vt[e]);
      Vt[e] = v;
      bf2 += zabs2(v);
    }
    bf2 = block_sum(bf2, red);
    double rowmax = 0.0;
    for (int c = threadIdx.x; c < lq; c += LR_NT) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += zabs2(Vt[(int64_t)c * n + j]);
      rowmax = fmax(rowmax, s);
    }
    for (int o = 16; o > 0; o >>= 1) rowmax = fmax(rowmax, __shfl_xor_sync(0xffffffffu, rowmax, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rowmax;
    __syncthreads();
    double s0 = 0.0;
    for (int w = 0; w < LR_NW; ++w) s0 = fmax(s0, red[w]);
    __syncthreads();
    s0 = sqrt(s0);
    const double resid = sqrt(fmax(pf2 - bf2, 0.0));
    if (exact || resid <= d.tol * s0 || 2 * l > d.cap) {
      if (threadIdx.x == 0) ranks[d.out_slot] = lq;
      return;
    }
    l *= 2;
    __syncthreads();
  }
}
}  // namespace

void launch_dense_lr(zc* arena, int* ranks, const DenseLRDesc* d_desc, int nd, int max_m, int max_n,
                     int max_cap, DBuf<zc>& scratch, cudaStream_t s) {
  if (nd == 0) return;
  const int64_t per = (int64_t)(max_m + max_n) * max_cap;
  const int wave = (int)std::max<int64_t>(1, (int64_t)ws_cap(1) / (per * (int64_t)sizeof(zc)));
  const size_t need = (size_t)std::min(wave, nd) * per;
  if (scratch.n < need) scratch.alloc(need);
  const size_t smem = (size_t)max_cap * (sizeof(zc) + sizeof(double)) + 32 +
                      (size_t)TG_K * (TG_R + 1 + 65) * sizeof(zc);
  CK(cudaFuncSetAttribute(k_dense_lr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int rmax = std::max(max_m, max_n), lmax = std::min(max_m, max_n);
  for (int b0 = 0; b0 < nd; b0 += wave) {
    int nb = std::min(wave, nd - b0);
    for (int mode = 0; mode < 3; ++mode) {
      k_dlr_range<<<dim3(ceil_div(rmax, 32), ceil_div(lmax, 32), nb), 256, 0, s>>>(arena, d_desc + b0, scratch.p,
                                                                                    per, mode);
      CKL();
    }
    k_dense_lr<<<nb, LR_NT, smem, s>>>(arena, ranks, d_desc + b0, scratch.p, per, 1);
    CKL();
  }
}

CBIE_FLOP_API(lowrank)

// Development benchmark of the Gram-path recompression kernel (tools/trunc_bench.py):
// nprob independent problems U (m x k) Vt (n x k), Gaussian columns scaled by
// 10^(-4 j / r_true) (numerical rank ~ r_true at tol 1e-4), recompressed reps times into
// a separate output region (inputs unchanged).  ms_out: mean launch time; prof_out (32):
// the CBIE_PROFILE cycle counters of the last launch; ranks_out (nprob): kept ranks.
extern "C" int cbie_trunc_bench(cbie_ctx* c, int m, int n, int k, int r_true, int nprob, double tol, int csize,
                                int reps, float* ms_out, unsigned long long* prof_out, int* ranks_out) {
  try {
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const int64_t per_in = (int64_t)(m + n) * k, per_out = (int64_t)(m + n) * k;
    std::vector<zc> h((size_t)per_in * nprob);
    uint64_t st = 0x9E3779B97F4A7C15ull;
    auto nrm = [&]() {   // Box-Muller on a 64-bit LCG
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const double u1 = ((st >> 11) + 1.0) / 9007199254740993.0;
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const double u2 = (st >> 11) / 9007199254740992.0;
      return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    };
    for (int p = 0; p < nprob; ++p)
      for (int l = 0; l < k; ++l) {
        const double sc = pow(10.0, -4.0 * l / std::max(1, r_true));
        zc* U = h.data() + (size_t)p * per_in;
        for (int i = 0; i < m; ++i) U[(size_t)l * m + i] = zmk(sc * nrm(), sc * nrm());
        zc* V = U + (size_t)m * k;
        for (int j = 0; j < n; ++j) V[(size_t)l * n + j] = zmk(nrm(), nrm());
      }
    DBuf<zc> ar, out;
    ar.upload(h, s);
    out.alloc((size_t)per_out * nprob);
    std::vector<TruncDesc> ds(nprob);
    for (int p = 0; p < nprob; ++p) {
      TruncDesc& d = ds[p];
      d.in_u = (int64_t)p * per_in;
      d.in_v = d.in_u + (int64_t)m * k;
      d.ldu = m;
      d.ldv = n;
      d.skip_slot = -1;
      d.out_u = (int64_t)p * per_out;
      d.out_v = d.out_u + (int64_t)m * k;
      d.m = m;
      d.n = n;
      d.k = k;
      d.k_slot = -1;
      d.cap = k;
      d.out_slot = p;
    }
    DBuf<TruncDesc> dd;
    dd.upload(ds, s);
    DBuf<int> ranks, defer;
    ranks.alloc(nprob);
    defer.alloc(nprob + 1);
    DBuf<unsigned long long> ovf;
    ovf.alloc(1);
    CK(cudaMemsetAsync(ovf.p, 0, 8, s));
    DBuf<zc> scratch;
    trunc_prof_enable(true, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float tot = 0.0f;
    for (int it = 0; it <= reps; ++it) {
      CK(cudaMemsetAsync(defer.p, 0, sizeof(int), s));
      CK(cudaMemsetAsync(g_trunc_prof, 0, 32 * sizeof(unsigned long long), s));
      cudaEventRecord(e0, s);
      launch_truncate_gram(ar.p, ranks.p, dd.p, nprob, tol, ovf.p, scratch, s, out.p, defer.p, nullptr,
                           k > 64 ? std::max(m, n) : 0, csize);
      cudaEventRecord(e1, s);
      CK(cudaEventSynchronize(e1));
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0) tot += ms;   // the first launch is a warm-up
    }
    *ms_out = tot / std::max(1, reps);
    CK(cudaMemcpy(prof_out, g_trunc_prof, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ranks_out, ranks.p, sizeof(int) * nprob, cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return CBIE_OK;
  } catch (const cbie_error& e) {
    c->err = e.what();
    return e.code;
  }
}
