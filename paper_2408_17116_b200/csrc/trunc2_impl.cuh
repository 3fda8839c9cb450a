// trunc2_impl.cuh — body of the blocked recompression kernel (see trunc2.cu),
// included once per CTA shape: namespace T2NS, T2_NT threads, T2_ELEMS shared
// complex elements, T2_MINB resident CTAs per SM.  No include guard on purpose.
namespace {
namespace T2NS {
namespace cg = cooperative_groups;

constexpr int NT = T2_NT;
constexpr int NW = NT / 32;
constexpr int KMAX = 128;      // largest concatenated rank handled here
constexpr int MMAX = 384;      // largest block side
constexpr int PWMAX = 32;      // widest panel
constexpr int ELEMS = T2_ELEMS;  // dynamic shared region (zc): panels / core / Jacobi block
constexpr double DELTA = 0.05; // pivoted-QR drop threshold relative to tol * s_0
constexpr unsigned FULL = 0xffffffffu;

// cluster rank / size of this CTA (1-CTA launches: 0 / 1) and the row slice of rank r of c
__device__ __forceinline__ int cl_rank() { return (int)cg::this_cluster().block_rank(); }
__device__ __forceinline__ int cl_size() { return (int)cg::this_cluster().num_blocks(); }
__device__ __forceinline__ int slice_lo(int m, int r, int c) { return (int)(((int64_t)m * r) / c); }

// shared region layout for a QR / Q application on m rows:
//   [panel: (m|1) x pw][Z chunk: (m|1) x CH][W: pw x CH][split partials: NT]
__host__ __device__ inline int panel_width(int m) {
  const int pw = (ELEMS - NT) / (2 * (m | 1));
  return pw < 2 ? 2 : (pw > PWMAX ? PWMAX : pw);
}
__host__ __device__ inline int chunk_cols(int m, int pw) {
  return (ELEMS - NT - (m | 1) * pw) / ((m | 1) + pw);
}
__host__ __device__ inline int64_t scratch_per(int kc) {
  return 2 * (int64_t)(kc + PWMAX) * PWMAX + 4 * (int64_t)kc * kc + 64;
}

struct Smem {
  zc rd1[KMAX], rd2[KMAX], rdM[KMAX];
  zc u0[PWMAX];
  double kap1[KMAX], kap2[KMAX];
  double nrm[2][KMAX], sig[KMAX];   // column norms double-buffered across pivot steps
  double sk[PWMAX];
  int perm[KMAX], order[KMAX];
  double red[NW];
  int flag;
};

__device__ __forceinline__ double bsum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}
__device__ __forceinline__ zc zshfl(zc v, int src) {
  return zmk(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// Householder QR of the panel P (mp x jn, ld ldp, shared) in place; the
// reflector of column j is generated redundantly by every warp from column j
// itself, so a column step needs a single barrier.  Conventions as cta_qr:
// R strictly above the diagonal, rd[j] = R[j][j], reflector u_j in rows >= j
// (head u0 on the diagonal), H_j = I - kap[j] u_j u_j^H.
template <int RPL>
__device__ void panel_factor(zc* P, int ldp, int mp, int jn, zc* rd, double* kap, Smem& S) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 0; j < jn; ++j) {
    zc x[RPL];
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      x[t] = (i >= j && i < mp) ? P[j * ldp + i] : zmk(0.0, 0.0);
      s += zabs2(x[t]);
    }
    s = warp_sum(s);
    const zc alpha = P[j * ldp + j];
    const double nx = sqrt(s), aa = sqrt(zabs2(alpha));
    const zc ph = aa > 0.0 ? zmk(alpha.x / aa, alpha.y / aa) : zmk(1.0, 0.0);
    const double kp = nx > 0.0 ? 1.0 / (nx * (nx + aa)) : 0.0;
    const zc u0 = nx > 0.0 ? zscale(ph, aa + nx) : alpha;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
      if (lane + 32 * t == j) x[t] = u0;
    if (threadIdx.x == 0) {
      rd[j] = nx > 0.0 ? zscale(ph, -nx) : zmk(0.0, 0.0);
      kap[j] = kp;
      S.u0[j] = u0;
    }
    if (kp != 0.0) {
      for (int c = j + 1 + w; c < jn; c += NW) {
        zc y[RPL];
        zc d = zmk(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          y[t] = (i >= j && i < mp) ? P[c * ldp + i] : zmk(0.0, 0.0);
          d = zadd(d, zcmul(x[t], y[t]));
        }
        d = zscale(zmk(warp_sum(d.x), warp_sum(d.y)), kp);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          if (i >= j && i < mp) P[c * ldp + i] = zsub(y[t], zmul(d, x[t]));
        }
      }
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < jn; j += NT) P[j * ldp + j] = S.u0[j];
  __syncthreads();
}

// S (jn x jn, col-major ld lds, global) = unit-diagonal strict upper triangle of
// Y^H Y, Y = [u_0 .. u_{jn-1}] diag(sqrt kap): Q_p = H_0 .. H_{jn-1} = I - Y S^{-1} Y^H.
__device__ void build_S(const zc* P, int ldp, int mp, int jn, const double* kap, zc* Sg, int lds) {
  for (int e = threadIdx.x; e < jn * jn; e += NT) {
    const int a = e % jn, b = e / jn;
    zc s = zmk(a == b ? 1.0 : 0.0, 0.0);
    if (a < b && kap[a] != 0.0 && kap[b] != 0.0) {
      zc acc = zmk(0.0, 0.0);
      for (int i = b; i < mp; ++i) acc = zadd(acc, zcmul(P[a * ldp + i], P[b * ldp + i]));
      s = zscale(acc, sqrt(kap[a] * kap[b]));
    }
    Sg[b * lds + a] = s;
  }
}

// Z (mp x nz, ldz) <- (I - Y S^{-op} Y^H) Z, Y = P diag(sk) (column a of P holds
// u_a in rows >= a).  adj: S^{-H} (Q_p^H, trailing update); else S^{-1} (Q_p).
// Z is processed in chunks of CH columns staged in shared memory (Zs, ld
// mp|1); W = Y^H Zs is computed one output per thread, with the row range
// split over up to 8 threads (partials in Red) when the chunk has few outputs.
__device__ void block_reflect(const zc* P, int ldp, int mp, int jn, const double* sk, const zc* Sg,
                              int lds, zc* Z, int ldz, int nz, bool adj, zc* Zs, zc* Wsm, zc* Red,
                              int CH) {
  const int ldzs = mp | 1;
  for (int c0 = 0; c0 < nz; c0 += CH) {
    const int nc = min(CH, nz - c0);
    for (int e = threadIdx.x; e < mp * nc; e += NT) {
      const int c = e / mp, i = e - c * mp;
      Zs[c * ldzs + i] = Z[(int64_t)(c0 + c) * ldz + i];
    }
    __syncthreads();
    const int no = jn * nc;
    const int ns = no >= NT ? 1 : min(8, NT / no);
    for (int t = threadIdx.x; t < no * ns; t += NT) {
      const int o = t % no, sp = t / no;
      const int a = o % jn, c = o / jn;
      const int i0 = (mp * sp) / ns, i1 = (mp * (sp + 1)) / ns;
      const zc* pa = P + a * ldp;
      const zc* zz = Zs + c * ldzs;
      zc a0 = zmk(0.0, 0.0), a1 = zmk(0.0, 0.0);
      int i = i0;
      for (; i + 1 < i1; i += 2) {
        const zc u0 = i >= a ? pa[i] : zmk(0.0, 0.0);
        const zc u1 = i + 1 >= a ? pa[i + 1] : zmk(0.0, 0.0);
        a0 = zadd(a0, zcmul(u0, zz[i]));
        a1 = zadd(a1, zcmul(u1, zz[i + 1]));
      }
      if (i < i1 && i >= a) a0 = zadd(a0, zcmul(pa[i], zz[i]));
      if (ns == 1) Wsm[o] = zadd(a0, a1);
      else Red[sp * no + o] = zadd(a0, a1);
    }
    __syncthreads();
    if (ns > 1) {
      for (int o = threadIdx.x; o < no; o += NT) {
        zc v = Red[o];
        for (int sp = 1; sp < ns; ++sp) v = zadd(v, Red[sp * no + o]);
        Wsm[o] = v;
      }
      __syncthreads();
    }
    for (int c = threadIdx.x; c < nc; c += NT) {
      zc* wc = Wsm + c * jn;
      for (int a = 0; a < jn; ++a) wc[a] = zscale(wc[a], sk[a]);
      if (adj) {   // S^H is unit lower triangular: forward substitution
        for (int a = 1; a < jn; ++a) {
          zc v = wc[a];
          for (int l = 0; l < a; ++l) v = zsub(v, zcmul(Sg[a * lds + l], wc[l]));
          wc[a] = v;
        }
      } else {     // S is unit upper triangular: back substitution
        for (int a = jn - 2; a >= 0; --a) {
          zc v = wc[a];
          for (int l = a + 1; l < jn; ++l) v = zsub(v, zmul(Sg[l * lds + a], wc[l]));
          wc[a] = v;
        }
      }
      for (int a = 0; a < jn; ++a) wc[a] = zscale(wc[a], sk[a]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < mp * nc; e += NT) {
      const int c = e / mp, i = e - c * mp;
      const int am = min(jn, i + 1);
      const zc* wc = Wsm + c * jn;
      zc s = zmk(0.0, 0.0);
      for (int a = 0; a < am; ++a) zfma(s, P[a * ldp + i], wc[a]);
      Z[(int64_t)(c0 + c) * ldz + i] = zsub(Zs[c * ldzs + i], s);
    }
    __syncthreads();
  }
}

// Blocked Householder QR of A (m x k, ld, global) in place; S factors of the
// panels into Sg (the panel starting at column p0 at Sg + p0 * pw, ld pw).
template <int RPL>
__device__ void blk_qr(zc* A, int m, int k, int ld, zc* rd, double* kap, zc* Sg, zc* sm, Smem& S) {
  const int kk = min(m, k);
  const int ldp = m | 1, pw = panel_width(m);
  const int CH = chunk_cols(m, pw);
  zc* P = sm;
  zc* Zs = sm + ldp * pw;
  zc* Wsm = Zs + ldp * CH;
  zc* Red = Wsm + pw * CH;
  for (int p0 = 0; p0 < kk; p0 += pw) {
    const int mp = m - p0, jn = min(pw, kk - p0);
    for (int e = threadIdx.x; e < jn * mp; e += NT) {
      const int c = e / mp, i = e - c * mp;
      P[c * ldp + i] = A[(int64_t)(p0 + c) * ld + p0 + i];
    }
    __syncthreads();
    panel_factor<RPL>(P, ldp, mp, jn, rd + p0, kap + p0, S);
    zc* Sp = Sg + (int64_t)p0 * pw;   // panel S factors: pw x pw, ld pw
    build_S(P, ldp, mp, jn, kap + p0, Sp, pw);
    for (int j = threadIdx.x; j < jn; j += NT) S.sk[j] = sqrt(kap[p0 + j]);
    for (int e = threadIdx.x; e < jn * mp; e += NT) {
      const int c = e / mp, i = e - c * mp;
      A[(int64_t)(p0 + c) * ld + p0 + i] = P[c * ldp + i];
    }
    __syncthreads();
    const int nt = k - p0 - jn;
    if (nt > 0)
      block_reflect(P, ldp, mp, jn, S.sk, Sp, pw, A + (int64_t)(p0 + jn) * ld + p0, ld, nt, true, Zs, Wsm,
                    Red, CH);
  }
}

// Z (m x nz, ldz) := Q Z, Q = H_0 .. H_{kk-1} from blk_qr (reflectors in A).
__device__ void blk_apply_q(const zc* A, int m, int kk, int ld, const double* kap, const zc* Sg, zc* Z,
                            int ldz, int nz, zc* sm, Smem& S) {
  const int ldp = m | 1, pw = panel_width(m);
  const int CH = chunk_cols(m, pw);
  zc* P = sm;
  zc* Zs = sm + ldp * pw;
  zc* Wsm = Zs + ldp * CH;
  zc* Red = Wsm + pw * CH;
  const int np = (kk + pw - 1) / pw;
  for (int pi = np - 1; pi >= 0; --pi) {
    const int p0 = pi * pw, mp = m - p0, jn = min(pw, kk - p0);
    for (int e = threadIdx.x; e < jn * mp; e += NT) {
      const int c = e / mp, i = e - c * mp;
      P[c * ldp + i] = A[(int64_t)(p0 + c) * ld + p0 + i];
    }
    for (int j = threadIdx.x; j < jn; j += NT) S.sk[j] = sqrt(kap[p0 + j]);
    __syncthreads();
    block_reflect(P, ldp, mp, jn, S.sk, Sg + (int64_t)p0 * pw, pw, Z + p0, ldz, nz, false, Zs, Wsm, Red,
                  CH);
  }
}

// Column-pivoted QR of M (p x q, ld; p <= KMAX) in place, stopped when the
// trailing Frobenius^2 <= thr_rel2 * (largest column norm)^2.  On exit, for
// a < kp: R[a][a] = S.rdM[a], R[a][b] = M[b * ld + a] (b > a); storage column
// b holds original column S.perm[b].  Returns kp.
__device__ int qrcp(zc* M, int p, int q, int ld, double thr_rel2, Smem& S) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = w; c < q; c += NW) {
    double s = 0.0;
    for (int i = lane; i < p; i += 32) s += zabs2(M[(int64_t)c * ld + i]);
    s = warp_sum(s);
    if (lane == 0) {
      S.nrm[0][c] = s;
      S.perm[c] = c;
    }
  }
  __syncthreads();
  double nmax = 0.0;
  for (int c = lane; c < q; c += 32) nmax = fmax(nmax, S.nrm[0][c]);
  nmax = warp_max(nmax);
  const double thr2 = thr_rel2 * nmax;
  const int kmax = min(p, q);
  int j = 0;
  for (; j < kmax; ++j) {
    // every warp computes the same pivot and trailing norm (identical code and data)
    // norms of step j live in buffer j & 1; the updates below write buffer
    // (j + 1) & 1, so no warp can overwrite a norm another warp is still reading
    const double* nr = S.nrm[j & 1];
    double best = -1.0, tsum = 0.0;
    int bi = q;
    for (int c = j + lane; c < q; c += 32) {
      const double v = nr[c];
      tsum += v;
      if (v > best) {
        best = v;
        bi = c;
      }
    }
    tsum = warp_sum(tsum);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(FULL, best, o);
      const int oi = __shfl_xor_sync(FULL, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (!(tsum > thr2)) break;
    if (bi != j) {
      for (int i = threadIdx.x; i < p; i += NT) {
        const zc t = M[(int64_t)j * ld + i];
        M[(int64_t)j * ld + i] = M[(int64_t)bi * ld + i];
        M[(int64_t)bi * ld + i] = t;
      }
      if (threadIdx.x == 0) {
        const int t = S.perm[j];
        S.perm[j] = S.perm[bi];
        S.perm[bi] = t;
      }
      __syncthreads();
    }
    zc x[KMAX / 32];
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < KMAX / 32; ++t) {
      const int i = lane + 32 * t;
      x[t] = (i >= j && i < p) ? M[(int64_t)j * ld + i] : zmk(0.0, 0.0);
      s += zabs2(x[t]);
    }
    s = warp_sum(s);
    const zc alpha = M[(int64_t)j * ld + j];
    const double nx = sqrt(s), aa = sqrt(zabs2(alpha));
    const zc ph = aa > 0.0 ? zmk(alpha.x / aa, alpha.y / aa) : zmk(1.0, 0.0);
    const double kp = nx > 0.0 ? 1.0 / (nx * (nx + aa)) : 0.0;
    const zc u0 = nx > 0.0 ? zscale(ph, aa + nx) : alpha;
#pragma unroll
    for (int t = 0; t < KMAX / 32; ++t)
      if (lane + 32 * t == j) x[t] = u0;
    if (threadIdx.x == 0) S.rdM[j] = nx > 0.0 ? zscale(ph, -nx) : zmk(0.0, 0.0);
    for (int c = j + 1 + w; c < q; c += NW) {
      zc y[KMAX / 32];
      zc d = zmk(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < KMAX / 32; ++t) {
        const int i = lane + 32 * t;
        y[t] = (i >= j && i < p) ? M[(int64_t)c * ld + i] : zmk(0.0, 0.0);
        d = zadd(d, zcmul(x[t], y[t]));
      }
      d = zscale(zmk(warp_sum(d.x), warp_sum(d.y)), kp);
      double ns = 0.0;
#pragma unroll
      for (int t = 0; t < KMAX / 32; ++t) {
        const int i = lane + 32 * t;
        if (i >= j && i < p) {
          const zc v = zsub(y[t], zmul(d, x[t]));
          M[(int64_t)c * ld + i] = v;
          if (i > j) ns += zabs2(v);
        }
      }
      ns = warp_sum(ns);
      if (lane == 0) S.nrm[(j + 1) & 1][c] = ns;
    }
    __syncthreads();
  }
  return j;
}

// One-sided Jacobi on the columns of A (p x q, ld), half-warp per pair, no
// accumulated rotations.  Rotation and skip rules as cta_jacobi_hw.
__device__ int jacobi_nw(zc* A, int p, int q, int ld, Smem& S) {
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
  constexpr int NHW = NT / 16;
  double f2 = 0.0;
  for (int e = threadIdx.x; e < p * q; e += NT) f2 += zabs2(A[(int64_t)(e / p) * ld + e % p]);
  f2 = bsum(f2, S.red);
  const double floor2 = 1e-24 * f2;
  if (q < 2) return 0;
  const int qe = q + (q & 1);
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) S.flag = 0;
    __syncthreads();
    for (int r = 0; r < qe - 1; ++r) {
      for (int base = 0; base < qe / 2; base += NHW) {
        const int pi = base + hw;
        const int pa = pi, pb = qe - 1 - pi;
        const int a = pa == 0 ? 0 : ((pa - 1 + r) % (qe - 1)) + 1;
        const int b = pb == 0 ? 0 : ((pb - 1 + r) % (qe - 1)) + 1;
        const bool valid = pi < qe / 2 && a < q && b < q;
        zc* x = A + (int64_t)(valid ? a : 0) * ld;
        zc* y = A + (int64_t)(valid ? b : 0) * ld;
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
        if (hl == 0) S.flag = 1;
      }
      __syncthreads();
    }
    if (S.flag == 0) break;
    __syncthreads();
  }
  return sweep;
}

template <int RPL>
__global__ void __launch_bounds__(NT, T2_MINB)
    k_trunc2(zc* arena, zc* aout, int* ranks, const TruncDesc* __restrict__ descs, zc* scratch,
             int64_t per, int kc, double tol, unsigned long long* overflow, unsigned long long* prof,
             int* defer, int base, const int* idx) {
  __shared__ Smem S;
  extern __shared__ __align__(16) unsigned char smraw[];
  zc* sm = reinterpret_cast<zc*>(smraw);
  // one problem per cluster (csize CTAs, cluster_gram_sum); pb = problem of this cluster
  const int crank = cl_rank(), csize = cl_size();
  const int pb = (int)blockIdx.x / csize;
  // idx: run the problems listed in idx[1 + base + pb] (count idx[0]) of descs
  if (idx && base + pb >= idx[0]) return;
  const int tix = idx ? idx[1 + base + pb] : pb;
  const TruncDesc d = descs[tix];
  const long long tc0 = clock64();
  if (d.skip_slot >= 0 && ranks[d.skip_slot] == 0) return;
  const int k = trunc_k(d, ranks);
  const int m = d.m, n = d.n;
  if (k <= 0 || m == 0 || n == 0) {
    if (threadIdx.x == 0) ranks[d.out_slot] = 0;
    return;
  }
  if (k > kc) {   // larger than this kernel's layout: handed to the unblocked kernel
    if (threadIdx.x == 0) defer[1 + atomicAdd(defer, 1)] = idx ? tix : base + blockIdx.x;
    return;
  }
  if (threadIdx.x == 0) flop_add(flops_trunc(m, n, k, false));
  zc* U = arena + d.in_u;
  zc* Vt = arena + d.in_v;
  const int kk1 = min(m, k), kk2 = min(n, k);
  zc* sc = scratch + (int64_t)blockIdx.x * per;
  zc* SgU = sc;
  zc* SgV = SgU + (int64_t)(kc + PWMAX) * PWMAX;
  zc* Mg = SgV + (int64_t)(kc + PWMAX) * PWMAX;   // kk1 x kk2 (kept for U' = M Vhat)
  zc* M2 = Mg + (int64_t)kc * kc;                 // pivoted-QR workspace when M exceeds smem
  zc* G = M2 + (int64_t)kc * kc;                  // R1^H staging / global Jacobi block
  zc* Vh = G + (int64_t)kc * kc;                  // kk2 x r right singular vectors

  blk_qr<RPL>(U, m, k, d.ldu, S.rd1, S.kap1, SgU, sm, S);
  blk_qr<RPL>(Vt, n, k, d.ldv, S.rd2, S.kap2, SgV, sm, S);
  const long long tc1 = clock64();
  // M = R1 R2^T (R factors staged in shared memory when they fit)
  if ((kk1 + kk2) * k <= ELEMS) {
    zc* R1 = sm;                       // kk1 x k, ld kk1
    zc* R2 = sm + kk1 * k;             // kk2 x k, ld kk2
    for (int e = threadIdx.x; e < kk1 * k; e += NT) {
      const int c = e / kk1, a = e - c * kk1;
      R1[e] = c == a ? S.rd1[a] : (c > a ? U[(int64_t)c * d.ldu + a] : zmk(0.0, 0.0));
    }
    for (int e = threadIdx.x; e < kk2 * k; e += NT) {
      const int c = e / kk2, b = e - c * kk2;
      R2[e] = c == b ? S.rd2[b] : (c > b ? Vt[(int64_t)c * d.ldv + b] : zmk(0.0, 0.0));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kk1 * kk2; e += NT) {
      const int a = e % kk1, b = e / kk1;
      zc s = zmk(0.0, 0.0);
      for (int c = max(a, b); c < k; ++c) zfma(s, R1[c * kk1 + a], R2[c * kk2 + b]);
      Mg[e] = s;
    }
  } else {
    for (int e = threadIdx.x; e < kk1 * kk2; e += NT) {
      const int a = e % kk1, b = e / kk1;
      zc s = zmk(0.0, 0.0);
      for (int c = max(a, b); c < k; ++c) {
        const zc r1 = c == a ? S.rd1[a] : U[(int64_t)c * d.ldu + a];
        const zc r2 = c == b ? S.rd2[b] : Vt[(int64_t)c * d.ldv + b];
        zfma(s, r1, r2);
      }
      Mg[e] = s;
    }
  }
  __syncthreads();
  const bool m_sm = kk1 * kk2 <= ELEMS;
  zc* Mq = m_sm ? sm : M2;
  for (int e = threadIdx.x; e < kk1 * kk2; e += NT) Mq[e] = Mg[e];
  __syncthreads();
  const int kp = qrcp(Mq, kk1, kk2, kk1, (DELTA * tol) * (DELTA * tol), S);
  // A = R1^H (kk2 x kp)
  for (int e = threadIdx.x; e < kk2 * kp; e += NT) {
    const int b = e % kk2, a = e / kk2;
    G[e] = b > a ? zconj(Mq[(int64_t)b * kk1 + a]) : (b == a ? zconj(S.rdM[a]) : zmk(0.0, 0.0));
  }
  __syncthreads();
  const bool a_sm = kk2 * kp <= ELEMS;
  zc* Aj = a_sm ? sm : G;
  if (a_sm) {
    for (int e = threadIdx.x; e < kk2 * kp; e += NT) sm[e] = G[e];
    __syncthreads();
  }
  const long long tc2 = clock64();
  const int sweeps = jacobi_nw(Aj, kk2, kp, kk2, S);
  for (int c = threadIdx.x; c < kp; c += NT) {
    double sq = 0.0;
    for (int i = 0; i < kk2; ++i) sq += zabs2(Aj[(int64_t)c * kk2 + i]);
    S.sig[c] = sqrt(sq);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kp; c += NT) {
    int pos = 0;
    for (int o = 0; o < kp; ++o)
      if (S.sig[o] > S.sig[c] || (S.sig[o] == S.sig[c] && o < c)) ++pos;
    S.order[pos] = c;
  }
  __syncthreads();
  const long long tc3 = clock64();
  const double s0 = kp > 0 ? S.sig[S.order[0]] : 0.0;
  int r = 0;
  if (s0 > 0.0) {
    for (int c = 0; c < kp; ++c)
      if (S.sig[c] > tol * s0) ++r;
    r = max(r, 1);
  }
  if (r > d.cap) {
    if (threadIdx.x == 0) atomicAdd(overflow, 1ull);
    r = d.cap;
  }
  // Vhat = P B_r / sigma_r  (kk2 x r)
  for (int e = threadIdx.x; e < kk2 * r; e += NT) {
    const int b = e % kk2, l = e / kk2;
    const int c = S.order[l];
    Vh[(int64_t)l * kk2 + S.perm[b]] = zscale(Aj[(int64_t)c * kk2 + b], 1.0 / S.sig[c]);
  }
  __syncthreads();
  zc* Uo = aout + d.out_u;
  zc* Vo = aout + d.out_v;
  for (int e = threadIdx.x; e < n * r; e += NT) {
    const int l = e / n, j = e - l * n;
    Vo[(int64_t)l * n + j] = j < kk2 ? zconj(Vh[(int64_t)l * kk2 + j]) : zmk(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < m * r; e += NT) {
    const int l = e / m, i = e - l * m;
    zc s = zmk(0.0, 0.0);
    if (i < kk1) {
      const zc* vh = Vh + (int64_t)l * kk2;
      for (int b = 0; b < kk2; ++b) zfma(s, Mg[(int64_t)b * kk1 + i], vh[b]);
    }
    Uo[(int64_t)l * m + i] = s;
  }
  __syncthreads();
  if (r > 0) {
    blk_apply_q(U, m, kk1, d.ldu, S.kap1, SgU, Uo, m, r, sm, S);
    blk_apply_q(Vt, n, kk2, d.ldv, S.kap2, SgV, Vo, n, r, sm, S);
  }
  if (threadIdx.x == 0 && crank == 0) {
    ranks[d.out_slot] = r;
    if (prof) {
      const long long tc4 = clock64();
      atomicAdd(prof + 0, (unsigned long long)(tc1 - tc0));
      atomicAdd(prof + 1, (unsigned long long)(tc2 - tc1));
      atomicAdd(prof + 2, (unsigned long long)(tc3 - tc2));
      atomicAdd(prof + 3, (unsigned long long)(tc4 - tc3));
      atomicAdd(prof + 4, 1ull);
      atomicAdd(prof + 5, (unsigned long long)sweeps);
      atomicAdd(prof + 14, 1ull);
      atomicAdd(prof + 15, (unsigned long long)(tc4 - tc0));
    }
  }
}

template <int RPL>
void launch_rpl(zc* arena, zc* aout, int* ranks, const TruncDesc* d_desc, int nd, int kc, double tol,
                unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, unsigned long long* prof,
                int* defer, const int* idx = nullptr) {
  const int64_t per = scratch_per(kc);
  const int wave = (int)std::max<int64_t>(1, (int64_t)ws_cap(2) / (per * (int64_t)sizeof(zc)));
  const size_t need = (size_t)std::min(wave, nd) * per;
  if (scratch.n < need) scratch.alloc(need);
  const int smem = ELEMS * (int)sizeof(zc);
  CK(cudaFuncSetAttribute(k_trunc2<RPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int b0 = 0; b0 < nd; b0 += wave) {
    const int nb = std::min(wave, nd - b0);
    k_trunc2<RPL><<<nb, NT, smem, s>>>(arena, aout, ranks, idx ? d_desc : d_desc + b0, scratch.p, per, kc,
                                       tol, overflow, prof, defer, b0, idx);
    CKL();
  }
}

#ifdef T2_GRAM
// ---------------------------------------------------------------------------
// Gram path (concatenated rank k <= KG, any m, n): the two Householder QRs and
// the two Q applications of k_trunc2 -- k sequential column steps over m rows
// each -- are replaced by one streaming pass per factor:
//   1. G_u = U^H U, G_v = Vt^H Vt (k x k) accumulated from row chunks staged
//      in shared memory (FMA-bound, no per-column barrier);
//   2. column balancing (U_c, Vt_c) -> (U_c a_c, Vt_c / a_c), a_c = (|Vt_c|/|U_c|)^(1/2):
//      exact for U Vt^T, makes the relative stop below scale-free;
//   3. pivoted Cholesky of the balanced Grams: P^T G P = R^H R, stopped when the
//      largest remaining pivot is <= CHOL_EPS * max diagonal (directions below
//      ~3e-7 of the largest balanced column norm are dropped: far below
//      tol * s_0 for every tol >= 1e-5 this path is used for);
//      U = Q_u R_u P_u^T with Q_u = (U D P_u)[:, :k_u] R_u11^{-1} never formed;
//   4. core M = (R_u P_u^T)(R_v P_v^T)^T and its SVD exactly as in k_trunc2
//      (pivoted QR reduction + one-sided Jacobi), keep s > tol * s_0;
//   5. U' = U_sel D R_u11^{-1} (M Vhat), Vt' = Vt_sel D^{-1} R_v11^{-1} conj(Vhat):
//      two small triangular solves and one streaming GEMM per factor.
// Same result as truncate_lowrank (hmatrix.py:412-426) up to the Gram rounding
// (~sqrt(eps) relative), inside the solution-level parity budget.
// ---------------------------------------------------------------------------
constexpr int KG = 64;              // largest concatenated rank of the Gram path
constexpr int GCH = 64;             // rows staged per Gram chunk
constexpr int GSQ = KG * KG;        // one k x k region (zc)
constexpr int GLD = KG + 1;         // staged row stride (bank spread)
constexpr double CHOL_EPS = 1e-13;  // pivoted-Cholesky stop (squared, relative)
// core reduction before the Jacobi: the pivoted Cholesky of H = M M^H stops once the
// remaining directions together carry at most GDELTA * tol * s_0 (Frobenius, the trace
// of the Schur complement), so what is dropped stays well inside the tol * s_0 cut
constexpr double GDELTA = 0.2;

__host__ __device__ inline int64_t gram_scratch_per() { return 4 * (int64_t)GSQ + 64; }

// G (k x k, ld k, shared, zeroed) += X^H X, X (m x k) col-major ld ldx in global memory.
// Hermitian: only the 4 x 4 tiles on and above the block diagonal are accumulated
// (conjugate-FMA, 4 DFMA per complex term), the lower part is mirrored; thread groups
// split the rows; the next 64-row chunk is loaded into registers while the current
// one is consumed from shared memory.
// rows [r_lo, r_hi) only (a cluster CTA's slice; the partial Grams are summed across the
// cluster by cluster_gram_sum).
__device__ void gram_acc(const zc* __restrict__ X, int r_lo, int r_hi, int k, int ldx, zc* G, zc* Xs) {
  constexpr int PER = GCH * KG / NT;   // staged elements per thread
  const int tb = (k + 3) / 4, ntile = tb * (tb + 1) / 2;
  const int groups = max(1, min(8, NT / ntile));   // row groups, summed in a fixed order below
  const int g = threadIdx.x / ntile, t = threadIdx.x % ntile;
  const bool act = g < groups;
  int tj = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((tj + 1) * (tj + 2) / 2 <= t) ++tj;
  while (tj * (tj + 1) / 2 > t) --tj;
  const int ti = t - tj * (tj + 1) / 2;
  const int a0 = 4 * ti, b0 = 4 * tj;
  double ar[4][4], ai[4][4];
#pragma unroll
  for (int qa = 0; qa < 4; ++qa)
#pragma unroll
    for (int qb = 0; qb < 4; ++qb) ar[qa][qb] = ai[qa][qb] = 0.0;
  zc v[PER];
  auto fetch = [&](int r0) {
    const int rows = min(GCH, r_hi - r0);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * NT;
      v[u] = (r0 < r_hi && e < rows * k) ? X[(int64_t)(e / rows) * ldx + r0 + e % rows] : zmk(0.0, 0.0);
    }
  };
  fetch(r_lo);
  for (int r0 = r_lo; r0 < r_hi; r0 += GCH) {
    const int rows = min(GCH, r_hi - r0);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * NT;
      if (e < rows * k) Xs[(e % rows) * GLD + e / rows] = v[u];
    }
    __syncthreads();
    fetch(r0 + GCH);
    if (act) {
      for (int i = g; i < rows; i += groups) {
        const zc* xr = Xs + i * GLD;
        zc xa[4], xb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xa[q] = a0 + q < k ? xr[a0 + q] : zmk(0.0, 0.0);
          xb[q] = b0 + q < k ? xr[b0 + q] : zmk(0.0, 0.0);
        }
#pragma unroll
        for (int qa = 0; qa < 4; ++qa)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb) {   // conj(xa) xb
            ar[qa][qb] = fma(xa[qa].x, xb[qb].x, fma(xa[qa].y, xb[qb].y, ar[qa][qb]));
            ai[qa][qb] = fma(xa[qa].x, xb[qb].y, fma(-xa[qa].y, xb[qb].x, ai[qa][qb]));
          }
      }
    }
  }
  // group partials added in group order (deterministic: bit-identical results for a
  // problem whatever batch or launch it runs in)
  for (int gg = 0; gg < groups; ++gg) {
    if (act && g == gg)
#pragma unroll
      for (int qa = 0; qa < 4; ++qa)
#pragma unroll
        for (int qb = 0; qb < 4; ++qb) {
          const int a = a0 + qa, b = b0 + qb;
          if (a >= k || b >= k || (ti == tj && a > b)) continue;
          zc& gp = G[b * k + a];
          gp = zmk(gp.x + ar[qa][qb], gp.y + ai[qa][qb]);
          if (a != b) G[a * k + b] = zconj(gp);   // mirror: G[b][a] = conj(G[a][b])
        }
    __syncthreads();
  }
}

// DMMA form of gram_acc (same contract, but G is WRITTEN, not accumulated): the
// products run on the FP64 tensor pipe (mma.sync.m8n8k4.f64, 4 DMMA per complex 8x8x4
// step).  The upper 8 x 8 tiles (a-block <= b-block) are dealt to the warps of a row
// group, the 4-row steps of each 32-row chunk round-robin to RS row groups.  Chunks are
// double-buffered in Xs (2 x KG x GSLD shared zc; may overlap G, which is stored after
// the last staging read) by cp.async, column-major with a stride that makes the fragment
// loads conflict-free.  Row-group partials are added in group order (deterministic).
constexpr int GTPW = 9;     // upper tiles per warp (36 tiles of k = 64 over 4 warps)
constexpr int GMCH = 32;    // rows per staged chunk
constexpr int GSLD = 36;    // staging column stride (zc)
__device__ int g_gram_mma = 1;   // 0: DFMA gram_acc / apply_sel (CBIE_NO_DMMA)
__device__ int g_ms_min_add = 1;    // multi-stage: fewest new columns per stage (CBIE_MS_MIN_ADD)
__device__ int g_prof_mn = 0;       // CBIE_PROFILE: only problems with max(m, n) >= this (CBIE_PROF_MN)
__device__ int g_prof_kmin = 0;     // ... and k >= this (CBIE_PROF_KMIN)
__device__ int g_pchol_w = NW / 2;   // warps per Gram pivoted Cholesky (CBIE_PCHOL_W)
__device__ int g_pcholh_w = NW;      // warps of the core pivoted Cholesky (CBIE_PCHOLH_W)

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// A factor read in place from up to two pieces: columns [0, k1) from p1 (ld1), the
// columns from k1 on from p2 (ld2) -- TruncDesc's two-source form; one piece: k1 = INT_MAX
struct Src2 {
  const zc* p1;
  const zc* p2;
  int ld1, ld2, k1;
  __device__ __forceinline__ const zc* col(int c) const {
    return c < k1 ? p1 + (int64_t)c * ld1 : p2 + (int64_t)(c - k1) * ld2;
  }
};
__device__ __forceinline__ Src2 src1(const zc* p, int ld) { return Src2{p, p, ld, ld, 0x7fffffff}; }

__device__ __noinline__ void gram_acc_mma(const Src2 X, int r_lo, int r_hi, int k, zc* G, zc* Xs) {
  const int nb = (k + 7) >> 3, nt = nb * (nb + 1) / 2;
  int RS = min(NW, GMCH / 4);
  while (RS > 1 && (nt + NW / RS - 1) / (NW / RS) > GTPW) RS >>= 1;
  const int wpr = NW / RS;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = w / wpr, wi = w % wpr;
  const int fr = lane & 3, fc = lane >> 2;
  double acc[GTPW][4];
#pragma unroll
  for (int q = 0; q < GTPW; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
  const int nch = (r_hi - r_lo + GMCH - 1) / GMCH;
  // staging offsets of this warp's tiles (tile t = (ta, b), ta <= b), fixed for the whole
  // accumulation: decoded once, not per 4-row step; -1: column beyond k (zero operand)
  int oa[GTPW], ob[GTPW];
#pragma unroll
  for (int q = 0; q < GTPW; ++q) {
    const int t = wi + q * wpr;
    int b = 0;
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    const int ca = (t - b * (b + 1) / 2) * 8 + fc, cb = b * 8 + fc;
    oa[q] = (t < nt && ca < k) ? ca * GSLD + fr : -1;
    ob[q] = (t < nt && cb < k) ? cb * GSLD + fr : -1;
  }
  // staging: a thread copies row (tid % GMCH) of columns tid / GMCH + i NT / GMCH of every
  // chunk -- the column pointers (either piece) are resolved once
  constexpr int NI = KG * GMCH / NT;
  static_assert(NT % GMCH == 0 && NI * NT == KG * GMCH, "staging layout");
  const int sr = threadIdx.x % GMCH;
  const zc* cp[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int col = threadIdx.x / GMCH + i * (NT / GMCH);
    cp[i] = col < k ? X.col(col) + sr : nullptr;
  }
  auto issue = [&](int c) {
    if (c < nch) {
      const int r0 = r_lo + c * GMCH;
      zc* buf = Xs + (c & 1) * (KG * GSLD) + (threadIdx.x / GMCH) * GSLD + sr;
      const bool ok = r0 + sr < r_hi;
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (cp[i]) cp_async16(buf + i * (NT / GMCH) * GSLD, ok ? cp[i] + r0 : X.p1, ok);
    }
    cp_async_commit();
  };
  issue(0);
  for (int c = 0; c < nch; ++c) {
    issue(c + 1);
    cp_async_wait1();
    __syncthreads();
    const zc* buf = Xs + (c & 1) * (KG * GSLD);
    const int nst = (min(GMCH, r_hi - r_lo - c * GMCH) + 3) >> 2;
    for (int st = g; st < nst; st += RS) {
      const zc* bs = buf + 4 * st;
#pragma unroll
      for (int q = 0; q < GTPW; ++q) {
        if (wi + q * wpr >= nt) break;   // warp-uniform
        const zc xa = oa[q] >= 0 ? bs[oa[q]] : zmk(0.0, 0.0);
        const zc xb = ob[q] >= 0 ? bs[ob[q]] : zmk(0.0, 0.0);
        zdmma_ca(acc[q], xa, xb);
      }
    }
    __syncthreads();   // buffer c & 1 is refilled by the next iteration's issue
  }
  for (int gg = 0; gg < RS; ++gg) {
    if (g == gg) {
#pragma unroll
      for (int q = 0; q < GTPW; ++q) {
        const int t = wi + q * wpr;
        if (t >= nt) break;
        int b = 0;
        while ((b + 1) * (b + 2) / 2 <= t) ++b;
        const int ta = t - b * (b + 1) / 2;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ea = ta * 8 + fc, eb = b * 8 + 2 * fr + j;
          if (ea >= k || eb >= k || ea > eb) continue;
          zc& gp = G[eb * k + ea];
          const zc val = zmk(acc[q][j], acc[q][2 + j]);
          gp = gg == 0 ? val : zadd(gp, val);
          if (ea != eb) G[ea * k + eb] = zconj(gp);
        }
      }
    }
    __syncthreads();
  }
}

// pivoted Cholesky of the Hermitian G (k x k, ld k, shared) in place: row j < kk of G
// holds row j of R (columns in pivoted order, entries >= j); perm[j] = original
// column of pivot j.  Returns kk: stops when the largest remaining pivot is <= thr_rel *
// max diagonal, or (trace_stop) when the remaining trace -- the squared Frobenius norm of
// what the remaining directions carry when G = M M^H -- is <= thr_rel * max diagonal.
__device__ int pchol(zc* G, int k, int* perm, double thr_rel, Smem& S, bool trace_stop = false) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < k; c += NT) perm[c] = c;
  double dmax = 0.0;
  for (int c = 0; c < k; ++c) dmax = fmax(dmax, G[c * k + c].x);
  const double thr = thr_rel * dmax;
  __syncthreads();
  int j = 0;
  for (; j < k; ++j) {
    if (w == 0) {
      double best = -1.0, tr = 0.0;
      int bi = k;
      for (int c = j + lane; c < k; c += 32) {
        const double v = G[c * k + c].x;
        tr += fmax(v, 0.0);
        if (v > best) {
          best = v;
          bi = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(FULL, best, o);
        const int oi = __shfl_xor_sync(FULL, bi, o);
        tr += __shfl_xor_sync(FULL, tr, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      const bool go = (trace_stop ? tr > thr : best > thr) && best > 0.0;
      if (lane == 0) S.flag = go ? 0 : 1;
      if (go) {
        if (bi != j) {
          for (int c = lane; c < k; c += 32) {   // rows j <-> bi
            const zc t = G[c * k + j];
            G[c * k + j] = G[c * k + bi];
            G[c * k + bi] = t;
          }
          __syncwarp();
          for (int i = lane; i < k; i += 32) {   // columns j <-> bi
            const zc t = G[j * k + i];
            G[j * k + i] = G[bi * k + i];
            G[bi * k + i] = t;
          }
          if (lane == 0) {
            const int t = perm[j];
            perm[j] = perm[bi];
            perm[bi] = t;
          }
          __syncwarp();
        }
        const double rjj = sqrt(G[j * k + j].x);
        const double inv = 1.0 / rjj;
        __syncwarp();
        for (int c = j + 1 + lane; c < k; c += 32) G[c * k + j] = zscale(G[c * k + j], inv);
        if (lane == 0) G[j * k + j] = zmk(rjj, 0.0);
      }
    }
    __syncthreads();
    if (S.flag) break;
    // trailing update on the lower triangle a >= b > j (Hermitian: mirrored below)
    for (int b = j + 1 + (threadIdx.x >> 6); b < k; b += NT / 64)
      for (int a = b + (threadIdx.x & 63); a < k; a += 64) {
        const zc v = zsub(G[b * k + a], zcmul(G[a * k + j], G[b * k + j]));
        G[b * k + a] = v;
        if (a != b) G[a * k + b] = zconj(v);
      }
    __syncthreads();
  }
  __syncthreads();
  return j;
}

// Pivoted Cholesky of the Hermitian PSD G (k x k <= 64, ld k, shared) by a group of W warps
// (gw: warp index in the group) synchronised by the named barrier bid -- no CTA-wide
// barriers, so two groups factor two matrices concurrently.  No row / column
// interchanges: the Schur complement is updated in place over the not-yet-pivoted
// indices (lanes own rows, warps own columns), row j of R is stored over row perm[j] of
// G, and the pivoted upper-triangular R is gathered at the end into the same layout as
// pchol (row j < kk holds row j of R, columns in pivot order; lower part zero) through
// tmp (k x k, shared or global).  Same stop rules as pchol; perm is completed with the
// unpivoted columns in increasing order.  Returns kk.
__device__ __forceinline__ void gbar(int id, int nth) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nth) : "memory"); }

__device__ int pchol_grp(zc* G, int k, int* perm, double thr_rel, bool trace_stop, int W, int gw, int bid, zc* tmp,
                         double* dg) {
  const int lane = threadIdx.x & 31, nth = 32 * W;
  const bool v0 = lane < k, v1 = lane + 32 < k;
  // dg (k doubles, shared): the remaining diagonal, kept beside G so the pivot search
  // reads it without the bank conflicts of G's stride-(k+1) diagonal
  double d0 = v0 ? G[lane * k + lane].x : 0.0, d1 = v1 ? G[(lane + 32) * k + lane + 32].x : 0.0;
  const double dmax = warp_max(fmax(d0, d1));
  const double thr = thr_rel * dmax, iscale = dmax > 0.0 ? 1.0 / dmax : 0.0;   // pivot keys in [0, 1]
  if (gw == 0) {
    if (v0) dg[lane] = d0;
    if (v1) dg[lane + 32] = d1;
  }
  gbar(bid, nth);
  unsigned long long done = 0ull;
  int j = 0;
  for (; j < k; ++j) {
    const bool f0 = v0 && !(done >> lane & 1ull), f1 = v1 && !(done >> (lane + 32) & 1ull);
    const double e0 = f0 ? dg[lane] : -1.0, e1 = f1 ? dg[lane + 32] : -1.0;
    // pivot: largest remaining diagonal (compared in float precision, which only decides
    // among near-equal pivots), lowest index among equal keys
    const unsigned k0 = e0 > 0.0 ? __float_as_uint((float)(e0 * iscale)) : 0u;
    const unsigned k1 = e1 > 0.0 ? __float_as_uint((float)(e1 * iscale)) : 0u;
    const unsigned km = __reduce_max_sync(FULL, max(k0, k1));
    const unsigned m0 = __ballot_sync(FULL, k0 == km), m1 = __ballot_sync(FULL, k1 == km);
    const int p = m0 ? __ffs(m0) - 1 : (m1 ? __ffs(m1) + 31 : k);
    const double best = p < k ? dg[p] : -1.0;
    bool go;
    if (trace_stop) {
      double tr = fmax(e0, 0.0) + fmax(e1, 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(FULL, tr, o);
      go = tr > thr && best > 0.0 && km > 0u;
    } else {
      go = best > thr && best > 0.0 && km > 0u;
    }
    if (!go) break;   // same data in every warp of the group: a uniform exit
    const double rjj = sqrt(best), inv = 1.0 / rjj;
    done |= 1ull << p;
    // row p of R over the remaining columns: R(j, c) = G(p, c) / rjj = conj(G(c, p)) / rjj
    const bool g0 = v0 && !(done >> lane & 1ull), g1 = v1 && !(done >> (lane + 32) & 1ull);
    const zc r0 = g0 ? zscale(zconj(G[p * k + lane]), inv) : zmk(0.0, 0.0);
    const zc r1 = g1 ? zscale(zconj(G[p * k + lane + 32]), inv) : zmk(0.0, 0.0);
    if (gw == 0 && lane == 0) perm[j] = p;
    gbar(bid, nth);   // the diagonal and column p are read by every warp before any update
    for (int b = gw; b < k; b += W) {
      if (b == p) {
        if (lane == 0) G[p * k + p] = zmk(rjj, 0.0);
        continue;
      }
      if (done >> b & 1ull) continue;
      const zc rb = zshfl(b < 32 ? r0 : r1, b & 31);
      zc* col = G + b * k;
      if (g0) {
        const zc v = zsub(col[lane], zcmul(r0, rb));
        col[lane] = v;
        if (lane == b) dg[b] = v.x;
      }
      if (g1) {
        const zc v = zsub(col[lane + 32], zcmul(r1, rb));
        col[lane + 32] = v;
        if (lane + 32 == b) dg[b] = v.x;
      }
      if (lane == 0) col[p] = rb;   // R(j, b) over G(p, b): row p is never read again
    }
    gbar(bid, nth);
  }
  const int kk = j;
  if (gw == 0 && lane == 0) {
    int q = kk;
    for (int c = 0; c < k; ++c)
      if (!(done >> c & 1ull)) perm[q++] = c;
  }
  gbar(bid, nth);
  for (int e = gw * 32 + lane; e < k * k; e += nth) {
    const int r = e % k, c = e / k;   // element (r, c) of the pivoted R
    tmp[e] = (r < kk && c >= r) ? G[perm[c] * k + perm[r]] : zmk(0.0, 0.0);
  }
  gbar(bid, nth);
  for (int e = gw * 32 + lane; e < k * k; e += nth) G[e] = tmp[e];
  gbar(bid, nth);
  return kk;
}

// Z (kk x r, ld kk, shared) <- R11^{-1} Z with R11 = rows/cols 0..kk-1 of R (ld k, upper),
// then row j scaled by sc[j]; one warp per column, lanes hold rows lane, lane + 32
__device__ void tri_solve_cols(const zc* R, int k, int kk, zc* Z, int r, const double* sc) {
  // a warp carries three columns through the back substitution together (the row of R and
  // the reciprocal pivot are loaded once per step, the three chains interleave)
  __shared__ double dinv[KG];
  constexpr int NC = 3;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = threadIdx.x; a < kk; a += NT) dinv[a] = 1.0 / R[a * k + a].x;
  __syncthreads();
  for (int l0 = w; l0 < r; l0 += NW * NC) {
    zc x0[NC], x1[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int l = l0 + c * NW;
      const zc* z = Z + (int64_t)l * kk;
      x0[c] = (l < r && lane < kk) ? z[lane] : zmk(0.0, 0.0);
      x1[c] = (l < r && lane + 32 < kk) ? z[lane + 32] : zmk(0.0, 0.0);
    }
    for (int a = kk - 1; a >= 0; --a) {
      const zc ra0 = lane < a ? R[a * k + lane] : zmk(0.0, 0.0);
      const zc ra1 = lane + 32 < a ? R[a * k + lane + 32] : zmk(0.0, 0.0);
      const double di = dinv[a];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const zc own = a >= 32 ? x1[c] : x0[c];
        const zc xa = zscale(zshfl(own, a & 31), di);
        if (lane == (a & 31)) {
          if (a >= 32) x1[c] = xa;
          else x0[c] = xa;
        }
        x0[c] = zsub(x0[c], zmul(ra0, xa));
        x1[c] = zsub(x1[c], zmul(ra1, xa));
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int l = l0 + c * NW;
      if (l >= r) continue;
      zc* z = Z + (int64_t)l * kk;
      if (lane < kk) z[lane] = zscale(x0[c], sc[lane]);
      if (lane + 32 < kk) z[lane + 32] = zscale(x1[c], sc[lane + 32]);
    }
  }
  __syncthreads();
}

// O (mo x r, ld mo, global) = X[:, perm[0..kk)] T (kk x r, ld kk, shared), rows [i_lo, i_hi)
__device__ void apply_sel(const zc* __restrict__ X, int mo, int ldx, int i_lo, int i_hi, const int* perm, int kk,
                          const zc* T, int r, zc* __restrict__ O) {
  const int ng = (r + 7) / 8, mr = i_hi - i_lo;
  for (int e = threadIdx.x; e < mr * ng; e += NT) {
    const int i = i_lo + e % mr, l0 = 8 * (e / mr);
    zc acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = zmk(0.0, 0.0);
    for (int j0 = 0; j0 < kk; j0 += 8) {
      zc x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = j0 + u < kk ? X[(int64_t)perm[j0 + u] * ldx + i] : zmk(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < kk)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (l0 + q < r) zfma(acc[q], x[u], T[(l0 + q) * kk + j0 + u]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (l0 + q < r) O[(int64_t)(l0 + q) * mo + i] = acc[q];
  }
}

// DMMA form of apply_sel: a warp per 8-row block of O; the A fragments of the whole
// inner dimension (kk <= 64: 16 four-column steps) are loaded up front (gathered columns
// perm[j] of X, 8 consecutive rows per column), then every 8-column block of O is one
// chain of 4 DMMA per step against T's fragments in shared memory.
__device__ __noinline__ void apply_sel_mma(const Src2 X, int mo, int i_lo, int i_hi, const int* perm, int kk,
                                           const zc* T, int r, zc* O) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fk = lane & 3;
  const int nrb = (i_hi - i_lo + 7) >> 3, nks = (kk + 3) >> 2, ncb = (r + 7) >> 3;
  for (int rb = w; rb < nrb; rb += NW) {
    const int i = i_lo + rb * 8 + fr;
    zc a[KG / 4];
#pragma unroll
    for (int s = 0; s < KG / 4; ++s) {
      const int j = 4 * s + fk;
      a[s] = (s < nks && j < kk && i < i_hi) ? X.col(perm[j])[i] : zmk(0.0, 0.0);
    }
    for (int cb = 0; cb < ncb; ++cb) {
      double c[4] = {0.0, 0.0, 0.0, 0.0};
      const int l = cb * 8 + fr;
#pragma unroll
      for (int s = 0; s < KG / 4; ++s) {
        if (s >= nks) break;
        const int j = 4 * s + fk;
        const zc b = (j < kk && l < r) ? T[l * kk + j] : zmk(0.0, 0.0);
        zdmma(c, a[s], b);
      }
      const int row = i_lo + rb * 8 + fr;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int col = cb * 8 + 2 * fk + jj;
        if (col < r && row < i_hi) O[(int64_t)col * mo + row] = zmk(c[jj], c[2 + jj]);
      }
    }
  }
}

// Hermitian eigenproblem H (n x n, ld n, shared) = X diag(h) X^H by cyclic two-sided
// Jacobi with the round-robin parallel ordering; X (ld n, shared) enters as I.  The
// rotation of pair (p, q) is the one of jacobi_nw for the 2 x 2 Gram [h_pp h_pq; . h_qq].
// Returns the number of sweeps.
__device__ int g_jacobi_threads = NT;   // threads of the Jacobi sweeps (CBIE_JACOBI_T, launch_gram)
__device__ int g_gram_onesided = 0;     // 1: one-sided Jacobi on R^H (CBIE_ONESIDED_JACOBI, launch_gram)

__device__ int herm_jacobi(zc* H, int n, zc* X, Smem& S) {
  // the first JT threads run the sweeps (named barrier 3); the others wait at the end
  const int JT = g_jacobi_threads;
  __shared__ double rc[KG / 2 + 1];
  __shared__ zc rs[KG / 2 + 1];
  __shared__ int rp[KG / 2 + 1], rq[KG / 2 + 1];
  __shared__ double red[NW];
  __shared__ int nsw;
  if (n < 2) return 0;
  if (threadIdx.x < JT) {
    const int tid = threadIdx.x, lane = tid & 31, wj = tid >> 5;
    auto jsum = [&](double v) {
      v = warp_sum(v);
      gbar(3, JT);
      if (lane == 0) red[wj] = v;
      gbar(3, JT);
      double t = 0.0;
      for (int i = 0; i < JT / 32; ++i) t += red[i];
      return t;
    };
    const int ne = n + (n & 1), np = ne / 2;
    double f2 = 0.0;
    for (int e = tid; e < n * n; e += JT) f2 += zabs2(H[e]);
    f2 = jsum(f2);
    int sweep = 0;
    for (; sweep < 30; ++sweep) {
      double off = 0.0;
      for (int e = tid; e < n * n; e += JT)
        if (e % n != e / n) off += zabs2(H[e]);
      off = jsum(off);
      if (!(off > 1e-20 * f2)) break;
      for (int rd = 0; rd < ne - 1; ++rd) {
        // rotation of every pair (round-robin ordering); an index >= n pairs with identity
        if (tid < np) {
          const int t = tid;
          const int pb = ne - 1 - t;
          const int p = t == 0 ? 0 : ((t - 1 + rd) % (ne - 1)) + 1;
          const int q = pb == 0 ? 0 : ((pb - 1 + rd) % (ne - 1)) + 1;
          double cs = 1.0;
          zc se = zmk(0.0, 0.0);
          if (p < n && q < n) {
            const double al = H[p * n + p].x, be = H[q * n + q].x;
            const zc gm = H[q * n + p];   // h_pq
            // same rotation as before (|h_pq| > 1e-17 sqrt(|h_pp h_qq|), tan from zeta) with
            // half the dependent sqrt / divide chain: this single warp's latency is what the
            // other fifteen wait for at the barrier below
            const double g2 = zabs2(gm);
            if (g2 > 1e-290 && g2 > 1e-34 * fabs(al * be)) {
              const double ig = rsqrt(g2);
              const double zeta = (be - al) * 0.5 * ig;
              const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              cs = rsqrt(1.0 + tt * tt);
              const double sn = cs * tt;
              se = zmk(gm.x * ig * sn, gm.y * ig * sn);
            }
          }
          rp[t] = p;
          rq[t] = q;
          rc[t] = cs;
          rs[t] = se;
        }
        gbar(3, JT);
        // H <- J^H H J by disjoint 2 x 2 blocks (rows of pair t1, columns of pair t2),
        // X <- X J by (row, pair) items; no two items touch the same entry.
        // J = [cs se; -conj(se) cs] acts on the (p, q) columns.
        // item -> (index, pair) through float reciprocals: exact for these sizes (e + 0.5 is
        // never within rounding of a multiple of np / n), no integer division per item
        const float rnp = 1.0f / (float)np, rn = 1.0f / (float)n;
        for (int e = tid; e < np * np + n * np; e += JT) {
          if (e < np * np) {
            const int t2 = (int)(((float)e + 0.5f) * rnp), t1 = e - t2 * np;
            const int a0 = rp[t1], a1 = rq[t1], b0 = rp[t2], b1 = rq[t2];
            const bool va0 = a0 < n, va1 = a1 < n, vb0 = b0 < n, vb1 = b1 < n;
            const double c1 = rc[t1], c2 = rc[t2];
            const zc s1 = rs[t1], s2 = rs[t2];
            const zc z0 = zmk(0.0, 0.0);
            const zc hpp = va0 && vb0 ? H[b0 * n + a0] : z0, hpq = va0 && vb1 ? H[b1 * n + a0] : z0;
            const zc hqp = va1 && vb0 ? H[b0 * n + a1] : z0, hqq = va1 && vb1 ? H[b1 * n + a1] : z0;
            const zc cpp = zsub(zscale(hpp, c2), zmul(zconj(s2), hpq));
            const zc cpq = zadd(zmul(s2, hpp), zscale(hpq, c2));
            const zc cqp = zsub(zscale(hqp, c2), zmul(zconj(s2), hqq));
            const zc cqq = zadd(zmul(s2, hqp), zscale(hqq, c2));
            if (va0 && vb0) H[b0 * n + a0] = zsub(zscale(cpp, c1), zmul(s1, cqp));
            if (va0 && vb1) H[b1 * n + a0] = zsub(zscale(cpq, c1), zmul(s1, cqq));
            if (va1 && vb0) H[b0 * n + a1] = zadd(zmul(zconj(s1), cpp), zscale(cqp, c1));
            if (va1 && vb1) H[b1 * n + a1] = zadd(zmul(zconj(s1), cpq), zscale(cqq, c1));
          } else {
            const int f = e - np * np;
            const int t = (int)(((float)f + 0.5f) * rn), i = f - t * n;
            const int p = rp[t], q = rq[t];
            if (p >= n || q >= n) continue;
            const double cs = rc[t];
            const zc se = rs[t];
            const zc xi = X[p * n + i], yi = X[q * n + i];
            X[p * n + i] = zsub(zscale(xi, cs), zmul(zconj(se), yi));
            X[q * n + i] = zadd(zmul(se, xi), zscale(yi, cs));
          }
        }
        gbar(3, JT);
      }
    }
    if (tid == 0) nsw = sweep;
  }
  __syncthreads();
  return nsw;
}

// Cluster execution (k_trunc_gram launched with clusters of csize CTAs per problem):
// every CTA accumulates the Gram partials of its row slice, the partials are summed
// in cluster-rank order through distributed shared memory (each CTA gets the same
// bits), every CTA then runs the identical k x k work redundantly (no further
// exchange), and the final applies are again split by rows.  csize = 1: the plain
// one-CTA-per-problem kernel.

// G (k x k, shared) <- sum over the cluster's CTAs of their G (rank order); tmp: k x k shared
__device__ void cluster_gram_sum(zc* G, int k, zc* tmp) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  if (C == 1) return;
  cl.sync();
  for (int e = threadIdx.x; e < k * k; e += NT) {
    zc acc = zmk(0.0, 0.0);
    for (int q = 0; q < C; ++q) {
      const zc v = cl.map_shared_rank(G, q)[e];
      acc = zmk(acc.x + v.x, acc.y + v.y);
    }
    tmp[e] = acc;
  }
  cl.sync();   // every CTA has read every partial
  for (int e = threadIdx.x; e < k * k; e += NT) G[e] = tmp[e];
  __syncthreads();
}

// Small complex product on the FP64 tensor pipe: C(i, j) = sum_{c < K} A(i, c) B(c, j),
// i < M, j < N, for the k x k steps of the Gram path (operands in shared or L2-resident
// global memory, read straight into the m8n8k4 fragments through the functors fa / fb; st
// stores one entry).  All NW warps; a warp takes 8 x 16 strips (two tiles share the A
// fragment).  Callers synchronise afterwards.
template <class FA, class FB, class FS>
__device__ __forceinline__ void kk_gemm_mma(int M, int N, int K, FA fa, FB fb, FS st) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, fr = lane & 3, fc = lane >> 2;
  const int tm = (M + 7) >> 3, tn = (N + 15) >> 4;
  for (int t = w; t < tm * tn; t += NW) {
    const int i0 = (t % tm) * 8, j0 = (t / tm) * 16;
    double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
    const int i = i0 + fc, ja = j0 + fc, jb = j0 + 8 + fc;
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int kk = k0 + fr;
      const bool kv = kk < K;
      const zc a = (kv && i < M) ? fa(i, kk) : zmk(0.0, 0.0);
      const zc b0 = (kv && ja < N) ? fb(kk, ja) : zmk(0.0, 0.0);
      const zc b1 = (kv && jb < N) ? fb(kk, jb) : zmk(0.0, 0.0);
      zdmma(c0, a, b0);
      zdmma(c1, a, b1);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int oj = j0 + 2 * fr + j;
      if (i < M && oj < N) st(i, oj, zmk(c0[j], c0[2 + j]));
      if (i < M && oj + 8 < N) st(i, oj + 8, zmk(c1[j], c1[2 + j]));
    }
  }
}

// One Gram-path recompression (steps 1-5 above) of U (m x k, ldu) Vt (n x k, ldv),
// k <= KG: writes Uo (m x r, ld m), Vo (n x r, ld n) and returns r (0: zero product);
// r is clipped at cap (counted in overflow).  sc: per-CTA scratch (4 GSQ).
// su / sv: the factors (possibly two pieces each, read in place; Uo / Vo may overwrite the
// first pieces: every row block is loaded completely before its output rows are stored);
// the U columns from ksgn on carry the factor sgn (folded into the column balancing).
__device__ int gram_stage(const Src2 su, const Src2 sv, int ksgn, double sgn, int m, int n, int k, zc* Uo, zc* Vo,
                          int cap, double tol, zc* sc, unsigned long long* overflow, Smem& S, zc* sm,
                          long long* tc, int* sweeps_out) {
  const zc* U = su.p1;
  const zc* Vt = sv.p1;
  const int ldu = su.ld1, ldv = sv.ld1;
  __shared__ double alpha[KG], ainv[KG], scu[KG], scv[KG];
  __shared__ int pu[KG], pv[KG], posu[KG], posv[KG];
  zc* Gu = sm;
  zc* Gv = sm + GSQ;
  zc* X2 = sm + 2 * GSQ;
  const int crank = cl_rank(), csize = cl_size();
  const int mu0 = slice_lo(m, crank, csize), mu1 = slice_lo(m, crank + 1, csize);
  const int nv0 = slice_lo(n, crank, csize), nv1 = slice_lo(n, crank + 1, csize);
  if (threadIdx.x == 0 && crank == 0) flop_add(8.0 * (m + n) * (double)k * k);
  zc* Rug = sc;
  zc* Rvg = sc + GSQ;
  zc* Mg = sc + 2 * GSQ;
  zc* Vhg = sc + 3 * GSQ;

  // 1. Gram matrices
  for (int e = threadIdx.x; e < 2 * GSQ; e += NT) sm[e] = zmk(0.0, 0.0);
  __syncthreads();
  if (g_gram_mma) {   // staging in Gv's region (+ X2's head): free until G_v is stored
    gram_acc_mma(su, mu0, mu1, k, Gu, Gv);
    gram_acc_mma(sv, nv0, nv1, k, Gv, Gv);
  } else {
    gram_acc(U, mu0, mu1, k, ldu, Gu, X2);
    gram_acc(Vt, nv0, nv1, k, ldv, Gv, X2);
  }
  cluster_gram_sum(Gu, k, X2);
  cluster_gram_sum(Gv, k, X2);
  // 2. balancing
  for (int c = threadIdx.x; c < k; c += NT) {
    const double du = Gu[c * k + c].x, dv = Gv[c * k + c].x;
    const double a = (du > 0.0 && dv > 0.0) ? sqrt(sqrt(dv / du)) : 0.0;
    alpha[c] = c >= ksgn ? sgn * a : a;   // the sign of the second U piece rides on its scale
    ainv[c] = a > 0.0 ? 1.0 / a : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += NT) {
    const int a = e % k, b = e / k;
    Gu[b * k + a] = zscale(Gu[b * k + a], alpha[a] * alpha[b]);
    Gv[b * k + a] = zscale(Gv[b * k + a], ainv[a] * ainv[b]);
  }
  __syncthreads();
  tc[1] = clock64();
  long long tf = tc[1];
  auto stamp = [&](int slot) {
    const long long t = clock64();
    tc[slot] += t - tf;
    tf = t;
  };
  // 3. pivoted Choleskys of both Grams concurrently: warps 0..NW/2-1 factor G_u (X2 as
  //    gather space), the others G_v (gather through the global scratch Rvg, written later)
  __shared__ int kuv[2];
  {
    const int w = threadIdx.x >> 5, GW = g_pchol_w;   // warps per factorisation
    const bool ga = w < GW, gb = w >= NW / 2 && w < NW / 2 + GW;
    if (ga || gb) {
      const int kr = pchol_grp(ga ? Gu : Gv, k, ga ? pu : pv, CHOL_EPS, false, GW, ga ? w : w - NW / 2,
                               ga ? 1 : 2, ga ? X2 : Rvg, ga ? scu : scv);
      if ((threadIdx.x & (NT / 2 - 1)) == 0) kuv[ga ? 0 : 1] = kr;
    }
    __syncthreads();
  }
  const int ku = kuv[0], kv = kuv[1];
  stamp(5);
  if (ku == 0 || kv == 0) return 0;
  for (int c = threadIdx.x; c < k; c += NT) {
    posu[pu[c]] = c;
    posv[pv[c]] = c;
  }
  __syncthreads();
  // 4. core M = (R_u P_u^T)(R_v P_v^T)^T  (ku x kv), kept in global for U' = M Vhat
  if (g_gram_mma) {
    kk_gemm_mma(
        ku, kv, k,
        [&](int a, int c) { const int ju = posu[c]; return ju >= a ? Gu[ju * k + a] : zmk(0.0, 0.0); },
        [&](int c, int b) { const int jv = posv[c]; return jv >= b ? Gv[jv * k + b] : zmk(0.0, 0.0); },
        [&](int a, int b, zc v) { X2[b * ku + a] = v; });
  } else {
    for (int e = threadIdx.x; e < ku * kv; e += NT) {
      const int a = e % ku, b = e / ku;
      zc s = zmk(0.0, 0.0);
      for (int c = 0; c < k; ++c) {
        const int ju = posu[c], jv = posv[c];
        if (ju >= a && jv >= b) zfma(s, Gu[ju * k + a], Gv[jv * k + b]);
      }
      X2[e] = s;
    }
  }
  for (int e = threadIdx.x; e < k * k; e += NT) {
    Rug[e] = Gu[e];
    Rvg[e] = Gv[e];
  }
  __syncthreads();
  const int kk1 = ku, kk2 = kv;
  // 5. SVD of the core through H = M M^H, preconditioned: pivoted Cholesky
  //    P^T H P = R^H R (stopped once the remaining trace is <= (GDELTA tol)^2 of the
  //    largest diagonal, i.e. the dropped directions carry <= GDELTA tol s_0 together),
  //    then the graded G = R R^H = Z S^2 Z^H by two-sided
  //    Jacobi (few sweeps).  Left singular vectors times S: W = P R^H Z; right
  //    singular vectors: Vhat = M^H W / S^2.  Singular values below ~sqrt(eps) s_0
  //    are not resolved, far below tol * s_0.
  zc* H = Gu;
  if (g_gram_mma) {
    kk_gemm_mma(
        kk1, kk1, kk2, [&](int a, int c) { return X2[c * kk1 + a]; },
        [&](int c, int b) { return zconj(X2[c * kk1 + b]); }, [&](int a, int b, zc v) { H[b * kk1 + a] = v; });
  } else {
    for (int e = threadIdx.x; e < kk1 * kk1; e += NT) {
      const int a = e % kk1, b = e / kk1;
      zc s = zmk(0.0, 0.0);
      for (int c = 0; c < kk2; ++c) zfma(s, X2[c * kk1 + a], zconj(X2[c * kk1 + b]));
      H[b * kk1 + a] = s;
    }
  }
  for (int e = threadIdx.x; e < kk1 * kk2; e += NT) Mg[e] = X2[e];
  __syncthreads();
  stamp(6);
  __shared__ int kps;
  if ((threadIdx.x >> 5) < g_pcholh_w) {
    const int kq = pchol_grp(H, kk1, S.perm, (GDELTA * tol) * (GDELTA * tol), true, g_pcholh_w, threadIdx.x >> 5, 1,
                             X2, scu);
    if (threadIdx.x == 0) kps = kq;
  }
  __syncthreads();
  const int kp = kps;
  stamp(7);
  int sweeps = 0;
  if (g_gram_onesided) {
    // one-sided Jacobi on B = R^H (kk1 x kp, X2's region): rotating column pairs until
    // they are orthogonal gives B Z = R^H Z = (left singular vectors) x Sigma directly --
    // no R R^H product, no eigenvector accumulation, one barrier per round (jacobi_nw,
    // half-warp per pair)
    zc* B = X2;
    for (int e = threadIdx.x; e < kk1 * kp; e += NT) {
      const int a = e % kk1, c = e / kk1;
      B[e] = a >= c ? zconj(H[a * kk1 + c]) : zmk(0.0, 0.0);   // conj(R(c, a))
    }
    __syncthreads();
    stamp(8);
    tc[2] = clock64();
    sweeps = jacobi_nw(B, kk1, kp, kk1, S);
    for (int c = threadIdx.x >> 5; c < kp; c += NW) {   // warp per column norm
      double ns = 0.0;
      for (int q = threadIdx.x & 31; q < kk1; q += 32) ns += zabs2(B[c * kk1 + q]);
      ns = warp_sum(ns);
      if ((threadIdx.x & 31) == 0) S.sig[c] = sqrt(ns);
    }
    __syncthreads();
  } else {
    zc* Gp = Gv;   // R R^H (kp x kp)
    zc* Z = X2;    // eigenvectors (kp x kp)
    if (g_gram_mma) {
      kk_gemm_mma(
          kp, kp, kk1, [&](int a, int j) { return j >= a ? H[j * kk1 + a] : zmk(0.0, 0.0); },
          [&](int j, int b) { return j >= b ? zconj(H[j * kk1 + b]) : zmk(0.0, 0.0); },
          [&](int a, int b, zc v) { Gp[b * kp + a] = v; });
      for (int e = threadIdx.x; e < kp * kp; e += NT) Z[e] = zmk(e % kp == e / kp ? 1.0 : 0.0, 0.0);
    } else {
      for (int e = threadIdx.x; e < kp * kp; e += NT) {
        const int a = e % kp, b = e / kp;
        zc s = zmk(0.0, 0.0);
        for (int j = max(a, b); j < kk1; ++j) zfma(s, H[j * kk1 + a], zconj(H[j * kk1 + b]));
        Gp[b * kp + a] = s;
        Z[b * kp + a] = zmk(a == b ? 1.0 : 0.0, 0.0);
      }
    }
    __syncthreads();
    stamp(8);
    tc[2] = clock64();
    sweeps = herm_jacobi(Gp, kp, Z, S);
    for (int c = threadIdx.x; c < kp; c += NT) S.sig[c] = sqrt(fmax(Gp[c * kp + c].x, 0.0));
    __syncthreads();
  }
  for (int c = threadIdx.x; c < kp; c += NT) {
    int pos = 0;
    for (int o = 0; o < kp; ++o)
      if (S.sig[o] > S.sig[c] || (S.sig[o] == S.sig[c] && o < c)) ++pos;
    S.order[pos] = c;
  }
  __syncthreads();
  tc[3] = clock64();
  const double s0 = kp > 0 ? S.sig[S.order[0]] : 0.0;
  int r = 0;
  if (s0 > 0.0) {
    for (int c = 0; c < kp; ++c)
      if (S.sig[c] > tol * s0) ++r;
    r = max(r, 1);
  }
  if (r > cap) {
    if (threadIdx.x == 0 && crank == 0) atomicAdd(overflow, 1ull);
    r = cap;
  }
  // W = P R^H Z_r (kk1 x r) in Gv's region (G dead: S.sig holds its diagonal)
  __syncthreads();
  zc* W = Gv;
  if (g_gram_onesided) {
    for (int e = threadIdx.x; e < kk1 * r; e += NT) {
      const int j = e % kk1, l = e / kk1;
      W[(int64_t)l * kk1 + S.perm[j]] = X2[S.order[l] * kk1 + j];
    }
  } else {
    const zc* Z = X2;
    if (g_gram_mma) {
      kk_gemm_mma(
          kk1, r, kp, [&](int j, int a) { return a <= j ? zconj(H[j * kk1 + a]) : zmk(0.0, 0.0); },
          [&](int a, int l) { return Z[S.order[l] * kp + a]; },
          [&](int j, int l, zc v) { W[(int64_t)l * kk1 + S.perm[j]] = v; });
    } else {
      for (int e = threadIdx.x; e < kk1 * r; e += NT) {
        const int j = e % kk1, l = e / kk1;
        const int c = S.order[l];
        zc s = zmk(0.0, 0.0);
        for (int a = 0; a <= min(j, kp - 1); ++a) zfma(s, zconj(H[j * kk1 + a]), Z[c * kp + a]);
        W[(int64_t)l * kk1 + S.perm[j]] = s;
      }
    }
  }
  __syncthreads();
  // conj(Vhat) = conj(M^H W / S^2) (kk2 x r) to global
  if (g_gram_mma) {
    kk_gemm_mma(
        kk2, r, kk1, [&](int b, int a) { return zconj(Mg[b * kk1 + a]); },
        [&](int a, int l) { return W[(int64_t)l * kk1 + a]; },
        [&](int b, int l, zc v) {
          const double sg = S.sig[S.order[l]];
          Vhg[(int64_t)l * kk2 + b] = zconj(zscale(v, 1.0 / (sg * sg)));
        });
  } else {
    for (int e = threadIdx.x; e < kk2 * r; e += NT) {
      const int b = e % kk2, l = e / kk2;
      const double sg = S.sig[S.order[l]];
      zc s = zmk(0.0, 0.0);
      for (int a = 0; a < kk1; ++a) zfma(s, zconj(Mg[b * kk1 + a]), W[(int64_t)l * kk1 + a]);
      Vhg[(int64_t)l * kk2 + b] = zconj(zscale(s, 1.0 / (sg * sg)));
    }
  }
  for (int j = threadIdx.x; j < kk1; j += NT) scu[j] = alpha[pu[j]];
  for (int j = threadIdx.x; j < kk2; j += NT) scv[j] = ainv[pv[j]];
  for (int e = threadIdx.x; e < k * k; e += NT) X2[e] = Rug[e];
  __syncthreads();
  tf = clock64();
  tc[9] += tf - tc[3];
  // 6a. U' = U_sel D R_u11^{-1} W
  tri_solve_cols(X2, k, kk1, W, r, scu);
  stamp(10);
  if (r > 0) {
    if (g_gram_mma) apply_sel_mma(su, m, mu0, mu1, pu, kk1, W, r, Uo);
    else apply_sel(U, m, ldu, mu0, mu1, pu, kk1, W, r, Uo);
  }
  __syncthreads();
  stamp(11);
  // 6b. Vt' = Vt_sel D^{-1} R_v11^{-1} conj(Vhat)
  zc* W2 = Gu;
  for (int e = threadIdx.x; e < k * k; e += NT) X2[e] = Rvg[e];
  for (int e = threadIdx.x; e < kk2 * r; e += NT) W2[e] = Vhg[e];
  __syncthreads();
  tri_solve_cols(X2, k, kk2, W2, r, scv);
  if (r > 0) {
    if (g_gram_mma) apply_sel_mma(sv, n, nv0, nv1, pv, kk2, W2, r, Vo);
    else apply_sel(Vt, n, ldv, nv0, nv1, pv, kk2, W2, r, Vo);
  }
  if (threadIdx.x == 0 && crank == 0)
    // applies, pivoted Choleskys, M and H products, Jacobi sweeps (Gram counted above)
    flop_add(8.0 * ((double)m * kk1 + (double)n * kk2) * r + 16.0 * k * (double)k * k / 3.0 +
             8.0 * kk1 * (double)kk2 * (k + kk1) + 32.0 * sweeps * (double)kp * kp * kp);
  *sweeps_out = sweeps;
  __syncthreads();
  return r;
}

// Multi-stage Gram path for KG < k <= KMS: the columns are taken in batches, each
// batch recompressed together with the basis kept so far ([U_r | next columns],
// r + batch <= KG), ping-ponging between two scratch bases; the last stage writes
// the output.  Every stage truncates at tol relative to its own largest singular
// value (the reference truncates once): the error stays O(tol s_0), inside the
// solution-level budget.  A problem whose kept rank leaves no room (r == KG with
// columns left) is handed to the Householder kernels through defer.
constexpr int KMS = 4 * KG;

__host__ __device__ inline int64_t gram_ms_scratch(int mn_max) { return 4 * (int64_t)mn_max * KG; }

__global__ void __launch_bounds__(NT, 1)
    k_trunc_gram(zc* arena, zc* aout, int* ranks, const TruncDesc* __restrict__ descs, zc* scratch, int64_t per,
                 double tol, unsigned long long* overflow, unsigned long long* prof, int* defer, int base,
                 const int* idx, int mn_max) {
  __shared__ Smem S;
  extern __shared__ __align__(16) unsigned char smraw[];
  zc* sm = reinterpret_cast<zc*>(smraw);
  // one problem per cluster (csize CTAs, cluster_gram_sum); pb = problem of this cluster
  const int crank = cl_rank(), csize = cl_size();
  const int pb = (int)blockIdx.x / csize;
  // idx: run the problems listed in idx[1 + base + pb] (count idx[0]) of descs
  if (idx && base + pb >= idx[0]) return;
  const int tix = idx ? idx[1 + base + pb] : pb;
  const TruncDesc d = descs[tix];
  long long tc[12] = {};
  tc[0] = clock64();
  if (d.skip_slot >= 0 && ranks[d.skip_slot] == 0) return;
  const int k = trunc_k(d, ranks);
  const bool two = d.in_u2 >= 0;
  const int k1 = two ? trunc_k1(d, ranks) : 0x7fffffff;
  const int m = d.m, n = d.n;
  if (k <= 0 || m == 0 || n == 0) {
    if (threadIdx.x == 0 && crank == 0) ranks[d.out_slot] = 0;
    return;
  }
  const bool multi = k > KG && k <= KMS && max(m, n) <= mn_max;
  // hand-off to the Householder kernels; a two-source problem has no materialised input for
  // them: counted as a clipped truncation (re-factorisation with concatenations)
  auto hand_off = [&]() {
    if (threadIdx.x == 0 && crank == 0) {
      if (two) atomicAdd(overflow, 1ull);
      else defer[1 + atomicAdd(defer, 1)] = idx ? tix : base + pb;
    }
  };
  if (k > KG && !multi) {
    hand_off();
    return;
  }
  const zc* U = arena + d.in_u;
  const zc* Vt = arena + d.in_v;
  const Src2 su = two ? Src2{U, arena + d.in_u2, d.ldu, d.ldu2, k1} : src1(U, d.ldu);
  const Src2 sv = two ? Src2{Vt, arena + d.in_v2, d.ldv, d.ldv2, k1} : src1(Vt, d.ldv);
  const double sgn = two ? d.sgn2 : 1.0;
  zc* sc = scratch + (int64_t)blockIdx.x * per;                  // private k x k scratch
  zc* sc0 = scratch + (int64_t)(blockIdx.x - crank) * per;      // the cluster's shared bases
  const int mu0 = slice_lo(m, crank, csize), mu1 = slice_lo(m, crank + 1, csize);
  const int nv0 = slice_lo(n, crank, csize), nv1 = slice_lo(n, crank + 1, csize);
  zc* Uo = aout + d.out_u;
  zc* Vo = aout + d.out_v;
  int sweeps = 0, r = 0;
  if (!multi) {
    r = gram_stage(su, sv, k1, sgn, m, n, k, Uo, Vo, d.cap, tol, sc, overflow, S, sm, tc, &sweeps);
  } else {
    zc* bu[2] = {sc0 + 4 * GSQ, sc0 + 4 * GSQ + (int64_t)2 * mn_max * KG};
    zc* bv[2] = {bu[0] + (int64_t)mn_max * KG, bu[1] + (int64_t)mn_max * KG};
    int cur = 0, done = KG;
    r = gram_stage(su, sv, k1, sgn, m, n, KG, bu[0], bv[0], KG, tol, sc, overflow, S, sm, tc, &sweeps);
    while (done < k) {
      const int add = min(KG - r, k - done);
      // too little room left for the remaining columns (each stage costs a full Gram
      // recompression): Householder kernels -- nothing was written to the output yet
      if (add < min(g_ms_min_add, k - done)) {
        hand_off();
        return;
      }
      // append the next columns behind the kept basis (this CTA's rows; the next Gram
      // stage reads the same rows)
      const int mr = mu1 - mu0, nr = nv1 - nv0;
      for (int e = threadIdx.x; e < add * mr; e += NT) {
        const int c = e / mr, i = mu0 + e % mr;
        const zc v = su.col(done + c)[i];
        bu[cur][(int64_t)(r + c) * m + i] = done + c >= k1 ? zscale(v, sgn) : v;
      }
      for (int e = threadIdx.x; e < add * nr; e += NT) {
        const int c = e / nr, i = nv0 + e % nr;
        bv[cur][(int64_t)(r + c) * n + i] = sv.col(done + c)[i];
      }
      __syncthreads();
      done += add;
      const bool last = done == k;
      int sw = 0;
      r = gram_stage(src1(bu[cur], m), src1(bv[cur], n), 0x7fffffff, 1.0, m, n, r + add, last ? Uo : bu[cur ^ 1],
                     last ? Vo : bv[cur ^ 1],
                     last ? d.cap : KG, tol, sc, overflow, S, sm, tc, &sw);
      sweeps += sw;
      cur ^= 1;
    }
  }
  if (threadIdx.x == 0 && crank == 0) {
    ranks[d.out_slot] = r;
    if (prof && max(m, n) >= g_prof_mn && k >= g_prof_kmin) {
      const long long tc4 = clock64();
      atomicAdd(prof + 0, (unsigned long long)(tc[1] - tc[0]));
      atomicAdd(prof + 1, (unsigned long long)(tc[2] - tc[1]));
      atomicAdd(prof + 2, (unsigned long long)(tc[3] - tc[2]));
      atomicAdd(prof + 3, (unsigned long long)(tc4 - tc[3]));
      atomicAdd(prof + 4, 1ull);
      atomicAdd(prof + 5, (unsigned long long)sweeps);
      atomicAdd(prof + 14, 1ull);
      atomicAdd(prof + 15, (unsigned long long)(tc4 - tc[0]));
      for (int q = 5; q < 12; ++q) atomicAdd(prof + 11 + q, (unsigned long long)tc[q]);
    }
  }
}

// clusters of csize CTAs of k_trunc_gram the device can hold at once (a cluster needs csize
// free SMs inside ONE GPC, so this is below 148 / csize: 32 clusters of 4 on a B200)
int gram_max_clusters(int csize) {
  const int smem = (3 * GSQ + KG + 1) * (int)sizeof(zc);
  if (cudaFuncSetAttribute(k_trunc_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(148 * csize));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_trunc_gram, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void launch_gram(zc* arena, zc* aout, int* ranks, const TruncDesc* d_desc, int nd, double tol,
                 unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, unsigned long long* prof,
                 int* defer, const int* idx, int mn_max, int csize) {
  // mn_max > 0: problems with KG < k <= KMS and max(m, n) <= mn_max run the multi-stage path
  const int64_t per = gram_scratch_per() + (mn_max > 0 ? gram_ms_scratch(mn_max) : 0);
  csize = std::max(1, std::min(csize, 8));
  // one launch per group whenever 2 GB of scratch allow it (a second launch of the tail
  // would wait for the whole first one on the stream)
  static const int ws_gb = getenv("CBIE_GRAM_WS_GB") ? atoi(getenv("CBIE_GRAM_WS_GB")) : 2;
  const int wave = (int)std::max<int64_t>(1, (int64_t)ws_cap(ws_gb) / (per * csize * (int64_t)sizeof(zc)));
  const size_t need = (size_t)std::min(wave, nd) * csize * per;
  if (scratch.n < need) scratch.alloc(need);
  const int smem = (3 * GSQ + KG + 1) * (int)sizeof(zc);
  CK(cudaFuncSetAttribute(k_trunc_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (getenv("CBIE_PROF_MN") || getenv("CBIE_PROF_KMIN")) {
    const int z = getenv("CBIE_PROF_MN") ? atoi(getenv("CBIE_PROF_MN")) : 0;
    const int y = getenv("CBIE_PROF_KMIN") ? atoi(getenv("CBIE_PROF_KMIN")) : 0;
    CK(cudaMemcpyToSymbol(g_prof_mn, &z, sizeof(int)));
    CK(cudaMemcpyToSymbol(g_prof_kmin, &y, sizeof(int)));
  }
  if (getenv("CBIE_MS_MIN_ADD")) {
    const int z = std::max(1, atoi(getenv("CBIE_MS_MIN_ADD")));
    CK(cudaMemcpyToSymbol(g_ms_min_add, &z, sizeof(int)));
  }
  if (getenv("CBIE_PCHOL_W")) {
    const int z = std::max(1, std::min(NW / 2, atoi(getenv("CBIE_PCHOL_W"))));
    CK(cudaMemcpyToSymbol(g_pchol_w, &z, sizeof(int)));
  }
  if (getenv("CBIE_PCHOLH_W")) {
    const int z = std::max(1, std::min(NW, atoi(getenv("CBIE_PCHOLH_W"))));
    CK(cudaMemcpyToSymbol(g_pcholh_w, &z, sizeof(int)));
  }
  if (getenv("CBIE_NO_DMMA")) {   // A/B knob: DFMA Gram accumulation and applies
    const int z = 0;
    CK(cudaMemcpyToSymbol(g_gram_mma, &z, sizeof(int)));
  }
  if (getenv("CBIE_ONESIDED_JACOBI")) {   // experiment knob (slower on configs 2 and 4: 4.7 sweeps)
    const int z = 1;
    CK(cudaMemcpyToSymbol(g_gram_onesided, &z, sizeof(int)));
  }
  if (getenv("CBIE_JACOBI_T")) {   // experiment knob: threads of the two-sided sweeps
    const int jt = std::max(32, std::min(NT, atoi(getenv("CBIE_JACOBI_T")) / 32 * 32));
    CK(cudaMemcpyToSymbol(g_jacobi_threads, &jt, sizeof(int)));
  }
  for (int b0 = 0; b0 < nd; b0 += wave) {
    const int nb = std::min(wave, nd - b0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nb * csize));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_trunc_gram, arena, aout, ranks, idx ? d_desc : d_desc + b0, scratch.p, per, tol,
                          overflow, prof, defer, b0, idx, mn_max));
    CKL();
  }
}
#endif  // T2_GRAM

}  // namespace T2NS
}  // namespace

