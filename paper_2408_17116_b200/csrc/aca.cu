// aca.cu — K5: batched partially pivoted ACA with on-the-fly rows/columns, and
// the H-matrix build driver (cluster tree -> block tree -> dense-leaf fill ->
// ACA -> recompression -> demotion) behind cbie_hmatrix_build.
//
// One CTA per admissible block runs the reference loop (hmatrix.py:352-409):
// row residual, pivot = argmax over unused columns (block reduction, first
// index on ties like np.argmax), column residual, incremental Frobenius
// estimate, budget check before the stop test, next row = argmax |u| over
// unused rows, zero-pivot skip to the first unused row.  Rows and columns come
// from entry_block() (near table or FAR kernel), scaled like
// EquilibratedGenerator (solver.py:119-125); no admissible block is ever
// materialised densely.
#include <algorithm>
#include <chrono>
#include <cstring>

#include "entry.cuh"
#include "hmatrix.h"
#include "lowrank.cuh"

namespace {

struct AcaDesc {
  int r_lo, r_hi, c_lo, c_hi;   // point ranges (permuted order)
  int m, n, budget, kmax;       // kmax + 1 slots are allocated
  int64_t off_u, off_v;         // scratch: U m x (kmax+1), Vt n x (kmax+1)
  int k_slot;                   // ranks[k_slot] <- accepted rank
};

struct ArgMax {
  double v;
  int i;
};
__device__ __forceinline__ ArgMax amax(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ ArgMax warp_amax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = amax(a, b);
  }
  return a;
}
__device__ ArgMax block_amax(ArgMax a, ArgMax* red) {
  a = warp_amax(a);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = a;
  __syncthreads();
  ArgMax t = red[0];
  for (int i = 1; i < LR_NW; ++i) t = amax(t, red[i]);
  return t;
}

// status: 0 converged, 1 rank over budget (demote), 2 scratch capacity too small
template <int C>
__global__ void __launch_bounds__(LR_NT) k_aca(const __grid_constant__ Tables t, Geom g,
                                               const __grid_constant__ Phys ph, NearTab nt,
                                               const AcaDesc* __restrict__ descs,
                                               const int32_t* __restrict__ pperm, zc* arena,
                                               int* ranks, double tol, int* status) {
  const AcaDesc d = descs[blockIdx.x];
  const int m = d.m, n = d.n, ncp = d.c_hi - d.c_lo, nrp = d.r_hi - d.r_lo;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zc* s_co = reinterpret_cast<zc*>(smem_raw);        // [kmax+1] U[i,l] or V[l,j]
  zc* s_du = s_co + (d.kmax + 1);                     // [kmax+1] <u_l, u>
  zc* s_dv = s_du + (d.kmax + 1);                     // [kmax+1] v . conj(v_l)
  uint8_t* urow = reinterpret_cast<uint8_t*>(s_dv + (d.kmax + 1));
  uint8_t* ucol = urow + m;
  __shared__ double red[LR_NW];
  __shared__ ArgMax ared[LR_NW];
  __shared__ int s_i, s_state;

  zc* U = arena + d.off_u;   // column l: U + l*m
  zc* V = arena + d.off_v;   // row l:    V + l*n   (Vt column-major)
  for (int i = threadIdx.x; i < m; i += LR_NT) urow[i] = 0;
  for (int j = threadIdx.x; j < n; j += LR_NT) ucol[j] = 0;
  double f2 = 0.0;   // thread 0 only
  int k = 0, st = 0;
  if (threadIdx.x == 0) s_i = 0;
  __syncthreads();
  while (true) {
    const int i = s_i;
    // ---- row residual into V[k, :] ----
    for (int l = threadIdx.x; l < k; l += LR_NT) s_co[l] = U[(int64_t)l * m + i];
    __syncthreads();
    const int pa = pperm[d.r_lo + i / C], b = i % C;
    ArgMax best{-1.0, 0x7fffffff};
    for (int cb = threadIdx.x; cb < ncp; cb += LR_NT) {
      zc blk[C][C];
      entry_block<C>(t, g, ph, nt, pa, pperm[d.c_lo + cb], blk);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int j = cb * C + c;
        zc v = zmul(blk[b][c], zmul(ph.rsc[b], ph.csc[c]));
        for (int l = 0; l < k; ++l) v = zsub(v, zmul(s_co[l], V[(int64_t)l * n + j]));
        V[(int64_t)k * n + j] = v;
        if (!ucol[j]) best = amax(best, ArgMax{hypot(v.x, v.y), j});
      }
    }
    best = block_amax(best, ared);
    if (threadIdx.x == 0) urow[i] = 1;
    if (best.i == 0x7fffffff) break;   // every column used
    const int jstar = best.i;
    const zc piv = V[(int64_t)k * n + jstar];
    __syncthreads();
    if (hypot(piv.x, piv.y) < 1e-300) {   // zero pivot: first unused row (hmatrix.py:379-384)
      if (threadIdx.x == 0) {
        int nxt = -1;
        for (int r = 0; r < m; ++r)
          if (!urow[r]) {
            nxt = r;
            break;
          }
        s_state = nxt;
        if (nxt >= 0) s_i = nxt;
      }
      __syncthreads();
      if (s_state < 0) break;
      continue;
    }
    for (int j = threadIdx.x; j < n; j += LR_NT) V[(int64_t)k * n + j] = zdiv(V[(int64_t)k * n + j], piv);
    for (int l = threadIdx.x; l < k; l += LR_NT) s_co[l] = V[(int64_t)l * n + jstar];
    __syncthreads();
    // ---- column residual into U[:, k] ----
    {
      const int pj = pperm[d.c_lo + jstar / C], c = jstar % C;
      for (int ra = threadIdx.x; ra < nrp; ra += LR_NT) {
        zc blk[C][C];
        entry_block<C>(t, g, ph, nt, pperm[d.r_lo + ra], pj, blk);
#pragma unroll
        for (int bb = 0; bb < C; ++bb) {
          const int ii = ra * C + bb;
          zc v = zmul(blk[bb][c], zmul(ph.rsc[bb], ph.csc[c]));
          for (int l = 0; l < k; ++l) v = zsub(v, zmul(s_co[l], U[(int64_t)l * m + ii]));
          U[(int64_t)k * m + ii] = v;
        }
      }
    }
    if (threadIdx.x == 0) ucol[jstar] = 1;
    __syncthreads();
    // ---- Frobenius estimate (hmatrix.py:391-393) ----
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const zc* u = U + (int64_t)k * m;
    const zc* v = V + (int64_t)k * n;
    for (int l = w; l < k; l += LR_NW) {
      const zc* ul = U + (int64_t)l * m;
      const zc* vl = V + (int64_t)l * n;
      zc a = zmk(0.0, 0.0), bsum = zmk(0.0, 0.0);
      for (int ii = lane; ii < m; ii += 32) a = zadd(a, zcmul(ul[ii], u[ii]));
      for (int j = lane; j < n; j += 32) bsum = zadd(bsum, zmulc(v[j], vl[j]));
      a = warp_sum(a);
      bsum = warp_sum(bsum);
      if (lane == 0) {
        s_du[l] = a;
        s_dv[l] = bsum;
      }
    }
    double su = 0.0, sv = 0.0;
    for (int ii = threadIdx.x; ii < m; ii += LR_NT) su += zabs2(u[ii]);
    su = block_sum(su, red);
    for (int j = threadIdx.x; j < n; j += LR_NT) sv += zabs2(v[j]);
    sv = block_sum(sv, red);
    const double nu = sqrt(su), nv = sqrt(sv);
    if (threadIdx.x == 0) {
      zc cross = zmk(0.0, 0.0);
      for (int l = 0; l < k; ++l) cross = zadd(cross, zmul(s_du[l], s_dv[l]));
      f2 += 2.0 * cross.x + (nu * nv) * (nu * nv);
      int state = 0;
      if (k + 1 > d.budget) state = 1;                 // RankOverflow -> demote
      else if (k + 1 > d.kmax) state = 2;              // scratch capacity: retry larger
      else if (nu * nv <= tol * sqrt(fmax(f2, 0.0))) state = 3;   // converged
      s_state = state;
      if (state == 0) {
        ArgMax bb{-1.0, 0x7fffffff};
        (void)bb;
      }
    }
    __syncthreads();
    const int state = s_state;
    if (state == 1 || state == 2) {
      st = state;
      break;
    }
    ++k;
    if (state == 3) break;
    // ---- next row: argmax |u| over unused rows ----
    ArgMax rb{-1.0, 0x7fffffff};
    for (int ii = threadIdx.x; ii < m; ii += LR_NT)
      if (!urow[ii]) rb = amax(rb, ArgMax{hypot(u[ii].x, u[ii].y), ii});
    rb = block_amax(rb, ared);
    if (rb.i == 0x7fffffff) break;   // every row used
    if (threadIdx.x == 0) s_i = rb.i;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    status[blockIdx.x] = st;
    ranks[d.k_slot] = k;
  }
}

// contribution of one leaf to y = H x (permuted order): ypart = leaf * x[cols]
__global__ void k_leaf_apply(const LeafInfo* __restrict__ lv, const int64_t* __restrict__ ypart_off,
                             const int* __restrict__ ranks, const zc* __restrict__ arena,
                             const zc* __restrict__ x, int nrhs, int64_t N, const int32_t* rowoff,
                             const int32_t* coloff, zc* ypart, zc* tmp, int64_t tmp_per) {
  const LeafInfo L = lv[blockIdx.x];
  const int m = L.m, n = L.n;
  const int64_t c0 = coloff[blockIdx.x];
  zc* yp = ypart + ypart_off[blockIdx.x];
  for (int rhs = 0; rhs < nrhs; ++rhs) {
    const zc* xs = x + (int64_t)rhs * N + c0;
    zc* y = yp + (int64_t)rhs * m;
    if (L.kind == BLK_DENSE) {
      const zc* D = arena + L.off_d;
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        zc s = zmk(0.0, 0.0);
        for (int j = 0; j < n; ++j) zfma(s, D[(int64_t)j * m + i], xs[j]);
        y[i] = s;
      }
    } else {
      const int r = ranks[blockIdx.x];
      const zc* Uu = arena + L.off_u;
      const zc* Vt = arena + L.off_v;
      zc* w = tmp + (int64_t)blockIdx.x * tmp_per;
      for (int l = threadIdx.x; l < r; l += blockDim.x) {
        zc s = zmk(0.0, 0.0);
        for (int j = 0; j < n; ++j) zfma(s, Vt[(int64_t)l * n + j], xs[j]);
        w[l] = s;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        zc s = zmk(0.0, 0.0);
        for (int l = 0; l < r; ++l) zfma(s, Uu[(int64_t)l * m + i], w[l]);
        y[i] = s;
      }
      __syncthreads();
    }
  }
  (void)rowoff;
}

// deterministic gather: y[i] = sum over the leaves covering row i, in leaf order
__global__ void k_gather_rows(const int32_t* __restrict__ rptr, const int64_t* __restrict__ rsrc,
                              const zc* __restrict__ ypart, int64_t N, int nrhs,
                              const int64_t* __restrict__ ypart_stride, zc* y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  for (int rhs = 0; rhs < nrhs; ++rhs) {
    zc s = zmk(0.0, 0.0);
    for (int e = rptr[i]; e < rptr[i + 1]; ++e) {
      const int64_t src = rsrc[e];   // offset of (leaf part, row) for rhs 0
      s = zadd(s, ypart[src + (int64_t)rhs * ypart_stride[e]]);
    }
    y[(int64_t)rhs * N + i] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// segment gather (staging -> arena)
// ---------------------------------------------------------------------------
__global__ void k_copy_segments(const CopySeg* __restrict__ segs, const zc* __restrict__ src,
                                zc* __restrict__ dst) {
  const CopySeg g = segs[blockIdx.x];
  for (int64_t e = threadIdx.x; e < g.count; e += blockDim.x) dst[g.dst + e] = src[g.src + e];
}

void launch_copy_segments(const std::vector<CopySeg>& segs, const zc* src, zc* dst, cudaStream_t s) {
  if (segs.empty()) return;
  DBuf<CopySeg> d;
  d.upload(segs, s);
  for (size_t b0 = 0; b0 < segs.size(); b0 += 65535) {
    const int nb = (int)std::min<size_t>(65535, segs.size() - b0);
    k_copy_segments<<<nb, 256, 0, s>>>(d.p + b0, src, dst);
    CKL();
  }
  CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// build driver
// ---------------------------------------------------------------------------
static int aca_budget(int m, int n) { return std::max(1, std::min(m, n) / 2); }

static void launch_aca(cbie_hmat* H, const std::vector<AcaDesc>& descs, zc* arena, int* d_status) {
  cbie_ctx* c = H->ctx;
  if (descs.empty()) return;
  cudaStream_t s = c->stream;
  DBuf<AcaDesc> dd;
  dd.upload(descs, s);
  int maxk = 0, maxmn = 0;
  for (auto& d : descs) {
    maxk = std::max(maxk, d.kmax);
    maxmn = std::max(maxmn, d.m + d.n);
  }
  size_t smem = 3 * sizeof(zc) * (maxk + 1) + maxmn;
  smem = (smem + 15) & ~size_t(15);
  if (c->C == 2) {
    CK(cudaFuncSetAttribute(k_aca<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_aca<2><<<(unsigned)descs.size(), LR_NT, smem, s>>>(c->tab, c->geom(), c->ph, c->near(), dd.p,
                                                          H->d_pperm.p, arena, H->rank.p, H->tol,
                                                          d_status);
  } else {
    CK(cudaFuncSetAttribute(k_aca<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_aca<4><<<(unsigned)descs.size(), LR_NT, smem, s>>>(c->tab, c->geom(), c->ph, c->near(), dd.p,
                                                          H->d_pperm.p, arena, H->rank.p, H->tol,
                                                          d_status);
  }
  CKL();
  CK(cudaStreamSynchronize(s));
}

void hlu_trim_cache(bool force);

static void hmatrix_build(cbie_hmat* H, int n_leaf) {
  cbie_ctx* c = H->ctx;
  hlu_trim_cache(false);
  cudaStream_t s = c->stream;
  Tree& T = H->tree;
  auto t0 = std::chrono::steady_clock::now();
  T.build_clusters(c->h_pos.data(), c->npts, c->C, n_leaf);
  T.build_blocks(H->eta);
  auto t1 = std::chrono::steady_clock::now();
  H->stat["tree_ms"] = std::chrono::duration<double, std::milli>(t1 - t0).count();
  H->N = c->N;
  const int nleaf = (int)T.leaves.size();
  // ---- storage: dense leaves first (m x n each); low-rank leaves are appended
  // wave by wave with their EXACT ranks (U m x r, Vt n x r), so the arena holds
  // sum (m+n) r instead of (m+n) * budget (config 5: ~20 GB instead of ~1.5 TB) ----
  // leaf ownership (single process: every leaf local); dense storage owner-major so
  // each process's dense leaves are one contiguous range (shard exchange)
  shard_assign(H);
  int64_t used = 0;
  for (int o = 0; o < H->shard_world; ++o)
    for (int li = 0; li < nleaf; ++li) {
      auto& L = T.leaves[li];
      if (L.kind == BLK_DENSE && (H->owner.empty() || H->owner[li] == o)) {
        L.off_d = used;
        used += (int64_t)L.m * L.n;
      }
    }
  // low-rank region: the capacity bound sum (m+n) min(budget, 128) when it fits in
  // half of the free HBM, else half of the free HBM (grown on demand, rarely)
  int64_t lr_bound = 0;
  for (auto& L : T.leaves)
    if (L.kind == BLK_LR) lr_bound += (int64_t)(L.m + L.n) * std::min(aca_budget(L.m, L.n), 128);
  {
    size_t fr = 0, tot = 0;
    fr = mem_free_bytes(&tot);
    const int64_t avail = (int64_t)(0.5 * ((double)fr - (double)used * sizeof(zc))) / (int64_t)sizeof(zc);
    const int64_t lr_alloc = std::max<int64_t>(std::min(lr_bound, avail), 1 << 20);
    H->arena.alloc(std::max<int64_t>(used + lr_alloc, 1));
  }
  std::vector<int> aca_leaf;
  for (int li = 0; li < nleaf; ++li)
    if (T.leaves[li].kind == BLK_LR) {
      if (H->owns(li)) {
        aca_leaf.push_back(li);
      } else {   // filled by another process
        T.leaves[li].cap = 1;
        T.leaves[li].off_u = T.leaves[li].off_v = -1;
      }
    }
  const int nadm = (int)aca_leaf.size();
  H->rank.alloc(nleaf + nadm + 1);
  CK(cudaMemsetAsync(H->rank.p, 0, sizeof(int) * H->rank.n, s));
  H->d_pperm.upload(T.pperm, s);
  EvTimer tm;
  tm.start(s);
  // ---- dense leaves ----
  std::vector<TileDesc> tiles;
  for (int li = 0; li < nleaf; ++li) {
    const auto& L = T.leaves[li];
    if (L.kind == BLK_DENSE && H->owns(li)) {
      const Cluster &R = T.cl[L.r], &Cc = T.cl[L.c];
      tiles.push_back(TileDesc{L.off_d, R.lo, R.hi, Cc.lo, Cc.hi});
    }
  }
  DBuf<TileDesc> dt;
  dt.upload(tiles, s);
  launch_fill_tiles(c, dt.p, (int)tiles.size(), H->d_pperm.p, H->arena.p, 1, s);
  const double dense_ms = tm.stop_ms(s);
  auto grow = [&](int64_t need) {
    if (need <= (int64_t)H->arena.n) return;
    DBuf<zc> bigger;
    bigger.alloc(std::max<int64_t>(need, (int64_t)H->arena.n + ((int64_t)1 << 28)));
    CK(cudaMemcpyAsync(bigger.p, H->arena.p, sizeof(zc) * used, cudaMemcpyDeviceToDevice, s));
    std::swap(bigger.p, H->arena.p);
    std::swap(bigger.n, H->arena.n);
  };
  // ---- admissible leaves in waves: ACA -> recompression -> exact-rank append ----
  const int KCAP = 128;
  const int64_t wave_elems =
      (int64_t)((getenv("CBIE_ACA_WAVE_GB") ? atof(getenv("CBIE_ACA_WAVE_GB")) : 8.0) *
                (double)(1ll << 30)) / (int64_t)sizeof(zc);
  DBuf<zc> scratch, staging;
  TruncWork tscratch;
  DBuf<int> d_status;
  DBuf<unsigned long long> ovf;
  ovf.alloc(1);
  CK(cudaMemsetAsync(ovf.p, 0, 8, s));
  double aca_ms = 0, trunc_ms = 0, demote_ms = 0;
  int demoted = 0, retries = 0, waves = 0;
  for (int w0 = 0; w0 < nadm;) {
    // wave: consecutive admissible leaves whose ACA scratch fits
    std::vector<AcaDesc> aca;
    int64_t soff = 0;
    int w1 = w0;
    for (; w1 < nadm; ++w1) {
      const auto& L = T.leaves[aca_leaf[w1]];
      const int budget = aca_budget(L.m, L.n);
      const int kmax = std::min(budget, KCAP);
      const int64_t need = (int64_t)(L.m + L.n) * (kmax + 1);
      if (w1 > w0 && soff + need > wave_elems) break;
      AcaDesc d;
      const Cluster &R = T.cl[L.r], &Cc = T.cl[L.c];
      d.r_lo = R.lo;
      d.r_hi = R.hi;
      d.c_lo = Cc.lo;
      d.c_hi = Cc.hi;
      d.m = L.m;
      d.n = L.n;
      d.budget = budget;
      d.kmax = kmax;
      d.off_u = soff;
      soff += (int64_t)L.m * (kmax + 1);
      d.off_v = soff;
      soff += (int64_t)L.n * (kmax + 1);
      d.k_slot = nleaf + w1;
      aca.push_back(d);
    }
    ++waves;
    EvTimer tw;
    tw.start(s);
    if ((int64_t)scratch.n < soff) scratch.alloc(soff);
    d_status.alloc(std::max<size_t>(aca.size(), 1));
    launch_aca(H, aca, scratch.p, d_status.p);
    std::vector<int> status(aca.size());
    CK(cudaMemcpy(status.data(), d_status.p, sizeof(int) * aca.size(), cudaMemcpyDeviceToHost));
    // capacity misses: rerun with twice the capacity (up to the budget) until every
    // block converged or overflowed its budget (the reference ACA has no capacity)
    int64_t roff = soff;
    for (int round = 0; round < 16; ++round) {
      std::vector<AcaDesc> retry;
      std::vector<int> retry_idx;
      int64_t base = roff;
      for (size_t a = 0; a < aca.size(); ++a)
        if (status[a] == 2) {
          AcaDesc d = aca[a];
          d.kmax = std::min(d.budget, 2 * d.kmax);
          d.off_u = roff;
          roff += (int64_t)d.m * (d.kmax + 1);
          d.off_v = roff;
          roff += (int64_t)d.n * (d.kmax + 1);
          aca[a] = d;
          retry.push_back(d);
          retry_idx.push_back((int)a);
        }
      if (retry.empty()) break;
      (void)base;
      DBuf<zc> bigger;
      bigger.alloc(roff);
      CK(cudaMemcpyAsync(bigger.p, scratch.p, sizeof(zc) * std::min<int64_t>(scratch.n, roff),
                         cudaMemcpyDeviceToDevice, s));
      std::swap(bigger.p, scratch.p);
      std::swap(bigger.n, scratch.n);
      DBuf<int> st2;
      st2.alloc(retry.size());
      launch_aca(H, retry, scratch.p, st2.p);
      std::vector<int> s2(retry.size());
      CK(cudaMemcpy(s2.data(), st2.p, sizeof(int) * retry.size(), cudaMemcpyDeviceToHost));
      for (size_t q = 0; q < retry.size(); ++q) status[retry_idx[q]] = s2[q];
      retries += (int)retry.size();
    }
    aca_ms += tw.stop_ms(s);
    // recompression into staging (capacity = the block's ACA capacity: r <= k)
    tw.start(s);
    std::vector<TruncDesc> td;
    std::vector<int> td_block;
    int64_t stoff = 0;
    int kmax_t = 1, kcm = 1, mnm = 1;
    for (size_t a = 0; a < aca.size(); ++a) {
      if (status[a] != 0) continue;
      const auto& d = aca[a];
      TruncDesc t;
      t.in_u = d.off_u;
      t.in_v = d.off_v;
      t.ldu = d.m;
      t.ldv = d.n;
      t.skip_slot = -1;
      t.m = d.m;
      t.n = d.n;
      t.k = 0;
      t.k_slot = d.k_slot;
      t.cap = std::min(d.kmax + 1, std::min(d.m, d.n));
      t.out_u = stoff;
      stoff += (int64_t)d.m * t.cap;
      t.out_v = stoff;
      stoff += (int64_t)d.n * t.cap;
      t.out_slot = aca_leaf[w0 + a];
      td.push_back(t);
      td_block.push_back((int)a);
      kmax_t = std::max(kmax_t, std::min(d.kmax + 1, std::max(d.m, d.n)));
      kcm = std::max(kcm, d.kmax + 1);
      mnm = std::max(mnm, std::max(d.m, d.n));
    }
    kmax_t = std::min(kmax_t, 384);
    if ((int64_t)staging.n < stoff) staging.alloc(std::max<int64_t>(stoff, 1));
    DBuf<TruncDesc> dtd;
    dtd.upload(td, s);
    // factor-form recompression: Gram path (multi-stage up to rank 256) at tol >= 1e-5,
    // like the H-LU (lowrank.cu launch_truncate_routed); Householder kernels otherwise
    if (H->tol >= 1e-5 && getenv("CBIE_NO_GRAM") == nullptr)
      launch_truncate_routed(scratch.p, H->rank.p, dtd.p, (int)td.size(), kmax_t, H->tol, ovf.p, tscratch, s, kcm,
                             mnm, nullptr, nullptr, staging.p);
    else
      launch_truncate(scratch.p, H->rank.p, dtd.p, (int)td.size(), kmax_t, H->tol, ovf.p, tscratch, s,
                      kcm, mnm, staging.p, TRUNC_NO_DENSE);
    std::vector<int> rk(nleaf);
    CK(cudaStreamSynchronize(s));   // ranks come from the (non-blocking) library stream
    CK(cudaMemcpy(rk.data(), H->rank.p, sizeof(int) * nleaf, cudaMemcpyDeviceToHost));
    // exact-rank append
    std::vector<CopySeg> segs;
    int64_t need = used;
    for (size_t q = 0; q < td.size(); ++q) {
      const int li = td[q].out_slot;
      need += (int64_t)(td[q].m + td[q].n) * std::max(rk[li], 1);
    }
    grow(need);
    for (size_t q = 0; q < td.size(); ++q) {
      const int li = td[q].out_slot;
      auto& L = T.leaves[li];
      const int r = rk[li];
      L.cap = std::max(r, 1);
      L.off_u = used;
      used += (int64_t)L.m * L.cap;
      L.off_v = used;
      used += (int64_t)L.n * L.cap;
      if (r > 0) {
        segs.push_back(CopySeg{td[q].out_u, L.off_u, (int64_t)L.m * r});
        segs.push_back(CopySeg{td[q].out_v, L.off_v, (int64_t)L.n * r});
      }
    }
    launch_copy_segments(segs, staging.p, H->arena.p, s);
    trunc_ms += tw.stop_ms(s);
    // demotion: RankOverflow -> dense leaf (hmatrix.py:259-263)
    std::vector<TileDesc> dtl;
    for (size_t a = 0; a < aca.size(); ++a)
      if (status[a] == 1) {
        auto& L = T.leaves[aca_leaf[w0 + a]];
        L.kind = BLK_DENSE;
        T.nodes[L.node].kind = BLK_DENSE;
        L.cap = 0;
        grow(used + (int64_t)L.m * L.n);
        L.off_d = used;
        used += (int64_t)L.m * L.n;
        const Cluster &R = T.cl[L.r], &Cc = T.cl[L.c];
        dtl.push_back(TileDesc{L.off_d, R.lo, R.hi, Cc.lo, Cc.hi});
      }
    if (!dtl.empty()) {
      tw.start(s);
      DBuf<TileDesc> dd;
      dd.upload(dtl, s);
      launch_fill_tiles(c, dd.p, (int)dtl.size(), H->d_pperm.p, H->arena.p, 1, s);
      demote_ms += tw.stop_ms(s);
      demoted += (int)dtl.size();
    }
    w0 = w1;
  }
  H->demoted = demoted;
  H->stat["aca_retries"] = retries;
  H->stat["aca_waves"] = waves;
  unsigned long long hovf = 0;
  CK(cudaMemcpy(&hovf, ovf.p, 8, cudaMemcpyDeviceToHost));
  H->overflow = (int64_t)hovf;
  H->h_rank.resize(nleaf);
  CK(cudaMemcpy(H->h_rank.data(), H->rank.p, sizeof(int) * nleaf, cudaMemcpyDeviceToHost));
  H->partial = H->shard_world > 1;
  int64_t stored = 0;
  for (int li = 0; li < nleaf; ++li) {
    auto& L = T.leaves[li];
    if (!H->owns(li)) continue;
    stored += L.kind == BLK_DENSE ? (int64_t)L.m * L.n : (int64_t)H->h_rank[li] * (L.m + L.n);
  }
  H->stat["arena_used"] = (double)used;
  H->stat["dense_fill_ms"] = dense_ms;
  H->stat["aca_ms"] = aca_ms;
  H->stat["recompress_ms"] = trunc_ms;
  H->stat["demote_fill_ms"] = demote_ms;
  H->stat["fill_ms"] = dense_ms + aca_ms + trunc_ms + demote_ms;
  H->stat["n_leaves"] = nleaf;
  H->stat["n_local_leaves"] = (double)(tiles.size() + aca_leaf.size());
  H->stat["n_dense"] = (double)tiles.size() + demoted;
  H->stat["n_lowrank"] = (double)(nadm - demoted);
  H->stat["demoted"] = (double)demoted;
  H->stat["trunc_overflow"] = (double)hovf;
  H->stat["stored_scalars"] = (double)stored;
  H->stat["compression_rate"] = 1.0 - (double)stored / ((double)H->N * (double)H->N);
  H->stat["arena_bytes"] = (double)used * sizeof(zc);
}

void hmatrix_build_entry(cbie_hmat* H, int n_leaf) { hmatrix_build(H, n_leaf); }

// ---------------------------------------------------------------------------
// matvec (HMatrix.matvec, hmatrix.py:267-274), deterministic
// ---------------------------------------------------------------------------
void hmat_apply(cbie_hmat* H, const zc* d_xp, zc* d_yp, int nrhs, cudaStream_t s);

// gather plan of the H-matvec for one nrhs: leaf partial products, then every row
// sums its contributions in leaf order (deterministic); built once per H-matrix
struct MatvecPlan {
  int nrhs = 0, nleaf = 0, maxr = 1;
  DBuf<LeafInfo> dl;
  DBuf<int64_t> dpo, drs, dst;
  DBuf<int32_t> dco, dro, drp;
  DBuf<zc> part, tmp;
};

void hmat_apply(cbie_hmat* H, const zc* d_xp, zc* d_yp, int nrhs, cudaStream_t s) {
  Tree& T = H->tree;
  const int nleaf = (int)T.leaves.size();
  const int64_t N = H->N;
  auto* MP = static_cast<MatvecPlan*>(H->mv_plan.get());
  if (!MP || MP->nrhs != nrhs) {
    auto mp = std::make_shared<MatvecPlan>();
    const int C = T.C;
    std::vector<int64_t> poff(nleaf);
    std::vector<int32_t> coloff(nleaf), rowoff(nleaf);
    int64_t tot = 0;
    int maxr = 1;
    for (int li = 0; li < nleaf; ++li) {
      poff[li] = tot;
      tot += (int64_t)T.leaves[li].m * nrhs;
      coloff[li] = T.cl[T.leaves[li].c].lo * C;
      rowoff[li] = T.cl[T.leaves[li].r].lo * C;
      maxr = std::max(maxr, T.leaves[li].cap);
    }
    // row -> contributing (leaf, local row) in leaf order
    std::vector<std::vector<std::pair<int64_t, int64_t>>> rows(N);
    std::vector<int32_t> rptr(N + 1, 0);
    std::vector<int64_t> rsrc, rstride;
    for (int li = 0; li < nleaf; ++li) {
      const auto& L = T.leaves[li];
      for (int i = 0; i < L.m; ++i) rows[rowoff[li] + i].push_back({poff[li] + i, L.m});
    }
    for (int64_t i = 0; i < N; ++i) {
      rptr[i + 1] = rptr[i] + (int32_t)rows[i].size();
      for (auto& pr : rows[i]) {
        rsrc.push_back(pr.first);
        rstride.push_back(pr.second);
      }
    }
    mp->nrhs = nrhs;
    mp->nleaf = nleaf;
    mp->maxr = maxr;
    mp->dl.upload(T.leaves, s);
    mp->dpo.upload(poff, s);
    mp->drs.upload(rsrc, s);
    mp->dst.upload(rstride, s);
    mp->dco.upload(coloff, s);
    mp->dro.upload(rowoff, s);
    mp->drp.upload(rptr, s);
    mp->part.alloc(std::max<int64_t>(tot, 1));
    mp->tmp.alloc((size_t)nleaf * maxr);
    H->mv_plan = mp;
    MP = mp.get();
  }
  k_leaf_apply<<<nleaf, 128, 0, s>>>(MP->dl.p, MP->dpo.p, H->rank.p, H->arena.p, d_xp, nrhs, N, MP->dro.p,
                                     MP->dco.p, MP->part.p, MP->tmp.p, MP->maxr);
  CKL();
  k_gather_rows<<<ceil_div(N, 128), 128, 0, s>>>(MP->drp.p, MP->drs.p, MP->part.p, N, nrhs, MP->dst.p, d_yp);
  CKL();
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
std::string stats_to_json(const std::map<std::string, double>& m);

extern "C" {

int cbie_hmatrix_build(cbie_ctx* c, int n_leaf, double eta, double aca_tol, cbie_hmat** out) {
  cbie_hmat* H = nullptr;
  try {
    cudaSetDevice(c->device);
    c->require(c->has_class, "classify first");
    if (!(aca_tol > 0.0 && aca_tol < 1.0)) throw cbie_error(CBIE_EINVALID, "aca_tol in (0,1)");
    H = new cbie_hmat();
    H->ctx = c;
    H->eta = eta;
    H->tol = aca_tol;
    hmatrix_build(H, n_leaf);
    *out = H;
  } catch (const cbie_error& e) {
    c->err = e.what();
    delete H;
    *out = nullptr;
    return e.code;
  }
  return CBIE_OK;
}

void cbie_hmatrix_destroy(cbie_hmat* h) { delete h; }

// leaf data to pinned host memory, mapped into the device address space (see cbie_hmat::pinned)
int cbie_hmatrix_offload(cbie_hmat* h) {
  try {
    cudaSetDevice(h->ctx->device);
    if (h->pinned) return CBIE_OK;
    const size_t n = h->arena.n;
    zc* host = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&host), sizeof(zc) * std::max<size_t>(n, 1), cudaHostAllocMapped));
    CK(cudaMemcpy(host, h->arena.p, sizeof(zc) * n, cudaMemcpyDeviceToHost));
    zc* dev = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
    h->arena.release();
    h->arena.p = dev;
    h->arena.n = n;
    h->arena.borrowed = true;
    h->pinned = host;
    h->stat["offloaded_bytes"] = (double)n * sizeof(zc);
  } catch (const cbie_error& e) {
    h->ctx->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}

int cbie_hmatrix_tree(cbie_hmat* h, int64_t* dof_perm, int64_t* leaves, int64_t* nleaf) {
  const Tree& T = h->tree;
  if (nleaf) *nleaf = (int64_t)T.leaves.size();
  if (dof_perm)
    for (size_t p = 0; p < T.pperm.size(); ++p)
      for (int c = 0; c < T.C; ++c) dof_perm[p * T.C + c] = (int64_t)T.pperm[p] * T.C + c;
  if (leaves)
    for (size_t li = 0; li < T.leaves.size(); ++li) {
      const auto& L = T.leaves[li];
      int64_t* o = leaves + 6 * li;
      o[0] = T.cl[L.r].lo;
      o[1] = T.cl[L.r].hi;
      o[2] = T.cl[L.c].lo;
      o[3] = T.cl[L.c].hi;
      o[4] = L.kind == BLK_LR ? 1 : 0;
      o[5] = L.kind == BLK_LR ? h->h_rank[li] : 0;
    }
  return CBIE_OK;
}

int cbie_hmatrix_leaf(cbie_hmat* h, int64_t leaf, int* kind, int* rank, cbie_c128* D_or_U,
                      cbie_c128* V) {
  try {
    const Tree& T = h->tree;
    if (leaf < 0 || leaf >= (int64_t)T.leaves.size()) throw cbie_error(CBIE_EINVALID, "leaf index");
    const auto& L = T.leaves[leaf];
    cudaSetDevice(h->ctx->device);
    if (h->partial && !h->owns((int)leaf)) {   // filled by another shard, not exchanged yet
      *kind = -1;
      *rank = 0;
      return CBIE_OK;
    }
    *kind = L.kind == BLK_LR ? 1 : 0;
    const int m = L.m, n = L.n;
    if (L.kind == BLK_DENSE) {
      *rank = 0;
      if (D_or_U) {
        std::vector<zc> cm((size_t)m * n);
        CK(cudaMemcpy(cm.data(), h->arena.p + L.off_d, sizeof(zc) * cm.size(), cudaMemcpyDeviceToHost));
        zc* o = reinterpret_cast<zc*>(D_or_U);
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < n; ++j) o[(size_t)i * n + j] = cm[(size_t)j * m + i];
      }
    } else {
      int r = 0;
      CK(cudaMemcpy(&r, h->rank.p + leaf, sizeof(int), cudaMemcpyDeviceToHost));
      *rank = r;
      if (D_or_U && r) {
        std::vector<zc> cu((size_t)m * r), cv((size_t)n * r);
        CK(cudaMemcpy(cu.data(), h->arena.p + L.off_u, sizeof(zc) * cu.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cv.data(), h->arena.p + L.off_v, sizeof(zc) * cv.size(), cudaMemcpyDeviceToHost));
        zc* ou = reinterpret_cast<zc*>(D_or_U);
        zc* ov = reinterpret_cast<zc*>(V);
        for (int i = 0; i < m; ++i)
          for (int l = 0; l < r; ++l) ou[(size_t)i * r + l] = cu[(size_t)l * m + i];
        for (int l = 0; l < r; ++l)
          for (int j = 0; j < n; ++j) ov[(size_t)l * n + j] = cv[(size_t)l * n + j];
      }
    }
  } catch (const cbie_error& e) {
    h->ctx->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}

int cbie_hmatvec(cbie_hmat* h, const cbie_c128* x, cbie_c128* y, int nrhs) {
  try {
    cudaSetDevice(h->ctx->device);
    if (h->partial) throw cbie_error(CBIE_ESTATE, "partial (sharded) H-matrix: exchange the shards first");
    cudaStream_t s = h->ctx->stream;
    const int64_t N = h->N;
    const int C = h->tree.C;
    // permute into tree order, column-major [nrhs][N]
    std::vector<zc> xp((size_t)N * nrhs), yp((size_t)N * nrhs);
    const zc* xx = reinterpret_cast<const zc*>(x);
    for (size_t p = 0; p < h->tree.pperm.size(); ++p)
      for (int c = 0; c < C; ++c) {
        const int64_t newi = (int64_t)p * C + c, oldi = (int64_t)h->tree.pperm[p] * C + c;
        for (int r = 0; r < nrhs; ++r) xp[(size_t)r * N + newi] = xx[(size_t)oldi * nrhs + r];
      }
    DBuf<zc> dx, dy;
    dx.upload(xp, s);
    dy.alloc((size_t)N * nrhs);
    hmat_apply(h, dx.p, dy.p, nrhs, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(yp.data(), dy.p, sizeof(zc) * yp.size(), cudaMemcpyDeviceToHost));
    zc* yy = reinterpret_cast<zc*>(y);
    for (size_t p = 0; p < h->tree.pperm.size(); ++p)
      for (int c = 0; c < C; ++c) {
        const int64_t newi = (int64_t)p * C + c, oldi = (int64_t)h->tree.pperm[p] * C + c;
        for (int r = 0; r < nrhs; ++r) yy[(size_t)oldi * nrhs + r] = yp[(size_t)r * N + newi];
      }
  } catch (const cbie_error& e) {
    h->ctx->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}

}  // extern "C"

std::string hmat_stats(const cbie_hmat* h) { return stats_to_json(h->stat); }
