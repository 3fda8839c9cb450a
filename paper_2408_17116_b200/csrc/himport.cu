// himport.cu — an H-matrix from host-evaluated leaves: the generator protocol of the
// reference's HMatrix.fill (hmatrix.py:207-264) with an arbitrary host generator (the
// reference's own tests drive hlu_factor with KernelGen / IdGen / ZeroGen,
// tests/test_hmatrix.py:9-36, 216-280).  The host evaluates each leaf's block through
// the generator; the device stores dense leaves and compresses admissible ones by the
// truncated SVD of the block (dense-mode recompression, lowrank.cu; keep s > tol s_0),
// demoting a block whose rank exceeds the ACA budget min(m, n) / 2 (hmatrix.py:259-263).
// The result is an ordinary cbie_hmat: cbie_hlu_factor / solve / hmatvec take it.
#include <algorithm>
#include <vector>

#include "hmatrix.h"

namespace {
int budget_of(int m, int n) { return std::max(1, std::min(m, n) / 2); }
}  // namespace

extern "C" {

int cbie_hmatrix_layout(const double* pts, int64_t npts, int C, int n_leaf, double eta, int64_t* dof_perm,
                        int64_t* leaves, int64_t* nleaf) {
  try {
    if (npts < 1 || C < 1 || n_leaf < 1) throw cbie_error(CBIE_EINVALID, "npts, C, n_leaf >= 1");
    Tree T;
    T.build_clusters(pts, (int)npts, C, n_leaf);
    T.build_blocks(eta);
    if (nleaf) *nleaf = (int64_t)T.leaves.size();
    if (dof_perm)
      for (size_t p = 0; p < T.pperm.size(); ++p)
        for (int c = 0; c < C; ++c) dof_perm[p * C + c] = (int64_t)T.pperm[p] * C + c;
    if (leaves)
      for (size_t li = 0; li < T.leaves.size(); ++li) {
        const auto& L = T.leaves[li];
        int64_t* o = leaves + 5 * li;
        o[0] = T.cl[L.r].lo;
        o[1] = T.cl[L.r].hi;
        o[2] = T.cl[L.c].lo;
        o[3] = T.cl[L.c].hi;
        o[4] = L.kind == BLK_LR ? 1 : 0;
      }
  } catch (const cbie_error& e) {
    return e.code;
  } catch (const std::exception&) {
    return CBIE_EINVALID;
  }
  return CBIE_OK;
}

int cbie_hmatrix_import(cbie_ctx* c, const double* pts, int64_t npts, int C, int n_leaf, double eta, double tol,
                        const cbie_c128* data, cbie_hmat** out) {
  cbie_hmat* H = nullptr;
  try {
    cudaSetDevice(c->device);
    if (!(tol > 0.0 && tol < 1.0)) throw cbie_error(CBIE_EINVALID, "tol in (0,1)");
    H = new cbie_hmat();
    H->ctx = c;
    H->eta = eta;
    H->tol = tol;
    Tree& T = H->tree;
    T.build_clusters(pts, (int)npts, C, n_leaf);
    T.build_blocks(eta);
    H->N = npts * C;
    cudaStream_t s = c->stream;
    const int nleaf = (int)T.leaves.size();
    const zc* src = reinterpret_cast<const zc*>(data);
    // host: leaf blocks (row-major, leaf order) -> column-major; dense leaves to the
    // arena, admissible ones to the recompression scratch
    std::vector<int64_t> soff(nleaf);
    int64_t dense_n = 0, adm_n = 0, pos = 0;
    for (int li = 0; li < nleaf; ++li) {
      auto& L = T.leaves[li];
      soff[li] = pos;
      pos += (int64_t)L.m * L.n;
      if (L.kind == BLK_DENSE) dense_n += (int64_t)L.m * L.n;
      else adm_n += (int64_t)L.m * L.n;
    }
    std::vector<zc> hd((size_t)std::max<int64_t>(dense_n, 1)), ha((size_t)std::max<int64_t>(adm_n, 1));
    std::vector<TruncDesc> td;
    int64_t d_used = 0, a_used = 0, st_used = 0;
    int kc = 1, mn = 1;
    for (int li = 0; li < nleaf; ++li) {
      auto& L = T.leaves[li];
      const zc* b = src + soff[li];
      zc* dst = L.kind == BLK_DENSE ? hd.data() + d_used : ha.data() + a_used;
      for (int i = 0; i < L.m; ++i)
        for (int j = 0; j < L.n; ++j) dst[(size_t)j * L.m + i] = b[(size_t)i * L.n + j];
      if (L.kind == BLK_DENSE) {
        L.off_d = d_used;
        d_used += (int64_t)L.m * L.n;
      } else {
        TruncDesc t{};
        t.in_u = a_used;
        t.in_v = -1;
        t.ldu = L.m;
        t.ldv = L.n;
        t.skip_slot = -1;
        t.m = L.m;
        t.n = L.n;
        t.k = L.n;
        t.k_slot = -1;
        t.cap = std::min(L.m, L.n);
        t.out_u = st_used;
        st_used += (int64_t)L.m * t.cap;
        t.out_v = st_used;
        st_used += (int64_t)L.n * t.cap;
        t.out_slot = li;
        td.push_back(t);
        a_used += (int64_t)L.m * L.n;
        kc = std::max(kc, L.n);
        mn = std::max(mn, std::max(L.m, L.n));
      }
    }
    H->rank.alloc(nleaf + 1);
    CK(cudaMemsetAsync(H->rank.p, 0, sizeof(int) * H->rank.n, s));
    std::vector<int> rk(nleaf, 0);
    DBuf<zc> scratch, staging;
    if (!td.empty()) {
      scratch.upload(ha, s);
      staging.alloc((size_t)std::max<int64_t>(st_used, 1));
      DBuf<TruncDesc> dtd;
      dtd.upload(td, s);
      DBuf<unsigned long long> ovf;
      ovf.alloc(1);
      CK(cudaMemsetAsync(ovf.p, 0, 8, s));
      TruncWork work;
      launch_truncate(scratch.p, H->rank.p, dtd.p, (int)td.size(), std::max(kc, mn), tol, ovf.p, work, s, kc, mn,
                      staging.p, 0);
      CK(cudaStreamSynchronize(s));
      CK(cudaMemcpy(rk.data(), H->rank.p, sizeof(int) * nleaf, cudaMemcpyDeviceToHost));
    }
    // demotion (rank above the ACA budget -> dense leaf), then the arena: dense leaves,
    // demoted leaves, low-rank leaves with their exact ranks
    int demoted = 0;
    std::vector<CopySeg> from_scratch, from_staging;
    int64_t used = d_used;
    for (const auto& t : td) {
      auto& L = T.leaves[t.out_slot];
      if (rk[t.out_slot] > budget_of(L.m, L.n)) {
        L.kind = BLK_DENSE;
        T.nodes[L.node].kind = BLK_DENSE;
        L.cap = 0;
        L.off_d = used;
        from_scratch.push_back(CopySeg{t.in_u, used, (int64_t)L.m * L.n});   // src: offset in ha
        used += (int64_t)L.m * L.n;
        rk[t.out_slot] = 0;
        ++demoted;
      }
    }
    for (const auto& t : td) {
      auto& L = T.leaves[t.out_slot];
      if (L.kind != BLK_LR) continue;
      const int r = rk[t.out_slot];
      L.cap = std::max(r, 1);
      L.off_u = used;
      used += (int64_t)L.m * L.cap;
      L.off_v = used;
      used += (int64_t)L.n * L.cap;
      if (r > 0) {
        from_staging.push_back(CopySeg{t.out_u, L.off_u, (int64_t)L.m * r});
        from_staging.push_back(CopySeg{t.out_v, L.off_v, (int64_t)L.n * r});
      }
    }
    H->arena.alloc((size_t)std::max<int64_t>(used, 1));
    if (d_used) CK(cudaMemcpyAsync(H->arena.p, hd.data(), sizeof(zc) * d_used, cudaMemcpyHostToDevice, s));
    // demoted leaves from the host copy (the recompression used its inputs as workspace)
    for (const auto& g : from_scratch)
      CK(cudaMemcpyAsync(H->arena.p + g.dst, ha.data() + g.src, sizeof(zc) * g.count, cudaMemcpyHostToDevice, s));
    if (!from_staging.empty()) launch_copy_segments(from_staging, staging.p, H->arena.p, s);
    CK(cudaMemcpyAsync(H->rank.p, rk.data(), sizeof(int) * nleaf, cudaMemcpyHostToDevice, s));
    H->d_pperm.upload(T.pperm, s);
    CK(cudaStreamSynchronize(s));
    H->h_rank = rk;
    H->demoted = demoted;
    int64_t stored = 0;
    for (int li = 0; li < nleaf; ++li) {
      const auto& L = T.leaves[li];
      stored += L.kind == BLK_DENSE ? (int64_t)L.m * L.n : (int64_t)rk[li] * (L.m + L.n);
    }
    H->stat["n_leaves"] = nleaf;
    H->stat["demoted"] = demoted;
    H->stat["stored_scalars"] = (double)stored;
    H->stat["compression_rate"] = 1.0 - (double)stored / ((double)H->N * (double)H->N);
    H->stat["arena_bytes"] = (double)used * sizeof(zc);
    H->stat["imported"] = 1;
    *out = H;
  } catch (const cbie_error& e) {
    c->err = e.what();
    delete H;
    *out = nullptr;
    return e.code;
  }
  return CBIE_OK;
}

}  // extern "C"
