// shard.cu — multi-GPU H-matrix fill: block-cluster-tree leaves are
// independent, so each process (one per GPU) fills only the leaves it owns and the
// shards are exchanged afterwards over NCCL (NVLink / NVSwitch on one node).
//
//   * ownership: LPT (longest processing time first) over an a-priori cost per leaf
//     -- dense leaf m n entries, admissible leaf ~3 k^ (m + n) generated entries with
//     k^ = min(budget, 24) -- identical on every rank (pure function of the tree);
//   * storage is owner-major: every process's dense leaves form one contiguous range
//     of the arena, and after the fill its low-rank / demoted leaves are laid out as
//     one contiguous tail (exact ranks, known after an NCCL all-reduce of the ranks);
//   * exchange: one in-place ncclBroadcast per owner for its dense range and one for
//     its tail, grouped (ncclGroupStart/End); every rank ends with the complete
//     H-matrix in the same layout, ready for the H-LU.
// No data-path collective during the fill itself.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include "hmatrix.h"

void launch_copy_segments(const std::vector<CopySeg>& segs, const zc* src, zc* dst, cudaStream_t s);

namespace {

struct NcclState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};
std::map<const cbie_ctx*, NcclState>& comms() {
  static std::map<const cbie_ctx*, NcclState> m;
  return m;
}

#define NCK(call)                                                                           \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess) throw cbie_error(CBIE_ENCCL, std::string("NCCL: ") + ncclGetErrorString(r_)); \
  } while (0)

int aca_budget_of(int m, int n) { return std::max(1, std::min(m, n) / 2); }

}  // namespace

// Global layout of the exchanged H-matrix (a pure function of the leaf shapes, the
// admissibility flags, the owners and the all-reduced (rank, demoted) pairs, so every
// rank computes the same one): dense leaves owner-major [dlo[o], dhi[o]) in leaf order,
// then each owner's tail [tlo[o], thi[o]) holding its demoted leaves (nd) and its
// low-rank leaves with their exact ranks (nu, nv; capacity max(r, 1)).
struct ShardLayout {
  std::vector<int64_t> dlo, dhi, tlo, thi, nu, nv, nd, dd;
  int64_t total = 0;
};
ShardLayout shard_layout(const int* m, const int* n, const uint8_t* adm, const int* owner, const int* info, int nleaf,
                         int W) {
  ShardLayout Y;
  Y.dlo.assign(W, 0);
  Y.dhi.assign(W, 0);
  Y.tlo.assign(W, 0);
  Y.thi.assign(W, 0);
  Y.nu.assign(nleaf, -1);
  Y.nv.assign(nleaf, -1);
  Y.nd.assign(nleaf, -1);
  Y.dd.assign(nleaf, -1);
  int64_t off = 0;
  for (int o = 0; o < W; ++o) {
    Y.dlo[o] = off;
    for (int li = 0; li < nleaf; ++li)
      if (!adm[li] && owner[li] == o) {
        Y.dd[li] = off;
        off += (int64_t)m[li] * n[li];
      }
    Y.dhi[o] = off;
  }
  for (int o = 0; o < W; ++o) {
    Y.tlo[o] = off;
    for (int li = 0; li < nleaf; ++li) {
      if (!adm[li] || owner[li] != o) continue;
      if (info[2 * li + 1]) {
        Y.nd[li] = off;
        off += (int64_t)m[li] * n[li];
      } else {
        const int cap = std::max(info[2 * li], 1);
        Y.nu[li] = off;
        off += (int64_t)m[li] * cap;
        Y.nv[li] = off;
        off += (int64_t)n[li] * cap;
      }
    }
    Y.thi[o] = off;
  }
  Y.total = off;
  return Y;
}

void shard_assign(cbie_hmat* H) {
  const Tree& T = H->tree;
  const int nleaf = (int)T.leaves.size();
  H->adm.assign(nleaf, 0);
  for (int li = 0; li < nleaf; ++li) H->adm[li] = T.leaves[li].kind == BLK_LR;
  if (H->shard_world <= 1) {
    H->owner.clear();
    return;
  }
  std::vector<double> cost(nleaf);
  for (int li = 0; li < nleaf; ++li) {
    const auto& L = T.leaves[li];
    cost[li] = L.kind == BLK_DENSE ? (double)L.m * L.n
                                   : 3.0 * std::min(aca_budget_of(L.m, L.n), 24) * (double)(L.m + L.n);
  }
  H->owner.assign(nleaf, 0);
  cbie_partition_lpt(cost.data(), nleaf, H->shard_world, H->owner.data());
}

void shard_exchange(cbie_hmat* H) {
  cbie_ctx* c = H->ctx;
  auto it = comms().find(c);
  if (it == comms().end() || !it->second.comm) throw cbie_error(CBIE_ESTATE, "cbie_dist_init first");
  NcclState& st = it->second;
  if (st.world != H->shard_world || st.rank != H->shard_rank)
    throw cbie_error(CBIE_EINVALID, "shard rank/world differ from the communicator's");
  cudaStream_t s = c->stream;
  Tree& T = H->tree;
  const int nleaf = (int)T.leaves.size();
  const int W = H->shard_world, me = H->shard_rank;
  auto t0 = std::chrono::steady_clock::now();
  EvTimer tm;
  tm.start(s);
  // a. ranks / demotion flags of every admissible leaf (owned entries, summed)
  std::vector<int> info(2 * (size_t)nleaf, 0);
  for (int li = 0; li < nleaf; ++li)
    if (H->adm[li] && H->owns(li)) {
      const bool dem = T.leaves[li].kind == BLK_DENSE;
      info[2 * li] = dem ? 0 : H->h_rank[li];
      info[2 * li + 1] = dem ? 1 : 0;
    }
  DBuf<int> dinfo;
  dinfo.upload(info, s);
  NCK(ncclAllReduce(dinfo.p, dinfo.p, info.size(), ncclInt32, ncclSum, st.comm, s));
  CK(cudaMemcpyAsync(info.data(), dinfo.p, sizeof(int) * info.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // b. global layout: dense ranges (unchanged, owner-major), then each owner's tail
  std::vector<int> lm(nleaf), ln(nleaf);
  for (int li = 0; li < nleaf; ++li) {
    lm[li] = T.leaves[li].m;
    ln[li] = T.leaves[li].n;
  }
  const ShardLayout Y = shard_layout(lm.data(), ln.data(), H->adm.data(), H->owner.data(), info.data(), nleaf, W);
  const auto &dlo = Y.dlo, &dhi = Y.dhi, &tlo = Y.tlo, &thi = Y.thi, &nu = Y.nu, &nv = Y.nv, &nd = Y.nd;
  const int64_t off = Y.total;
  // c. new arena with this rank's data in place
  DBuf<zc> na;
  na.alloc(std::max<int64_t>(off, 1));
  std::vector<CopySeg> segs;
  if (dhi[me] > dlo[me]) segs.push_back(CopySeg{dlo[me], dlo[me], dhi[me] - dlo[me]});
  for (int li = 0; li < nleaf; ++li) {
    if (!H->adm[li] || H->owner[li] != me) continue;
    const auto& L = T.leaves[li];
    if (info[2 * li + 1]) {
      segs.push_back(CopySeg{L.off_d, nd[li], (int64_t)L.m * L.n});
    } else if (info[2 * li] > 0) {
      const int r = info[2 * li];
      segs.push_back(CopySeg{L.off_u, nu[li], (int64_t)L.m * r});
      segs.push_back(CopySeg{L.off_v, nv[li], (int64_t)L.n * r});
    }
  }
  launch_copy_segments(segs, H->arena.p, na.p, s);
  // d. every owner broadcasts its dense range and its tail, in place
  NCK(ncclGroupStart());
  for (int o = 0; o < W; ++o) {
    if (dhi[o] > dlo[o])
      NCK(ncclBroadcast(na.p + dlo[o], na.p + dlo[o], 2 * (size_t)(dhi[o] - dlo[o]), ncclDouble, o, st.comm, s));
    if (thi[o] > tlo[o])
      NCK(ncclBroadcast(na.p + tlo[o], na.p + tlo[o], 2 * (size_t)(thi[o] - tlo[o]), ncclDouble, o, st.comm, s));
  }
  NCK(ncclGroupEnd());
  // e. descriptors, ranks, kinds
  int demoted = 0;
  std::vector<int> rk(H->rank.n, 0);
  for (int li = 0; li < nleaf; ++li) {
    auto& L = T.leaves[li];
    if (!H->adm[li]) continue;
    if (info[2 * li + 1]) {
      L.kind = BLK_DENSE;
      T.nodes[L.node].kind = BLK_DENSE;
      L.cap = 0;
      L.off_d = nd[li];
      L.off_u = L.off_v = -1;
      H->h_rank[li] = 0;
      ++demoted;
    } else {
      L.kind = BLK_LR;
      T.nodes[L.node].kind = BLK_LR;
      L.cap = std::max(info[2 * li], 1);
      L.off_u = nu[li];
      L.off_v = nv[li];
      H->h_rank[li] = info[2 * li];
      rk[li] = info[2 * li];
    }
  }
  CK(cudaMemcpyAsync(H->rank.p, rk.data(), sizeof(int) * rk.size(), cudaMemcpyHostToDevice, s));
  std::swap(H->arena.p, na.p);
  std::swap(H->arena.n, na.n);
  const double xms = tm.stop_ms(s);
  CK(cudaStreamSynchronize(s));
  H->partial = false;
  H->demoted = demoted;
  int64_t stored = 0;
  for (int li = 0; li < nleaf; ++li) {
    const auto& L = T.leaves[li];
    stored += L.kind == BLK_DENSE ? (int64_t)L.m * L.n : (int64_t)H->h_rank[li] * (L.m + L.n);
  }
  H->stat["exchange_ms"] = xms;
  H->stat["exchange_bytes"] = (double)off * sizeof(zc);
  H->stat["exchange_host_ms"] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  H->stat["demoted"] = demoted;
  H->stat["stored_scalars"] = (double)stored;
  H->stat["compression_rate"] = 1.0 - (double)stored / ((double)H->N * (double)H->N);
  H->stat["arena_bytes"] = (double)off * sizeof(zc);
}

std::string stats_to_json(const std::map<std::string, double>& m);
void hmatrix_build_entry(cbie_hmat* H, int n_leaf);

bool dist_comm_of(const cbie_ctx* c, ncclComm_t* comm, int* rank, int* world) {
  auto it = comms().find(c);
  if (it == comms().end() || !it->second.comm) return false;
  *comm = it->second.comm;
  *rank = it->second.rank;
  *world = it->second.world;
  return true;
}

extern "C" {

void cbie_partition_lpt(const double* cost, int64_t n, int world, int* owner) {
  std::vector<int64_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(std::max(world, 1), 0.0);
  for (int64_t i : ord) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    owner[i] = best;
    load[best] += cost[i];
  }
}

// host only: the exchange layout of shard.cu (shard_layout) for the gloo tests
//   leaf_off [nleaf][3]: dense offset (dense / demoted leaves), U offset, V offset (-1: none)
//   ranges   [world][4]: dense range lo, hi, tail lo, hi;  total: arena size (elements)
int cbie_shard_layout_host(int nleaf, const int* m, const int* n, const uint8_t* adm, const int* owner,
                           const int* info, int world, int64_t* leaf_off, int64_t* ranges, int64_t* total) {
  if (nleaf < 0 || world < 1) return CBIE_EINVALID;
  const ShardLayout Y = shard_layout(m, n, adm, owner, info, nleaf, world);
  for (int li = 0; li < nleaf; ++li) {
    leaf_off[3 * li] = Y.nd[li] >= 0 ? Y.nd[li] : Y.dd[li];
    leaf_off[3 * li + 1] = Y.nu[li];
    leaf_off[3 * li + 2] = Y.nv[li];
  }
  for (int o = 0; o < world; ++o) {
    ranges[4 * o] = Y.dlo[o];
    ranges[4 * o + 1] = Y.dhi[o];
    ranges[4 * o + 2] = Y.tlo[o];
    ranges[4 * o + 3] = Y.thi[o];
  }
  *total = Y.total;
  return CBIE_OK;
}

int cbie_nccl_unique_id(char* out, int cap) {
  if (cap < (int)sizeof(ncclUniqueId)) return CBIE_EINVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CBIE_ENCCL;
  memcpy(out, &id, sizeof(id));
  return CBIE_OK;
}

int cbie_dist_init(cbie_ctx* c, const char* id, int rank, int world) {
  try {
    cudaSetDevice(c->device);
    if (world < 1 || rank < 0 || rank >= world) throw cbie_error(CBIE_EINVALID, "rank / world");
    NcclState& st = comms()[c];
    if (st.comm) {
      ncclCommDestroy(st.comm);
      st.comm = nullptr;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    NCK(ncclCommInitRank(&st.comm, world, uid, rank));
    st.rank = rank;
    st.world = world;
  } catch (const cbie_error& e) {
    c->err = e.what();
    return e.code;
  }
  return CBIE_OK;
}

void cbie_dist_finalize(cbie_ctx* c) {
  auto it = comms().find(c);
  if (it == comms().end()) return;
  if (it->second.comm) ncclCommDestroy(it->second.comm);
  comms().erase(it);
}

int cbie_hmatrix_build_shard(cbie_ctx* c, int n_leaf, double eta, double aca_tol, int rank, int world,
                             int exchange, cbie_hmat** out) {
  cbie_hmat* H = nullptr;
  try {
    cudaSetDevice(c->device);
    c->require(c->has_class, "classify first");
    if (!(aca_tol > 0.0 && aca_tol < 1.0)) throw cbie_error(CBIE_EINVALID, "aca_tol in (0,1)");
    if (world < 1 || rank < 0 || rank >= world) throw cbie_error(CBIE_EINVALID, "rank / world");
    H = new cbie_hmat();
    H->ctx = c;
    H->eta = eta;
    H->tol = aca_tol;
    H->shard_rank = rank;
    H->shard_world = world;
    hmatrix_build_entry(H, n_leaf);
    if (exchange && world > 1) shard_exchange(H);
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
