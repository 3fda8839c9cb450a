// hmatrix.h — host-side H-matrix structure (cluster tree, block tree, leaf
// storage descriptors) and the device-resident leaf data.
//
// Restates hmatrix.py:31-89 (ClusterTree, admissible), 96-204 (block kinds,
// block tree) with flat arrays so the device kernels can address leaves by index.
#pragma once
#include <algorithm>
#include <memory>
#include <vector>

#include "context.h"

struct Cluster {
  int lo = 0, hi = 0;          // point range in permuted order
  double blo[3], bhi[3];       // bounding box of the cluster's points
  int kid[2] = {-1, -1};
  int nkid = 0;
  int level = 0;
};

enum { BLK_H = 0, BLK_DENSE = 1, BLK_LR = 2 };

struct BNode {                 // block-tree node (hmatrix.py:146-162)
  int r = -1, c = -1;          // cluster ids
  int kind = BLK_H;
  int nr = 0, nc = 0;          // children grid nr x nc
  int kid[4] = {-1, -1, -1, -1};
  int leaf = -1;               // leaf index for DENSE / LR
};

struct LeafInfo {
  int node = -1;
  int r = -1, c = -1;          // clusters
  int m = 0, n = 0;            // rows / cols in dofs
  int kind = BLK_DENSE;        // BLK_DENSE or BLK_LR
  int cap = 0;                 // rank capacity (LR)
  int64_t off_d = -1;          // dense: column-major m x n at arena + off_d
  int64_t off_u = -1;          // LR: U m x cap col-major
  int64_t off_v = -1;          // LR: Vt n x cap col-major (Vt[l*n + j] = V[l][j])
};

struct Tree {
  int C = 2;
  std::vector<Cluster> cl;
  std::vector<int32_t> pperm;  // new -> old point index
  std::vector<BNode> nodes;
  std::vector<LeafInfo> leaves;
  int root_cl = 0, root_node = 0;
  void build_clusters(const double* pts, int npts, int C, int n_leaf);
  void build_blocks(double eta);
  int dofs(int cl_id) const { return (cl[cl_id].hi - cl[cl_id].lo) * C; }
};

struct cbie_hmat {
  cbie_ctx* ctx = nullptr;
  Tree tree;
  double eta = 1.0, tol = 1e-4;
  int64_t N = 0;
  DBuf<zc> arena;              // all leaf data
  DBuf<int> rank;              // [nleaf] device ranks (LR)
  std::vector<int> h_rank;     // host copy after fill
  DBuf<int32_t> d_pperm;
  int demoted = 0;
  int64_t overflow = 0;        // truncations clipped at capacity
  std::map<std::string, double> stat;
  // leaf sharding (shard.cu): this process fills the leaves with owner[li] == shard_rank
  int shard_rank = 0, shard_world = 1;
  std::vector<int> owner;      // [nleaf], empty = every leaf local
  std::vector<uint8_t> adm;    // [nleaf] admissible in the block tree (before demotion)
  bool partial = false;        // true until the shards were exchanged
  bool owns(int li) const { return owner.empty() || owner[li] == shard_rank; }
  std::shared_ptr<void> mv_plan;   // cached H-matvec gather plan (aca.cu hmat_apply)
  // cbie_hmatrix_offload: the leaf data moved to pinned host memory, mapped into the device
  // address space (arena.p is its device alias, arena.borrowed): kernels read it over the
  // host link, the device memory is free for the H-LU of problems too large for both
  zc* pinned = nullptr;
  ~cbie_hmat() {
    arena.release();
    if (pinned) cudaFreeHost(pinned);
  }
};

// shard.cu: LPT partition of the leaves over `world` processes by estimated fill cost
void shard_assign(cbie_hmat* H);
// shard.cu: exchange the shards over the context's NCCL communicator (every rank ends
// up with the complete H-matrix, same layout on all ranks)
void shard_exchange(cbie_hmat* H);

// lowrank.cu: batched truncation  (hmatrix.py:412-426, 605-609)
// inputs are col-major U (m x k) and Vt (n x k) = V^T; they are used as workspace.
// in_v < 0 means V = identity (n x n, k = n): truncated SVD of the dense U (m x n).
struct TruncDesc {
  int64_t in_u, in_v;          // arena offsets of the inputs
  int64_t out_u, out_v;        // arena offsets of the outputs (m x cap, n x cap)
  int ldu, ldv;                // leading dimensions of the inputs
  int skip_slot;               // >= 0 and ranks[skip_slot] == 0: no-op (adding rank 0)
  int m, n;
  int k;                       // static rank if k_slot < 0
  int k_slot;                  // >= 0: k = ranks[k_slot] (device-resident)
  int cap;                     // output capacity (columns)
  int out_slot;                // ranks[out_slot] <- r
  // Two-source form (in_u2 >= 0; Gram path only): the input is [piece 1 | sgn2 * piece 2]
  // read in place -- columns [0, k1) from in_u / in_v, columns [k1, k1 + k2) from in_u2 /
  // in_v2 -- instead of a materialised concatenation; k = k1 + k2 with k1 = ranks[k1_slot]
  // (k1 if the slot is < 0), k2 likewise.  The output may overwrite piece 1 (T += s U V^H).
  int64_t in_u2 = -1, in_v2 = -1;
  int ldu2 = 0, ldv2 = 0;
  int k1 = 0, k1_slot = -1, k2 = 0, k2_slot = -1;
  double sgn2 = 1.0;
};
// concatenated rank of a descriptor on the device
#ifdef __CUDACC__
__device__ __forceinline__ int trunc_k1(const TruncDesc& d, const int* ranks) {
  return d.k1_slot >= 0 ? ranks[d.k1_slot] : d.k1;
}
__device__ __forceinline__ int trunc_k(const TruncDesc& d, const int* ranks) {
  if (d.in_u2 >= 0) return trunc_k1(d, ranks) + (d.k2_slot >= 0 ? ranks[d.k2_slot] : d.k2);
  return d.k_slot >= 0 ? ranks[d.k_slot] : d.k;
}
#endif
// kmax >= every min(m,k), min(n,k) (dense mode: min(m,n) and n) in the batch
// kc_max / mn_max: largest concatenated capacity and max(m, n) (randomized-path scratch);
// arena_out (if non-null) receives the outputs (out_u / out_v offsets are relative to it)
// flags & TRUNC_NO_DENSE: the caller guarantees no dense-mode (in_v < 0) descriptor, so
// batches with mn_max <= 512 run the blocked kernel (trunc2.cu); problems whose device-side
// rank exceeds 128 are deferred by it to the unblocked kernel (second launch)
constexpr int TRUNC_NO_DENSE = 1;
// per-stream workspace of the recompression launches (kept across calls)
struct TruncWork {
  DBuf<zc> scratch;    // per-CTA scratch of the blocked / unblocked kernels
  DBuf<int> defer;     // problems the blocked kernel hands to the unblocked one
  DBuf<int> gdefer;    // problems the Gram kernel hands to the Householder kernels
  DBuf<zc> dscratch;   // scratch of the deferred launch
  void release() {
    scratch.release();
    defer.release();
    gdefer.release();
    dscratch.release();
  }
};
void launch_truncate(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, int kmax, double tol,
                     unsigned long long* overflow, TruncWork& work, cudaStream_t s,
                     int kc_max = 0, int mn_max = 0, zc* arena_out = nullptr, int flags = 0);
// factor-form problems only: Gram path for device-side ranks <= 64 (trunc2.cu), the
// others handed on to the blocked (k <= 128, max(m, n) <= 384) / unblocked kernels
// With a second stream / workspace the Householder share runs concurrently with the
// Gram kernel: a routing kernel splits the problems by their device-side rank first.
// big: descriptors [nsmall, nd) are large blocks (host-partitioned); their Gram-path
// problems run with clusters of cbig CTAs per problem on stream s3 (workspace work3),
// concurrently with the small ones (nsmall < 0: no split)
struct TruncBig {
  int nsmall = -1, cbig = 1, mn_small = 0;
  TruncWork* work3 = nullptr;
  cudaStream_t s3 = nullptr;
};
void launch_truncate_routed(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, int kmax, double tol,
                            unsigned long long* overflow, TruncWork& work, cudaStream_t s, int kc_max,
                            int mn_max, TruncWork* work2 = nullptr, cudaStream_t s2 = nullptr,
                            zc* arena_out = nullptr, const TruncBig* big = nullptr);
int truncate_gram_max_clusters(int csize);
void launch_truncate_gram(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, double tol,
                          unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, zc* arena_out,
                          int* defer, const int* idx = nullptr, int mn_multi = 0, int csize = 1);
bool launch_truncate_blocked(zc* arena, int* ranks, const TruncDesc* d_desc, int nd, double tol,
                             unsigned long long* overflow, DBuf<zc>& scratch, cudaStream_t s, int kc_max,
                             int mn_max, zc* arena_out, int* defer, const int* idx = nullptr);

// Per-launch workspace cap of the recompression kernels: `gb` GiB normally, 1 GiB in
// tight-memory mode (lean factor capacities, hlu.cu), so that the per-lane workspaces fit
// beside a factor arena that fills most of HBM (config 5).
extern bool g_ws_tight;
inline bool ws_tight() { return g_ws_tight; }
inline size_t ws_cap(int gb) { return (size_t)(g_ws_tight ? std::min(gb, 1) : gb) << 30; }

// contiguous segment copies src[src + i] -> dst[dst + i] (aca.cu)
struct CopySeg {
  int64_t src, dst, count;
};
void launch_copy_segments(const std::vector<CopySeg>& segs, const zc* src, zc* dst, cudaStream_t s);

// lowrank.cu: dense block -> (Q, B) by an adaptive randomized range finder
struct DenseLRDesc {
  int64_t p;                   // arena offset of P (col-major, ld)
  int64_t out_u, out_v;        // U m x cap, Vt n x cap
  int m, n, ld, cap;
  int out_slot;                // ranks[out_slot] <- l
  int l0;                      // initial sample size
  double tol;
};
void launch_dense_lr(zc* arena, int* ranks, const DenseLRDesc* d_desc, int nd, int max_m, int max_n,
                     int max_cap, DBuf<zc>& scratch, cudaStream_t s);
