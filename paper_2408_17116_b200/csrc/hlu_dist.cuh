// hlu_dist.cuh — block-row-distributed H-LU, included by hlu.cu.
//
// The reference factors on one core (hmatrix.py:827-858).  Here the recorded tape
// of that recursion (hlu.cu) is split over W processes, one per GPU:
//
//   * block rows: the clusters of the first tree level with >= 2 W clusters are
//     dealt cyclically to the ranks; a leaf belongs to the owner of its row cluster
//     (so the diagonal block of row k, its U panel and every Schur update into row i
//     run where those rows live, as in a block-row LU);
//   * every task that writes a leaf runs on the leaf's owner; a task that only
//     writes temporaries runs where its first consumer runs (reverse pass over the
//     tape), so product / concatenation temporaries never cross ranks;
//   * every rank records the same tape (same layout, same arena offsets), runs its
//     own tasks level-synchronously, and after level l sends the buffers another
//     rank reads at level l + 1: a snapshot of the whole buffer (factor leaves with
//     their rank slots and pivots -- the factored diagonal blocks and U panels of the
//     block-row scheme) taken at the latest level before the reader, which is exact
//     for the rectangle the reader touches (tape order + levels, see dist_plan);
//   * transfers are packed per (level, src, dst) into one staging message and moved
//     with ncclSend / ncclRecv (NVLink / NVSwitch) on the factorisation stream, so
//     the sender's later writes are ordered after the send;
//   * at the end every owner broadcasts its factored leaves (+ pivots, rcond): every
//     rank holds the complete factors, and the H-solve runs unchanged.
// cbie_hlu_factor_emulated runs the same plan with W virtual ranks in ONE process
// on one GPU (W arenas, sequential levels, device copies instead of NCCL): it checks
// that the ownership and transfer plan is complete without several GPUs.

bool dist_comm_of(const cbie_ctx* c, ncclComm_t* comm, int* rank, int* world);

namespace {

#define NCKH(call)                                                                                   \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess) throw cbie_error(CBIE_ENCCL, std::string("NCCL: ") + ncclGetErrorString(r_)); \
  } while (0)

// one contiguous piece of a transfer: 0 arena (complex), 1 rank slots, 2 pivots, 3 rcond
struct XSeg {
  int type;
  int64_t off, len, soff;
};

__global__ void k_xfer_pack(const XSeg* __restrict__ segs, zc* arena, int* ranks, int* piv, double* rcond,
                            zc* stage, int unpack) {
  const XSeg g = segs[blockIdx.x];
  for (int64_t i = threadIdx.x; i < g.len; i += blockDim.x) {
    zc* st = stage + g.soff + i;
    switch (g.type) {
      case 0:
        if (unpack) arena[g.off + i] = *st;
        else *st = arena[g.off + i];
        break;
      case 1:
        if (unpack) ranks[g.off + i] = (int)st->x;
        else *st = zmk((double)ranks[g.off + i], 0.0);
        break;
      case 2:
        if (unpack) piv[g.off + i] = (int)st->x;
        else *st = zmk((double)piv[g.off + i], 0.0);
        break;
      default:
        if (unpack) rcond[g.off + i] = st->x;
        else *st = zmk(rcond[g.off + i], 0.0);
        break;
    }
  }
}

struct Msg {
  int src = 0, dst = -1;   // dst -1: broadcast from src to every rank
  int64_t elems = 0;
  std::vector<XSeg> segs;
  std::shared_ptr<DBuf<XSeg>> dsegs = std::make_shared<DBuf<XSeg>>();
};

struct DistPlan {
  int W = 1, Ld = 0, max_level = 0;
  std::vector<int> leaf_owner, task_owner;
  std::map<int, std::vector<Msg>> after;   // messages sent after level l
  std::vector<Msg> final;                  // one broadcast per owner
  int64_t xfer_elems = 0, n_xfer = 0, n_msgs = 0, conflicts = 0;
  std::vector<int64_t> tasks_of;
};

// block rows: clusters of the first level with >= 2 W clusters (coarser leaf clusters
// included), in dof order, dealt cyclically; a leaf belongs to its row cluster's owner
void dist_owners(const Tree& T, int W, DistPlan& D) {
  int maxlv = 0;
  for (const auto& c : T.cl) maxlv = std::max(maxlv, c.level);
  std::vector<int> front;
  int d = 0;
  for (;; ++d) {
    front.clear();
    for (int i = 0; i < (int)T.cl.size(); ++i) {
      const Cluster& c = T.cl[i];
      if (c.level == d || (c.level < d && c.nkid == 0)) front.push_back(i);
    }
    if ((int)front.size() >= 2 * W || d >= maxlv) break;
  }
  D.Ld = d;
  std::sort(front.begin(), front.end(), [&](int a, int b) { return T.cl[a].lo < T.cl[b].lo; });
  int npt = 0;
  for (const auto& c : T.cl) npt = std::max(npt, c.hi);
  std::vector<int> pt_owner(npt, 0);
  for (size_t j = 0; j < front.size(); ++j)
    for (int p = T.cl[front[j]].lo; p < T.cl[front[j]].hi; ++p) pt_owner[p] = (int)(j % W);
  D.leaf_owner.resize(T.leaves.size());
  for (size_t li = 0; li < T.leaves.size(); ++li) D.leaf_owner[li] = pt_owner[T.cl[T.leaves[li].r].lo];
}

void add_buf_segs(const Recorder& R, const cbie_hlu& F, const std::vector<std::vector<int>>& slots_of, int b,
                  bool with_rcond, Msg& m) {
  const int nleaf = (int)F.tree.leaves.size();
  auto push = [&](int type, int64_t off, int64_t len) {
    if (len <= 0) return;
    m.segs.push_back(XSeg{type, off, len, m.elems});
    m.elems += len;
  };
  if (b < nleaf) {
    const LeafInfo& L = F.tree.leaves[b];
    if (L.kind == BLK_DENSE) {
      push(0, L.off_d, (int64_t)L.m * L.n);
      if (F.pivoff[b] >= 0) {
        push(2, F.pivoff[b], L.m);
        if (with_rcond) push(3, b, 1);
      }
    } else {
      push(0, L.off_u, (int64_t)(L.m + L.n) * L.cap);
    }
  } else {
    push(0, R.buf_off[b], R.buf_len[b]);
  }
  for (int sl : slots_of[b]) push(1, sl, 1);
}

void dist_plan(const Recorder& R, const cbie_hlu& F, int W, DistPlan& D, cudaStream_t s, bool upload = true) {
  const Tree& T = F.tree;
  const int nleaf = (int)T.leaves.size();
  const int nt = (int)R.tasks.size();
  D.W = W;
  dist_owners(T, W, D);
  auto acc_of = [&](int i, int j) { return R.acc_buf[R.acc_start[i] + j]; };
  auto nacc = [&](int i) { return (int)(R.acc_start[i + 1] - R.acc_start[i]); };
  // 1. task owners (reverse pass): leaf writers -> leaf owner; temp writers -> their first reader
  D.task_owner.assign(nt, 0);
  {
    std::vector<int> want(R.nbuf, -1);
    int ri = (int)R.reuse_at.size() - 1, next = 0;
    for (int i = nt - 1; i >= 0; --i) {
      int o = -1;
      for (int j = 0; j < nacc(i) && o < 0; ++j) {
        const int a = acc_of(i, j);
        if (a < 0 && ~a < nleaf) o = D.leaf_owner[~a];
      }
      for (int j = 0; j < nacc(i) && o < 0; ++j) {
        const int a = acc_of(i, j);
        if (a < 0 && want[~a] >= 0) o = want[~a];
      }
      if (o < 0) o = next;
      D.task_owner[i] = o;
      next = o;
      for (int j = 0; j < nacc(i); ++j) {
        const int a = acc_of(i, j);
        const int b = a >= 0 ? a : ~a;
        if (b >= nleaf) want[b] = o;
      }
      for (; ri >= 0 && R.reuse_at[ri].first == i; --ri) want[R.reuse_at[ri].second] = -1;
    }
  }
  D.tasks_of.assign(W, 0);
  for (int i = 0; i < nt; ++i) D.tasks_of[D.task_owner[i]]++;
  // 2. transfers (forward pass in tape order): a reader on rank o of a buffer last
  //    written on rank h != o needs a snapshot taken at a level t with
  //    (latest write of the buffer so far) <= t <= (reader level - 1)
  std::vector<std::vector<int>> slots_of(R.nbuf);
  for (size_t sl = 0; sl < R.slot_owner.size(); ++sl)
    if (R.slot_owner[sl] >= 0) slots_of[R.slot_owner[sl]].push_back((int)sl);
  std::vector<int> home(R.nbuf, -1), wmax(R.nbuf, -1);
  std::vector<int> sched((size_t)R.nbuf * W, -1);
  std::map<std::tuple<int, int, int>, std::vector<int>> want_x;   // (level, src, dst) -> buffers
  size_t ri = 0;
  for (int i = 0; i < nt; ++i) {
    for (; ri < R.reuse_at.size() && R.reuse_at[ri].first == i; ++ri) {
      const int b = R.reuse_at[ri].second;
      home[b] = -1;
      wmax[b] = -1;
      for (int q = 0; q < W; ++q) sched[(size_t)b * W + q] = -1;
    }
    const int o = D.task_owner[i], lv = R.tasks[i].level;
    D.max_level = std::max(D.max_level, lv);
    for (int j = 0; j < nacc(i); ++j) {
      const int a = acc_of(i, j);
      const int b = a >= 0 ? a : ~a;
      const int h = home[b];
      if (h < 0 || h == o) continue;
      int& t = sched[(size_t)b * W + o];
      if (!(t >= wmax[b] && t <= lv - 1) && t != lv - 1) {
        want_x[std::make_tuple(lv - 1, h, o)].push_back(b);
        t = lv - 1;
      }
      if (a < 0) ++D.conflicts;   // a second writer rank of one buffer generation
    }
    for (int j = 0; j < nacc(i); ++j) {
      const int a = acc_of(i, j);
      if (a >= 0) continue;
      home[~a] = o;
      wmax[~a] = std::max(wmax[~a], lv);
    }
  }
  if (D.conflicts)
    throw cbie_error(CBIE_EINVALID, "distributed H-LU: " + std::to_string(D.conflicts) +
                                        " buffers written by two ranks (ownership rule incomplete)");
  for (auto& kv : want_x) {
    Msg m;
    m.src = std::get<1>(kv.first);
    m.dst = std::get<2>(kv.first);
    std::vector<int> bs = kv.second;
    std::sort(bs.begin(), bs.end());
    bs.erase(std::unique(bs.begin(), bs.end()), bs.end());
    for (int b : bs) add_buf_segs(R, F, slots_of, b, false, m);
    D.xfer_elems += m.elems;
    D.n_xfer += (int64_t)bs.size();
    ++D.n_msgs;
    if (upload) m.dsegs->upload(m.segs, s);
    D.after[std::get<0>(kv.first)].push_back(std::move(m));
  }
  // 3. final: every owner broadcasts the leaves it wrote
  D.final.resize(W);
  for (int p = 0; p < W; ++p) D.final[p].src = p;
  for (int b = 0; b < nleaf; ++b)
    if (home[b] >= 0) add_buf_segs(R, F, slots_of, b, true, D.final[home[b]]);
  if (upload)
    for (auto& m : D.final) m.dsegs->upload(m.segs, s);
}

void xfer_pack(const Msg& m, zc* arena, int* ranks, int* piv, double* rcond, zc* stage, bool unpack,
               cudaStream_t s) {
  if (m.segs.empty()) return;
  k_xfer_pack<<<(unsigned)m.segs.size(), 256, 0, s>>>(m.dsegs->p, arena, ranks, piv, rcond, stage, unpack ? 1 : 0);
  CKL();
}

// per-rank device state of the factorisation
struct RankState {
  DBuf<zc> work;
  DBuf<int> ranks, piv, flag;
  DBuf<double> rcond;
  DBuf<unsigned long long> ovf;
  TruncWork tw[TW_PER_LANE * TRUNC_LANES];
  Plan plan;
};

void rank_state_init(RankState& S, const cbie_hlu& F, const Recorder& R, const std::vector<CopySeg>& segs,
                     int64_t leaf_end, const DistPlan& D, int me, cudaStream_t s) {
  const cbie_hmat* H = F.H;
  const int nleaf = (int)F.tree.leaves.size();
  S.work.alloc((size_t)(leaf_end + R.pool_top + 1));
  launch_copy_segments(segs, H->arena.p, S.work.p, s);
  std::vector<int> r0 = R.init_ranks;
  for (int li = 0; li < nleaf; ++li) r0[li] = H->h_rank[li];
  S.ranks.upload(r0, s);
  S.piv.alloc(std::max<int64_t>(F.npiv, 1));
  S.rcond.alloc(nleaf);
  CK(cudaMemsetAsync(S.rcond.p, 0, sizeof(double) * nleaf, s));
  S.flag.alloc(1);
  CK(cudaMemsetAsync(S.flag.p, 0, sizeof(int), s));
  S.ovf.alloc(1);
  CK(cudaMemsetAsync(S.ovf.p, 0, 8, s));
  make_plan(S.plan, s, &R, &D.task_owner, me);
}

void dist_finish(cbie_hlu* F, RankState& S, int64_t leaf_end, int hflag, unsigned long long hovf,
                 const DistPlan& D, cudaStream_t s) {
  const int nleaf = (int)F->tree.leaves.size();
  F->arena.alloc((size_t)leaf_end + 1);
  CK(cudaMemcpyAsync(F->arena.p, S.work.p, sizeof(zc) * leaf_end, cudaMemcpyDeviceToDevice, s));
  F->own();
  std::swap(F->ranks.p, S.ranks.p);
  std::swap(F->ranks.n, S.ranks.n);
  std::swap(F->piv.p, S.piv.p);
  std::swap(F->piv.n, S.piv.n);
  std::swap(F->rcond.p, S.rcond.p);
  std::swap(F->rcond.n, S.rcond.n);
  CK(cudaStreamSynchronize(s));
  F->leaf_end = leaf_end;
  F->stat["dist_world"] = D.W;
  F->stat["dist_row_level"] = D.Ld;
  F->stat["dist_levels"] = D.max_level;
  F->stat["dist_msgs"] = (double)D.n_msgs;
  F->stat["dist_xfer_buffers"] = (double)D.n_xfer;
  F->stat["dist_xfer_bytes"] = (double)D.xfer_elems * sizeof(zc);
  int64_t fb = 0;
  for (auto& m : D.final) fb += m.elems;
  F->stat["dist_final_bytes"] = (double)fb * sizeof(zc);
  int64_t tmin = INT64_MAX, tmax = 0;
  for (auto t : D.tasks_of) {
    tmin = std::min(tmin, t);
    tmax = std::max(tmax, t);
  }
  F->stat["dist_tasks_min"] = (double)tmin;
  F->stat["dist_tasks_max"] = (double)tmax;
  F->stat["trunc_overflow"] = (double)hovf;
  if (hflag) {
    std::vector<double> rc(nleaf);
    CK(cudaMemcpy(rc.data(), F->rcond.p, sizeof(double) * nleaf, cudaMemcpyDeviceToHost));
    double mn = 1e300;
    for (int li = 0; li < nleaf; ++li)
      if (F->pivoff[li] >= 0) mn = std::min(mn, rc[li]);
    throw cbie_error(CBIE_ESINGULAR_DIAGONAL, "diagonal block rcond " + std::to_string(mn));
  }
}

// W virtual ranks in this process (emulated == true) or rank `me` of the NCCL communicator
void hlu_factor_dist_impl(cbie_hlu* F, int W, bool emulated) {
  cbie_hmat* H = F->H;
  cudaStream_t s = H->ctx->stream;
  ncclComm_t comm = nullptr;
  int me = 0;
  if (!emulated) {
    int w = 0;
    if (!dist_comm_of(H->ctx, &comm, &me, &w)) throw cbie_error(CBIE_ESTATE, "cbie_dist_init first");
    W = w;
  }
  if (W < 1 || W > 64) throw cbie_error(CBIE_EINVALID, "distributed H-LU: world size in [1, 64]");
  std::vector<CopySeg> segs;
  const int64_t leaf_end = hlu_layout(F, segs);
  auto t0 = std::chrono::steady_clock::now();
  // identical tape on every rank: the temporary pool budget is the minimum over ranks
  int64_t budget = hlu_pool_budget(leaf_end, emulated ? W : 1);
  if (!emulated) {
    DBuf<int64_t> db;
    db.upload(std::vector<int64_t>{budget}, s);
    NCKH(ncclAllReduce(db.p, db.p, 1, ncclInt64, ncclMin, comm, s));
    CK(cudaMemcpyAsync(&budget, db.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  Recorder R;
  hlu_record(F, R, leaf_end, budget, true);
  DistPlan D;
  dist_plan(R, *F, W, D, s);
  F->stat["record_ms"] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  const int nv = emulated ? W : 1;   // rank states held by this process
  std::vector<RankState> S(nv);
  for (int v = 0; v < nv; ++v) rank_state_init(S[v], *F, R, segs, leaf_end, D, emulated ? v : me, s);
  int64_t maxmsg = 1;
  for (auto& kv : D.after)
    for (auto& m : kv.second) maxmsg = std::max(maxmsg, m.elems);
  for (auto& m : D.final) maxmsg = std::max(maxmsg, m.elems);
  CK(cudaStreamSynchronize(s));
  EvTimer tm;
  tm.start(s);
  // stage: emulated -- one message at a time; NCCL -- every message of a level this rank takes part in
  auto exchange = [&](const std::vector<Msg>& ms) {
    if (emulated) {
      DBuf<zc> st;
      st.alloc((size_t)maxmsg);
      for (const Msg& m : ms) {
        RankState& a = S[m.src];
        xfer_pack(m, a.work.p, a.ranks.p, a.piv.p, a.rcond.p, st.p, false, s);
        for (int v = 0; v < W; ++v) {
          if (v == m.src || (m.dst >= 0 && v != m.dst)) continue;
          RankState& b = S[v];
          xfer_pack(m, b.work.p, b.ranks.p, b.piv.p, b.rcond.p, st.p, true, s);
        }
      }
      return;
    }
    int64_t tot = 0;
    std::vector<int64_t> at(ms.size(), -1);
    for (size_t i = 0; i < ms.size(); ++i)
      if (ms[i].src == me || ms[i].dst == me || ms[i].dst < 0) {
        at[i] = tot;
        tot += ms[i].elems;
      }
    if (tot == 0) return;
    DBuf<zc> st;
    st.alloc((size_t)tot);
    RankState& a = S[0];
    for (size_t i = 0; i < ms.size(); ++i)
      if (at[i] >= 0 && ms[i].src == me) xfer_pack(ms[i], a.work.p, a.ranks.p, a.piv.p, a.rcond.p, st.p + at[i], false, s);
    NCKH(ncclGroupStart());
    for (size_t i = 0; i < ms.size(); ++i) {
      if (at[i] < 0 || ms[i].elems == 0) continue;
      const Msg& m = ms[i];
      if (m.dst < 0) {
        NCKH(ncclBroadcast(st.p + at[i], st.p + at[i], 2 * (size_t)m.elems, ncclDouble, m.src, comm, s));
      } else if (m.src == me) {
        NCKH(ncclSend(st.p + at[i], 2 * (size_t)m.elems, ncclDouble, m.dst, comm, s));
      } else {
        NCKH(ncclRecv(st.p + at[i], 2 * (size_t)m.elems, ncclDouble, m.src, comm, s));
      }
    }
    NCKH(ncclGroupEnd());
    for (size_t i = 0; i < ms.size(); ++i)
      if (at[i] >= 0 && ms[i].src != me) xfer_pack(ms[i], a.work.p, a.ranks.p, a.piv.p, a.rcond.p, st.p + at[i], true, s);
    CK(cudaStreamSynchronize(s));   // the staging buffer is released on return
  };
  for (int l = 0; l <= D.max_level; ++l) {
    if (l > 0)
      for (int v = 0; v < nv; ++v) {
        RankState& x = S[v];
        run_plan(x.plan, x.work.p, x.ranks.p, x.piv.p, x.rcond.p, x.flag.p, x.ovf.p, x.tw, F->tol, s, l, l);
      }
    auto it = D.after.find(l);
    if (it != D.after.end()) exchange(it->second);
  }
  exchange(D.final);
  F->stat["factor_device_ms"] = tm.stop_ms(s);
  // SingularDiagonal / clipped truncations from every rank
  int hflag = 0;
  unsigned long long hovf = 0;
  if (emulated) {
    for (int v = 0; v < nv; ++v) {
      int f = 0;
      unsigned long long o = 0;
      CK(cudaMemcpy(&f, S[v].flag.p, sizeof(int), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&o, S[v].ovf.p, 8, cudaMemcpyDeviceToHost));
      hflag |= f;
      hovf += o;
    }
  } else {
    NCKH(ncclAllReduce(S[0].flag.p, S[0].flag.p, 1, ncclInt32, ncclMax, comm, s));
    NCKH(ncclAllReduce(S[0].ovf.p, S[0].ovf.p, 1, ncclUint64, ncclSum, comm, s));
    CK(cudaMemcpyAsync(&hflag, S[0].flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hovf, S[0].ovf.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  F->stat["tasks"] = (double)R.tasks.size();
  dist_finish(F, S[0], leaf_end, hflag, hovf, D, s);
}

}  // namespace
