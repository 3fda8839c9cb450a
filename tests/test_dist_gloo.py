"""Multi-process (world_size 2, gloo) checks of the N > 1 host logic on CPU:
max-over-ranks timing, whole-job throughput aggregation, and the leaf-sharded
fill's ownership (cbie_partition_lpt, shard.cu) plus its owner-major exchange plan
(every owner broadcasts one contiguous range; all ranks end with every leaf)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 100.0 + 50.0 * rank
    t = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, float(t.item()), bench._dist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_max_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [o[1] for o in out] == [150.0, 150.0]
    assert out[0][2] == (0, 2, 0) and out[1][2][:2] == (1, 2)
    # whole-job value = ranks * N / max time
    N = 12288
    assert 2 * N / (150.0 / 1e3) == pytest.approx(163840.0)


def _leaf_costs(seed=5, n_dense=1272, n_lr=2008):
    """Config-2-like leaf population: 192^2 dense leaves, 192^2 / 384^2 admissible ones
    (the cost model of shard.cu: m n for dense, 3 min(budget, 24) (m + n) otherwise)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    m = rng.choice([192, 384], size=n_lr, p=[0.8, 0.2])
    cost = np.concatenate([np.full(n_dense, 192.0 * 192.0), 3.0 * np.minimum(m // 2, 24) * (2.0 * m)])
    return cost[rng.permutation(cost.size)]


def _leaf_shapes(seed=5, n_dense=1272, n_lr=2008):
    """Config-2-like leaf population: 192^2 dense leaves, 192^2 / 384^2 admissible ones."""
    import numpy as np
    rng = np.random.default_rng(seed)
    m = np.concatenate([np.full(n_dense, 192), rng.choice([192, 384], size=n_lr, p=[0.8, 0.2])])
    adm = np.concatenate([np.zeros(n_dense, np.uint8), np.ones(n_lr, np.uint8)])
    perm = rng.permutation(m.size)
    return m[perm].astype(np.int32), m[perm].astype(np.int32), adm[perm]


def _shard_worker(rank, world, port, q):
    """The exchange of csrc/shard.cu with gloo standing in for NCCL: the LPT partition
    (cbie_partition_lpt) and the post-fill layout (cbie_shard_layout_host, the same
    function shard_exchange calls) come from the library; the all-reduce of the
    (rank, demoted) pairs and the per-owner broadcasts of the dense range and the tail
    are the same collectives, issued through torch.distributed."""
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_17116_b200 import dist as cdist
    m, n, adm = _leaf_shapes()
    nleaf = m.size
    cap = np.minimum(np.minimum(m, n) // 2, 24)
    cost = np.where(adm == 1, 3.0 * cap * (m + n), m.astype(float) * n)   # shard.cu cost model
    owner = cdist.partition_lpt(cost, world)          # computed independently per rank
    allo = [torch.zeros(nleaf, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(allo, torch.from_numpy(owner.astype(np.int32)))
    same = all(torch.equal(allo[0], a) for a in allo)
    # local fill: every owned admissible leaf gets a rank (a deterministic function of the
    # leaf, as the ACA would give on any rank), one in 50 is demoted
    rk = (np.arange(nleaf) * 7919 % 23 + 1).astype(np.int32)
    dem = (np.arange(nleaf) % 50 == 3) & (adm == 1)
    info = np.zeros(2 * nleaf, np.int32)
    mine = owner == rank
    info[0::2] = np.where(mine & (adm == 1) & ~dem, rk, 0)
    info[1::2] = np.where(mine & dem, 1, 0)
    t = torch.from_numpy(info.copy())
    dist.all_reduce(t)                                # ncclAllReduce(sum) in shard.cu
    info = t.numpy()
    off, ranges, total = cdist.shard_layout(m, n, adm, owner, info, world)
    # arena: every entry of a leaf holds the leaf index (dense / demoted: m n entries;
    # low rank: U m r then V n r); this rank writes only its own leaves
    arena = torch.full((total,), -1.0, dtype=torch.float64)
    for li in np.flatnonzero(mine):
        if off[li, 0] >= 0:
            arena[off[li, 0]:off[li, 0] + m[li] * n[li]] = float(li)
        elif info[2 * li] > 0:
            r = info[2 * li]
            arena[off[li, 1]:off[li, 1] + m[li] * r] = float(li)
            arena[off[li, 2]:off[li, 2] + n[li] * r] = float(li)
    for o in range(world):                            # grouped ncclBroadcast in shard.cu
        for lo, hi in ((ranges[o, 0], ranges[o, 1]), (ranges[o, 2], ranges[o, 3])):
            if hi > lo:
                seg = arena[lo:hi].clone()
                dist.broadcast(seg, src=o)
                arena[lo:hi] = seg
    a = arena.numpy()
    ok = True
    covered = 0
    for li in range(nleaf):
        if off[li, 0] >= 0:
            sl = a[off[li, 0]:off[li, 0] + m[li] * n[li]]
        else:
            r = info[2 * li]
            sl = np.concatenate([a[off[li, 1]:off[li, 1] + m[li] * r], a[off[li, 2]:off[li, 2] + n[li] * r]])
        ok &= bool(np.all(sl == li))
        covered += sl.size
    spans = sum(int(ranges[o, 1] - ranges[o, 0] + ranges[o, 3] - ranges[o, 2]) for o in range(world))
    loads = [float(cost[owner == o].sum()) for o in range(world)]
    q.put((rank, same, ok, loads, bool(np.all(a >= 0)) and spans == total, float(cost.max())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_leaf_sharding_and_exchange_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, same, ok, loads, dense_cover, cmax in out:
        assert same and ok and dense_cover
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(loads) / 2 + cmax
        assert max(loads) / min(loads) < 1.01


def test_lpt_partition_covers_every_leaf_once():
    import numpy as np
    from paper_2408_17116_b200 import dist as cdist
    cost = _leaf_costs()
    for world in (1, 2, 4, 8):
        owner = cdist.partition_lpt(cost, world)
        assert owner.min() >= 0 and owner.max() < world
        loads = np.bincount(owner, weights=cost, minlength=world)
        assert loads.max() <= cost.sum() / world + cost.max()
        assert np.array_equal(owner, cdist.partition_lpt(cost, world))   # deterministic


def _sphere_points(n=864, seed=3):
    import numpy as np
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((n, 3))
    return p / np.linalg.norm(p, axis=1)[:, None]


def _hlu_plan_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_17116_b200 import dist as cdist
    st, owner = cdist.hlu_dist_plan(_sphere_points(), 2, 64, 1.0, world)
    # every rank derives the same plan from the same structure (no negotiation needed)
    t = torch.tensor(owner.astype(np.int64))
    ts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(ts, t)
    same = all(torch.equal(ts[0], x) for x in ts)
    q.put((rank, st, owner.tolist(), same))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_distributed_hlu_plan():
    """Block-row-distributed H-LU plan (hlu_dist.cuh) on 2 gloo ranks, host only: both
    ranks derive the identical leaf ownership, every rank owns leaves and tasks,
    no buffer has two writer ranks, and factored blocks cross ranks between levels."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_hlu_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (_, st0, own0, same0), (_, st1, own1, same1) = out
    assert same0 and same1 and own0 == own1 and st0 == st1
    assert st0["conflicts"] == 0
    assert set(own0) == {0, 1}
    assert st0["tasks_min"] > 0 and st0["messages"] > 0 and st0["xfer_elems"] > 0
    assert st0["final_elems"] > 0


def test_distributed_hlu_plan_world_sizes():
    """World 1 needs no transfers; more ranks spread the tasks (max share shrinks)."""
    from paper_2408_17116_b200 import dist as cdist
    pts = _sphere_points()
    s1, o1 = cdist.hlu_dist_plan(pts, 2, 64, 1.0, 1)
    assert s1["messages"] == 0 and s1["xfer_elems"] == 0 and set(o1.tolist()) == {0}
    s4, o4 = cdist.hlu_dist_plan(pts, 2, 64, 1.0, 4)
    assert set(o4.tolist()) == {0, 1, 2, 3}
    assert s4["tasks"] == s1["tasks"]                     # same tape, split over ranks
    assert s4["tasks_max"] < s1["tasks_max"]
    assert s4["conflicts"] == 0
