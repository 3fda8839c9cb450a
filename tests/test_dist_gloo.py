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


def _shard_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_17116_b200 import dist as cdist
    cost = _leaf_costs()
    owner = cdist.partition_lpt(cost, world)          # computed independently per rank
    allo = [torch.zeros(cost.size, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(allo, torch.from_numpy(owner.astype(np.int32)))
    same = all(torch.equal(allo[0], a) for a in allo)
    # owner-major exchange plan: leaf data (here: its index repeated by size) packed in
    # owner order, each owner broadcasts its contiguous range
    size = (cost / cost.min()).round().astype(np.int64)
    order = np.concatenate([np.flatnonzero(owner == o) for o in range(world)])
    off = np.zeros(cost.size, np.int64)
    off[order] = np.concatenate([[0], np.cumsum(size[order])[:-1]])
    arena = torch.full((int(size.sum()),), -1.0, dtype=torch.float64)
    for li in np.flatnonzero(owner == rank):
        arena[off[li]:off[li] + size[li]] = float(li)
    lo = [int(off[owner == o].min()) for o in range(world)]
    hi = [int((off + size)[owner == o].max()) for o in range(world)]
    for o in range(world):
        seg = arena[lo[o]:hi[o]].clone()
        dist.broadcast(seg, src=o)
        arena[lo[o]:hi[o]] = seg
    expect = np.repeat(np.arange(cost.size)[order], size[order]).astype(np.float64)
    ok = bool(np.array_equal(arena.numpy(), expect))
    loads = [float(cost[owner == o].sum()) for o in range(world)]
    contiguous = all(hi[o] - lo[o] == int(size[owner == o].sum()) for o in range(world))
    q.put((rank, same, ok, loads, contiguous))
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
    cost = _leaf_costs()
    for rank, same, ok, loads, contiguous in out:
        assert same and ok and contiguous
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(loads) / 2 + cost.max()
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
