"""Multi-rank logic of the sharded paths, run as 2 CPU processes over gloo
(the driver's GPU boxes have one B200; NCCL uses the same calls)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_02779_b200 import distributed as rkd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


# ---------------------------------------------------------------- workers (module level: picklable)

def _gather_job(rank, world):
    t = torch.arange(3 + 2 * rank, dtype=torch.float64).reshape(-1, 1) + 100 * rank
    g = rkd.all_gather_varsize(t)
    return g.squeeze(1).tolist()


def _broadcast_job(rank, world):
    frames = torch.full((2, 4, 8), float(rank), dtype=torch.float32)
    poses = torch.full((2, 12), float(rank), dtype=torch.float64)
    if rank == 0:
        frames[:] = torch.arange(64, dtype=torch.float32).reshape(2, 4, 8)
        poses[:] = 7.0
    rkd.broadcast_frames(frames, poses, src=0)
    return float(frames.sum()), float(poses.sum())


def _touch_job(rank, world):
    stats = torch.tensor([10 + rank, 1000 * (rank + 1)], dtype=torch.int64)
    rkd.reduce_touch_stats(stats)
    return stats.tolist()


def _touch_frames_job(rank, world):
    stats = torch.tensor([[10 + rank, 1000 * (rank + 1)], [5, 7 - rank], [0, 0]], dtype=torch.int64)
    return rkd.reduce_touch_stats_frames(stats).tolist()


def _pair_shard_job(rank, world):
    """Each rank 'registers' its slice (a stand-in transform of the pair id);
    the gathered poses must equal the single-rank result in order."""
    n = 37
    lo, hi = rkd.shard(n, rank, world)
    local = torch.arange(lo, hi, dtype=torch.float64).reshape(-1, 1).repeat(1, 12) * 0.5
    return rkd.all_gather_varsize(local)[:, 0].tolist()


# ---------------------------------------------------------------- tests

@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (65536, 8), (99, 3), (5, 8)])
def test_shard_partition(n, world):
    spans = [rkd.shard(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [hi - lo for lo, hi in spans]
    assert max(sizes) - min(sizes) <= 1


def test_all_gather_varsize_gloo():
    out = run_ranks(_gather_job)
    expect = [0.0, 1.0, 2.0] + [100.0, 101.0, 102.0, 103.0, 104.0]
    assert out[0] == expect and out[1] == expect


def test_broadcast_frames_gloo():
    out = run_ranks(_broadcast_job)
    assert out[0] == out[1] == (float(sum(range(64))), 7.0 * 24)


def test_reduce_touch_stats_gloo():
    out = run_ranks(_touch_job)
    assert out[0] == out[1] == [21, 2000]


def test_reduce_touch_stats_frames_gloo():
    """The batched sharded sequence reduces all F frames' pairs in one collective."""
    out = run_ranks(_touch_frames_job)
    assert out[0] == out[1] == [[21, 2000], [10, 7], [0, 0]]


def test_sharded_pairs_gather_in_order_gloo():
    out = run_ranks(_pair_shard_job)
    assert out[0] == out[1] == [0.5 * i for i in range(37)]


def test_halo_plan_selects_exactly_the_foreign_neighbours():
    g = np.random.default_rng(3)
    keys = np.unique(g.integers(-4, 5, size=(300, 3)), axis=0)
    owner = np.arange(len(keys)) % 3
    by_rank = [keys[owner == r] for r in range(3)]
    plan = rkd.halo_plan(by_rank)
    for s_ in range(3):
        for r in range(3):
            got = {tuple(k) for k in by_rank[r][plan[r][s_]].tolist()}
            if r == s_:
                assert not got
                continue
            want = {tuple(k) for k in by_rank[r].tolist()
                    if np.any(np.abs(by_rank[s_] - np.array(k)).max(axis=1) == 1)}
            assert got == want


def test_merge_meshes_dedups_shared_boundary_vertices():
    V0 = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    V1 = np.array([[1.0, 0, 0], [0, 1, 0], [1, 1, 0]])       # two vertices shared with V0
    T0, T1 = np.array([[0, 1, 2]]), np.array([[0, 2, 1]])
    N0, N1 = np.tile([0, 0, 1.0], (3, 1)), np.tile([0, 0, 1.0], (3, 1))
    V, T, N = rkd.merge_meshes([(V0, T0, N0), (V1, T1, N1)])
    assert V.shape == (4, 3) and T.shape == (2, 3)
    tris = {tuple(sorted(map(tuple, V[t].tolist()))) for t in T}
    assert tris == {tuple(sorted(map(tuple, V0.tolist()))), tuple(sorted(map(tuple, V1.tolist())))}


def _halo_exchange_job(rank, world):
    """The all-to-all of halo keys as ShardedGrid.extract_mesh does it (CPU)."""
    keys = np.array([[x, 0, 0] for x in range(6)])
    mine = keys[np.arange(6) % world == rank]
    allk = [keys[np.arange(6) % world == q] for q in range(world)]
    plan = rkd.halo_plan(allk)
    send = torch.from_numpy(np.concatenate([mine[plan[rank][s_]] for s_ in range(world)]).astype(np.int32))
    out_split = [int(plan[q][rank].size) for q in range(world)]
    in_split = [int(plan[rank][s_].size) for s_ in range(world)]
    recv = torch.empty((sum(out_split), 3), dtype=torch.int32)
    torch.distributed.all_to_all_single(recv, send, out_split, in_split)
    return sorted(recv[:, 0].tolist())


def test_halo_exchange_gloo():
    out = run_ranks(_halo_exchange_job)
    assert out[0] == [1, 3, 5] and out[1] == [0, 2, 4]     # x-neighbours owned by the other rank


def test_block_owner_partitions_keys(golden_tsdf):
    keys = golden_tsdf["street_keys"]
    for world in (2, 4, 8):
        own = rkd.block_owner(keys, world)
        assert own.min() >= 0 and own.max() < world
        counts = np.bincount(own, minlength=world)
        assert counts.min() > 0.7 * len(keys) / world      # hash spreads blocks evenly
        again = rkd.block_owner(keys[::-1], world)[::-1]
        assert np.array_equal(own, again)                    # pure function of the key
