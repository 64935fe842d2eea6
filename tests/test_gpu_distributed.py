"""Two real processes on the one B200: the hash-sharded TSDF path end to end
(ShardedGrid.integrate_frames with recorded CUDA graphs, the halo all-to-all
and the gather-to-root device mesh merge) over a CPU-staged gloo group,
compared bit for bit with the single-grid pipeline.  The ranks' kernels never
wait on each other -- only the host-side collectives synchronise them -- so
sharing one GPU is safe (B200_PROFILING.md)."""

import hashlib
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VOXEL, FRAMES = 0.1, 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _sharded_job(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, "ERROR " + repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _inputs():
    import torch

    from paper_2112_02779_b200 import pipeline, scenes
    intr = scenes.ouster64()
    traj = scenes.street_trajectory(FRAMES, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    return intr, frames, poses, inv


def _block_hashes(grid):
    keys, vox = grid.export_blocks()
    return {tuple(k): hashlib.sha1(vox[i].tobytes()).hexdigest() for i, k in enumerate(keys.tolist())}


def _sharded_job(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch

    from paper_2112_02779_b200 import distributed as rkd
    from paper_2112_02779_b200 import pipeline
    d = rkd.CpuStagedDist()
    intr, frames, poses, inv = _inputs()
    if rank != 0:  # the frames reach the other ranks by broadcast, as in the bench
        frames.zero_()
        poses.zero_()
    rkd.broadcast_frames(frames, poses, 0, d)
    d.broadcast(inv, 0)
    sg = rkd.ShardedGrid(VOXEL, rank, world, dist=d, capacity=8192)
    counts = []
    for rep in range(2):  # record, then replay the two graphs
        pipeline.clear_grid(sg.grid)
        upd = sg.integrate_frames(intr, frames, poses, inv, clip_max=30.0, graph=True)
        tot = upd.clone()
        d.all_reduce(tot)
        counts.append(int(tot.item()))
    mesh = sg.extract_mesh(root=0)
    out = {"counts": counts, "blocks": _block_hashes(sg.grid), "graphs": len(sg.grid._graphs)}
    if mesh is not None:
        out["mesh"] = (mesh.vertices, mesh.triangles, mesh.normals)
    torch.cuda.synchronize()
    return out


def test_two_process_sharded_tsdf_and_mesh_equal_single_grid():
    import torch.multiprocessing as mp

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import distributed as rkd
    from paper_2112_02779_b200 import pipeline
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        assert res[r]["graphs"] == 1          # recorded once, replayed once
    # the single-grid reference on this process
    intr, frames, poses, inv = _inputs()
    full = rk.VoxelBlockGrid(voxel_size=VOXEL, capacity=8192)
    upd = pipeline.integrate_sequence(full, intr, frames, poses, inv, clip_max=30.0)
    n_full = int(upd.item())
    ref = _block_hashes(full)
    assert res[0]["counts"] == [n_full, n_full] == res[1]["counts"]
    owned = {}
    for r in range(world):
        for k, h in res[r]["blocks"].items():
            assert k not in owned, f"block {k} on two ranks"
            owned[k] = h
            assert int(rkd.block_owner(np.array([k]), world)[0]) == r
    assert owned == ref                        # same blocks, bit-identical voxels
    V, T, N = res[0]["mesh"]
    m = rk.extract_mesh(full)
    assert V.shape[0] == m.n_vertices and T.shape[0] == m.n_triangles > 1000
    pos = {tuple(p): i for i, p in enumerate(m.vertices.tolist())}
    remap = np.array([pos[tuple(p)] for p in V.tolist()])
    assert np.array_equal(N, m.normals[remap])
    canon = lambda tris: {tuple(np.roll(t, -int(np.argmin(t)))) for t in tris.tolist()}  # noqa: E731
    assert canon(remap[T]) == canon(m.triangles)
    assert "mesh" not in res[1]                # gathered to the root only
