"""One process per GPU (torch.distributed over NCCL/NVLink) for the paths that
shard:

* ICP: independent pairs are split into contiguous slices (``shard``); the
  only collective is the final pose all-gather (``all_gather_varsize``).
* TSDF: voxel blocks are hash-sharded across ranks -- rank r allocates and
  integrates only blocks with ``owner(key) == r`` (``rk_grid_set_shard``).
  Per frame the range image + pose are broadcast once; the frame's touched
  count / largest key are reduced so every rank reproduces the reference's
  sorted-chunk arithmetic.  Meshing: each rank receives the halo blocks it
  needs (26-neighbours owned elsewhere) in one all-to-all, runs marching
  cubes on its own blocks, and the partial meshes are gathered to one rank
  and merged there on the device by exact vertex position (the reference's
  own dedup rule).

The communication helpers take plain tensors so they run under the ``gloo``
backend on CPU as well (tests/test_distributed.py); ``ShardedGrid`` adds the
device grid on top.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native as nat


def init_from_env(backend: str | None = None):
    """torch.distributed from torchrun's env (RANK/WORLD_SIZE/MASTER_*);
    returns (dist or None, rank, world)."""
    if "RANK" not in os.environ or int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return None, 0, 1
    import torch
    import torch.distributed as dist
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if not dist.is_initialized():
        dist.init_process_group(backend)
    return dist, dist.get_rank(), dist.get_world_size()


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n independent units for one rank; slices
    differ in size by at most one and cover 0..n exactly."""
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def all_gather_varsize(t, dist=None):
    """All-gather tensors whose first dimension differs per rank (counts
    first, then one padded all_gather); returns the concatenation in rank order."""
    import torch
    import torch.distributed as tdist
    d = dist or tdist
    world = d.get_world_size()
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    width = max(counts) if counts else 0
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    d.all_gather(bufs, pad)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)])


def gather_varsize_to(t, dst: int = 0, dist=None):
    """Gather tensors whose first dimension differs per rank onto rank
    ``dst`` only (counts all-gathered first, then one padded gather); returns
    the rank-order concatenation on ``dst`` and None elsewhere."""
    import torch
    import torch.distributed as tdist
    d = dist or tdist
    world, rank = d.get_world_size(), d.get_rank()
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    width = max(counts) if counts else 0
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    d.gather(pad, bufs, dst=dst)
    if rank != dst:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)])


class CpuStagedDist:
    """torch.distributed's collectives for CUDA tensors over a CPU-only
    backend (gloo): every call stages through host memory.  Lets several
    ranks share one GPU in tests (the driver's boxes have one B200); the
    production path passes torch.distributed itself (NCCL)."""

    def __init__(self, dist=None):
        import torch.distributed as tdist
        self.d = dist or tdist
        self.ReduceOp = self.d.ReduceOp

    def get_world_size(self):
        return self.d.get_world_size()

    def get_rank(self):
        return self.d.get_rank()

    def barrier(self):
        self.d.barrier()

    def broadcast(self, t, src):
        h = t.cpu()
        self.d.broadcast(h, src)
        t.copy_(h)

    def all_reduce(self, t, op=None):
        h = t.cpu()
        self.d.all_reduce(h, op=op or self.d.ReduceOp.SUM)
        t.copy_(h)

    def all_gather(self, out, t):
        hs = [o.cpu() for o in out]
        self.d.all_gather(hs, t.cpu())
        for o, h in zip(out, hs):
            o.copy_(h)

    def gather(self, t, gather_list=None, dst=0):
        hs = [o.cpu() for o in gather_list] if gather_list is not None else None
        self.d.gather(t.cpu(), hs, dst=dst)
        if gather_list is not None:
            for o, h in zip(gather_list, hs):
                o.copy_(h)

    def all_to_all_single(self, out, inp, out_split=None, in_split=None):
        h = out.cpu()
        self.d.all_to_all_single(h, inp.cpu(), out_split, in_split)
        out.copy_(h)


def broadcast_frames(frames, poses, src: int = 0, dist=None):
    """Broadcast (F,H,W) float32 frames and (F,12) float64 poses from src."""
    import torch.distributed as tdist
    d = dist or tdist
    d.broadcast(frames, src)
    d.broadcast(poses, src)
    return frames, poses


def reduce_touch_stats(stats, dist=None):
    """{local touched count, local max key} -> {global count, global max key}
    (int64[2] tensor, in place)."""
    import torch
    import torch.distributed as tdist
    d = dist or tdist
    world = d.get_world_size()
    bufs = [torch.empty_like(stats) for _ in range(world)]
    d.all_gather(bufs, stats)
    allv = torch.stack(bufs)
    stats[0] = allv[:, 0].sum()
    stats[1] = allv[:, 1].max()
    return stats


def reduce_touch_stats_frames(stats, dist=None):
    """(F, 2) per-frame {local count, local max key} -> global {sum, max}
    with one all-gather for the whole sequence (returns a new tensor)."""
    import torch
    import torch.distributed as tdist
    d = dist or tdist
    bufs = [torch.empty_like(stats) for _ in range(d.get_world_size())]
    d.all_gather(bufs, stats.contiguous())
    allv = torch.stack(bufs)                     # (world, F, 2)
    return torch.stack([allv[..., 0].sum(0), allv[..., 1].max(0).values], -1).contiguous()


def block_owner(keys, world: int) -> np.ndarray:
    """Owning rank of each block key (host mirror of the device owner hash)."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.int32).reshape(-1, 3))
    out = np.empty(k.shape[0], dtype=np.int32)
    nat.call("rk_block_owner", k.ctypes.data, k.shape[0], int(world), out.ctypes.data)
    return out


class ShardedGrid:
    """A VoxelBlockGrid whose blocks are hash-sharded over the ranks."""

    def __init__(self, voxel_size, rank, world, dist=None, **grid_kw):
        from .sdf_volume import VoxelBlockGrid
        self.grid = VoxelBlockGrid(voxel_size=voxel_size, **grid_kw)
        self.rank, self.world, self.dist = rank, world, dist
        self._slots = 0   # touched-set slots reserved so far (graphs live in grid._graphs)
        nat.call("rk_grid_set_shard", self.grid._ensure(), int(rank), int(world))

    def integrate_frames(self, intr, frames, poses_w, inv_w, clip_min=0.0, clip_max=np.inf,
                         updated=None, graph: bool = False, reduce=None):
        """integrate_cloud_frame for F frames on this rank's shard.  frames /
        poses must already be identical on every rank (see broadcast_frames).

        All F frames are activated first (one touched-set slot each), the
        per-frame {count, max key} pairs are reduced across ranks in one
        collective (the reference's sorted-chunk arithmetic needs the global
        values), then the F integrations run back to back.

        graph=True records the two device phases (3F activation launches +
        the stats export; F integrations) as two CUDA graphs on the first
        call with these buffers and replays them afterwards, so a step costs
        two graph launches and one collective instead of ~4F kernel launches
        (at 8 ranks the per-rank GPU work of a 100-frame sequence is shorter
        than issuing those launches).  ``reduce`` overrides the collective
        (tests emulate several shards in one process).

        The caller presizes the pool (``self.grid.reserve``): unlike the
        single-GPU per-frame API there is no grow-and-retry here, so an
        activation that overflows raises DeviceError (checked after eager
        activations and after the first replay of a recorded graph).
        Returns the device int64 updated-voxel counter."""
        from . import lidar_model as lm
        g = self.grid
        h = g._prepare()
        sensor = lm.device_sensor(intr)
        own_upd = updated is None
        if own_upd:
            updated = nat.zeros((1,), np.int64)
        F = int(frames.shape[0])
        cmin, cmax = float(np.float32(clip_min)), float(np.float32(clip_max))
        frames, poses_w, inv_w = frames.contiguous(), poses_w.contiguous(), inv_w.contiguous()
        sharded = self.world > 1 or reduce is not None
        red = reduce or (lambda st: reduce_touch_stats_frames(st, self.dist))
        if F > self._slots:
            # growing the touched-set slots reallocates them: recorded graphs
            # (this grid's, incl. integrate_sequence's) point at the old ones
            g._graphs.clear()
            self._slots = F
        nat.call("rk_grid_reserve_slots", h, F, nat.stream_ptr())
        # a counter this call allocates is owned by the cache entry (zeroed
        # per replay), so it does not key the cache
        key = ("sharded", sensor, frames.data_ptr(), F, poses_w.data_ptr(), inv_w.data_ptr(),
               None if own_upd else updated.data_ptr(), cmin, cmax, lm.default_math())
        bufs = g._graphs.get(key) if graph else None
        if bufs is None:
            bufs = dict(stats=nat.zeros((F, 2), np.int64), glob=nat.zeros((F, 2), np.int64),
                        upd=updated)
        elif own_upd:
            bufs["upd"].zero_()
        upd = bufs["upd"]

        def activate():
            st = nat.stream_ptr()
            nat.call("rk_grid_activate_frames", h, sensor, nat.ptr(frames), F, nat.ptr(poses_w),
                     float(g.truncation), cmin, cmax, st)
            if sharded:
                nat.call("rk_grid_touch_stats_frames", h, F, nat.ptr(bufs["stats"]), st)

        def integrate():
            nat.call("rk_grid_integrate_activated", h, sensor, nat.ptr(frames), F, nat.ptr(inv_w),
                     nat.ptr(bufs["glob"]) if sharded else None, cmin, cmax, lm.default_math(),
                     nat.ptr(upd), nat.stream_ptr())

        # The pool must be presized (grid.reserve): an activation that runs
        # out of slots leaves new blocks unallocated and K5 would skip them,
        # so the overflow flag is checked after every eager activation and
        # after the first replay of a freshly recorded graph, before any
        # integration runs.
        if not graph:
            activate()
            g.check_overflow()
            if sharded:
                bufs["glob"].copy_(red(bufs["stats"]))
            integrate()
        else:
            if "ga" not in bufs:
                torch = nat.torch()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                for name, fn in (("ga", activate), ("gi", integrate)):
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, stream=side, capture_error_mode="thread_local"):
                        fn()
                    bufs[name] = gr
                torch.cuda.current_stream().wait_stream(side)
                g.cache_graph(key, bufs)
                bufs["ga"].replay()
                g.check_overflow()
            else:
                bufs["ga"].replay()
            if sharded:
                bufs["glob"].copy_(red(bufs["stats"]))
            bufs["gi"].replay()
        g.blocks._bump()
        return upd.clone() if own_upd else upd

    def extract_mesh(self, min_weight: float = 1.0, root: int = 0):
        """Distributed marching cubes: the block keys are all-gathered (12 B
        per block) and every rank derives the halo plan on the device; one
        all-to-all moves the halo blocks; each rank meshes its own blocks; the
        partial meshes are gathered to ``root`` only and merged there on the
        device by exact vertex position (the reference's dedup rule,
        mesh_extract.py:146-151, which also joins the edges both neighbouring
        ranks produce on a shard boundary).  Returns a host TriangleMesh on
        ``root`` and None on the other ranks."""
        import torch

        from .mesh_extract import TriangleMesh
        d, world, rank = self.dist, self.world, self.rank
        keys, vox = self.grid.export_blocks(device=True)
        if world == 1:
            V, T, N = merge_meshes_device([mesh_from_shard(self.grid, 0, 1, min_weight=min_weight)])
            return TriangleMesh(nat.to_host(V), nat.to_host(T), nat.to_host(N))
        n = torch.tensor([keys.shape[0]], dtype=torch.int64, device=keys.device)
        counts = [torch.zeros_like(n) for _ in range(world)]
        d.all_gather(counts, n)
        counts = [int(c.item()) for c in counts]
        all_keys = all_gather_varsize(keys, d)
        bounds = np.cumsum([0] + counts)
        by_rank = [all_keys[bounds[q]:bounds[q + 1]] for q in range(world)]
        send = halo_send(by_rank, rank)                      # my blocks each rank needs
        recv_n = [int(halo_send(by_rank, q, only=rank)[rank].numel()) for q in range(world)]
        in_split = [int(send[q].numel()) for q in range(world)]
        sel = torch.cat(send) if send else torch.zeros(0, dtype=torch.int64, device=keys.device)
        k_send = keys[sel].contiguous()
        v_send = vox[sel].reshape(-1, 8192).contiguous()
        k_recv = torch.empty((sum(recv_n), 3), dtype=keys.dtype, device=keys.device)
        v_recv = torch.empty((sum(recv_n), 8192), dtype=vox.dtype, device=vox.device)
        d.all_to_all_single(k_recv, k_send, recv_n, in_split)
        d.all_to_all_single(v_recv, v_send, recv_n, in_split)
        V, T, N = mesh_from_shard(self.grid, rank, world, k_recv, v_recv, min_weight)
        nvs = [torch.zeros(1, dtype=torch.int64, device=V.device) for _ in range(world)]
        d.all_gather(nvs, torch.tensor([V.shape[0]], dtype=torch.int64, device=V.device))
        base = sum(int(c.item()) for c in nvs[:rank])
        Vg = gather_varsize_to(V, root, d)
        Ng = gather_varsize_to(N, root, d)
        Tg = gather_varsize_to(T.to(torch.int64) + base, root, d)
        if rank != root:
            return None
        Vm, Tm, Nm = merge_meshes_device([(Vg, Tg, Ng)])
        return TriangleMesh(nat.to_host(Vm), nat.to_host(Tm), nat.to_host(Nm))

    def gather_blocks(self):
        """All ranks' (keys (n,3) int32, voxels (n,4096,2) float32), device, rank order."""
        g = self.grid
        keys = nat.to_dev(g._export_keys(touched=False), np.int32)
        vox = nat.empty((keys.shape[0], 4096, 2), np.float32)
        if keys.shape[0]:
            nat.call("rk_grid_read_blocks", g._handle, nat.ptr(keys), keys.shape[0], nat.ptr(vox), None,
                     nat.stream_ptr())
        if self.world == 1:
            return keys, vox
        return all_gather_varsize(keys, self.dist), all_gather_varsize(vox, self.dist)

    def merged_grid(self):
        """A single-device grid holding every rank's blocks (for meshing)."""
        from .sdf_volume import VoxelBlockGrid
        keys, vox = self.gather_blocks()
        n = int(keys.shape[0])
        out = VoxelBlockGrid(voxel_size=self.grid.voxel_size, truncation=self.grid.truncation,
                             max_weight=self.grid.max_weight, capacity=max(1024, 2 * n))
        if n:
            nat.call("rk_grid_write_blocks", out._ensure(), nat.ptr(keys.contiguous()), n,
                     nat.ptr(vox.contiguous()), nat.stream_ptr())
            out.blocks._bump()
        return out


# ---------------------------------------------------------------- sharded meshing

_NEIGH = np.array([(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
                   if (dx, dy, dz) != (0, 0, 0)], dtype=np.int64)


def _codes(keys) -> np.ndarray:
    k = np.asarray(keys, dtype=np.int64).reshape(-1, 3) + (1 << 17)
    return (k[:, 0] << 36) | (k[:, 1] << 18) | k[:, 2]   # sdf_volume.py:64-71 packing


def _codes_t(keys):
    """sdf_volume.py:64-71 packing of (n, 3) integer keys, torch (any device)."""
    import torch
    k = keys.to(torch.int64).reshape(-1, 3) + (1 << 17)
    return (k[:, 0] << 36) | (k[:, 1] << 18) | k[:, 2]


def halo_send(keys_by_rank, r: int, only: int | None = None):
    """send[s]: indices into rank r's block list (a torch tensor on any
    device) of the blocks rank s needs as halo -- the 26-neighbours of s's
    blocks that r owns (marching cubes reads a 19^3 window,
    mesh_extract.py:58-82).  ``only`` restricts the work to one s."""
    import torch
    world = len(keys_by_rank)
    kr = keys_by_rank[r]
    dev = kr.device
    neigh = torch.from_numpy(_NEIGH).to(dev)
    codes_r = _codes_t(kr)
    out = [torch.zeros(0, dtype=torch.int64, device=dev) for _ in range(world)]
    for s_ in range(world):
        if s_ == r or (only is not None and s_ != only):
            continue
        ks = keys_by_rank[s_].to(torch.int64).reshape(-1, 3)
        if ks.shape[0] == 0 or codes_r.numel() == 0:
            continue
        need = _codes_t((ks[:, None, :] + neigh[None]).reshape(-1, 3))
        out[s_] = torch.nonzero(torch.isin(codes_r, need)).reshape(-1)
    return out


def halo_plan(keys_by_rank):
    """send[r][s] for every pair of ranks as host index arrays (the same
    device computation, ``halo_send``, run per rank)."""
    import torch
    kt = [torch.as_tensor(np.asarray(k, dtype=np.int64).reshape(-1, 3)) for k in keys_by_rank]
    return [[x.cpu().numpy() for x in halo_send(kt, r)] for r in range(len(kt))]


def mesh_from_shard(grid, rank: int, world: int, halo_keys=None, halo_vox=None,
                    min_weight: float = 1.0):
    """Marching cubes over the blocks this rank owns, with the halo blocks of
    other ranks as read-only neighbours: (V, T, N) CUDA tensors."""
    from .mesh_extract import extract_mesh_device
    from .sdf_volume import VoxelBlockGrid
    keys, vox = grid.export_blocks(device=True)
    n_halo = 0 if halo_keys is None else int(halo_keys.shape[0])
    tmp = VoxelBlockGrid(voxel_size=grid.voxel_size, truncation=grid.truncation,
                         max_weight=grid.max_weight,
                         capacity=max(1024, 2 * (int(keys.shape[0]) + n_halo)))
    tmp.import_blocks(keys, vox)
    if n_halo:
        tmp.import_blocks(halo_keys, halo_vox)
    nat.call("rk_grid_set_shard", tmp._ensure(), int(rank), int(world))
    return extract_mesh_device(tmp, min_weight)


def merge_meshes_device(parts):
    """Concatenate per-rank (V, T, N) meshes (tensors on one device) and merge
    vertices at the same exact float64 position, keeping each position's
    first normal -- np.unique(V, axis=0) semantics (lexicographically sorted
    unique positions), on the device.  Returns (V, T int32, N) tensors."""
    import torch
    Vs, Ts, Ns, base = [], [], [], 0
    for v, t, n in parts:
        v = torch.as_tensor(v, dtype=torch.float64).reshape(-1, 3)
        Vs.append(v)
        Ts.append(torch.as_tensor(t).to(device=v.device, dtype=torch.int64).reshape(-1, 3) + base)
        Ns.append(torch.as_tensor(n, dtype=torch.float64).to(v.device).reshape(-1, 3))
        base += v.shape[0]
    V, T, N = torch.cat(Vs), torch.cat(Ts), torch.cat(Ns)
    if V.shape[0] == 0:
        return V, T.to(torch.int32), N
    # -0.0 and 0.0 are one position for np.unique (they compare equal)
    V = V + 0.0
    uniq, inv = torch.unique(V, dim=0, return_inverse=True)
    pos = torch.arange(V.shape[0], device=V.device)
    first = torch.full((uniq.shape[0],), V.shape[0], dtype=torch.int64, device=V.device)
    first = first.scatter_reduce(0, inv, pos, reduce="amin")
    return uniq, inv[T].to(torch.int32), N[first]


def merge_meshes(parts):
    """Host wrapper of merge_meshes_device: returns numpy (V, T, N)."""
    import torch
    parts = [tuple(x if nat.is_tensor(x) else torch.as_tensor(np.asarray(x)) for x in p) for p in parts]
    V, T, N = merge_meshes_device(parts)
    return V.cpu().numpy(), T.cpu().numpy(), N.cpu().numpy()
