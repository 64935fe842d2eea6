#!/usr/bin/env python
"""Benchmark of the rangekit hot path on B200 (BASELINE.json metric:
"ICP registrations/sec (64x1024 pairs) and TSDF frames/sec @5cm, % HBM roofline").

One step =
  (a) ICP: C4 -- a batch of 65,536 independent 64x1024 scan pairs (strong
      scaling: each of N ranks registers its contiguous 65,536/N slice), drawn
      from a device-rendered pool of 2,048 unique street pairs; K1 normals of
      every pool destination + one K3 launch running the full multi-scale
      schedule (4:20, 2:20, 1:10, early exit) for every pair;
  (b) TSDF: C2 -- the 100-frame 64x1024 street sequence integrated at 5 cm
      voxels (tau 0.2 m, max_weight 100, clip 30 m) into a freshly cleared grid.
``value`` is (a) in registrations/s over all ranks; (b) is reported under
"tsdf".  Inputs live in HBM before the timed region; the ICP pool (>3 GB) is
far larger than the 126 MB L2.  ``e2e`` repeats (a)+(b) through the public API
with pinned-host inputs copied in and poses / voxel counts copied out inside
the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ICP registrations/sec (64x1024 pairs) and TSDF frames/sec @5cm, % HBM roofline"
ICP_BYTES_PER_PT_IT = 20      # src range 4 + dst range 4 + dst normal 12
TSDF_BYTES_PER_VOXEL = 16     # 8 B read + 8 B write of {tsdf, weight}
TSDF_BYTES_PER_PIXEL = 4
TSDF_VOXEL = {"c2": 0.05, "c3": 0.10, "c5": 0.03}
TSDF_DESC = {"c2": "C2: {n}-frame 64x1024 street sequence, TSDF 5 cm",
             "c3": "C3: {n}-frame HDL-64 64x2048 street sequence, TSDF 10 cm",
             "c5": "C5: {n}-frame OS-128 128x2048 extended-street sequence (0.5 m/frame), TSDF 3 cm"}
TSDF_CAPACITY = {"c2": 65536, "c3": 65536, "c5": 262144}   # voxel blocks (32 KB each)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=65536)
    ap.add_argument("--pool", type=int, default=2048)
    ap.add_argument("--frames", type=int, default=100)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra one-GPU lines (math modes, K1 per pair, independent-pair e2e, "
                         "C5 TSDF, per-kernel rooflines)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    # TSDF sequence shape: c2 (default; 64x1024 Ouster-like, 5 cm), c3 (HDL-64
    # 64x2048, 10 cm), c5 (OS-128 128x2048, 3 cm) -- BASELINE.json configs
    ap.add_argument("--tsdf-config", default="c2", choices=["c2", "c3", "c5"])
    # projection arithmetic: np = numpy-exact (the reference's bits), fast =
    # minimax transcendentals + float32 ICP move, cr = correctly rounded
    ap.add_argument("--math", default=None, choices=["np", "fast", "cr"])
    # diagnostic only (not a bench configuration): every pair reads pool image 0's
    # destination, isolating the cost of the data-dependent surfel gather
    ap.add_argument("--diag-same-dst", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ workloads

def make_inputs(args, rank, world, device):
    """Render the ICP pool and the TSDF sequence on the device."""
    import torch

    from paper_2112_02779_b200 import pipeline, scenes
    intr = scenes.ouster64()
    street = scenes.street_scene()
    pool = scenes.pair_pool_poses(args.pool, seed=0)
    dst_poses = [b for b, _ in pool]
    src_poses = [b @ gt for b, gt in pool]
    src = pipeline.render_batch(intr, street, src_poses)
    dst = pipeline.render_batch(intr, street, dst_poses)
    lo, hi = pipeline.shard(args.pairs, rank, world)
    # spread concurrent CTAs over different pool images (golden-ratio stride)
    idx = (np.arange(lo, hi, dtype=np.int64) * 1237) % args.pool
    pair_idx = torch.from_numpy(idx.astype(np.int32)).to(device)
    tintr = {"c2": intr, "c3": scenes.hdl64(), "c5": scenes.os128()}[args.tsdf_config]
    if args.tsdf_config == "c5":
        # C5: the extended street at 0.5 m/frame
        # small twist jitter: over 1,000 frames the default +-2 mrad random walk
        # takes the sensor below the ground slab (z drifts ~4 m)
        traj = scenes.street_trajectory(args.frames, seed=0, step_m=0.5, jitter=0.0002)
        frames = pipeline.render_batch(tintr, scenes.extended_street_scene(0.5 * args.frames + 30.0), traj)
    else:
        traj = scenes.street_trajectory(args.frames, seed=0)
        frames = pipeline.render_batch(tintr, street, traj)
    poses_w = torch.from_numpy(pipeline.poses_to_rows(traj)).to(device)
    inv_w = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).to(device)
    gts = np.stack([gt.as_row12() for _, gt in pool])
    torch.cuda.synchronize()
    pair_dst = torch.zeros_like(pair_idx) if args.diag_same_dst else pair_idx
    return dict(intr=intr, tintr=tintr, src=src, dst=dst, pair_idx=pair_idx, pair_dst=pair_dst,
                n_pairs=hi - lo,
                frames=frames,
                poses_w=poses_w, inv_w=inv_w, traj=traj, gts=gts)


class TsdfRunner:
    """C2 sequence integration: one grid on one GPU; at N > 1 the blocks are
    hash-sharded over the ranks (each integrates its own blocks for every
    frame) and rank 0 broadcasts the frames + poses over NCCL first."""

    def __init__(self, intr, rank, world, dist, voxel=0.05, capacity=65536):
        import paper_2112_02779_b200 as rk
        from paper_2112_02779_b200 import distributed as rkd
        self.intr, self.world, self.dist = intr, world, dist
        if world > 1:
            self.sharded = rkd.ShardedGrid(voxel, rank, world, dist, capacity=capacity)
            self.grid = self.sharded.grid
        else:
            self.sharded = None
            self.grid = rk.VoxelBlockGrid(voxel_size=voxel, capacity=capacity)

    def run(self, frames, poses_w, inv_w, updated):
        from paper_2112_02779_b200 import distributed as rkd
        from paper_2112_02779_b200 import pipeline
        pipeline.clear_grid(self.grid)
        if self.sharded is None:
            # one CUDA graph replay per sequence (recorded on the first call)
            return pipeline.integrate_sequence(self.grid, self.intr, frames, poses_w, inv_w,
                                               clip_max=30.0, updated=updated, graph=True)
        rkd.broadcast_frames(frames, poses_w, src=0, dist=self.dist)
        self.dist.broadcast(inv_w, 0)
        return self.sharded.integrate_frames(self.intr, frames, poses_w, inv_w, clip_max=30.0,
                                             updated=updated, graph=True)


def run_ours(args, rank, world, dist):
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import pipeline
    from paper_2112_02779_b200.range_image import normals_cross_batch

    device = torch.device("cuda", torch.cuda.current_device())
    D = make_inputs(args, rank, world, device)
    intr = D["intr"]
    cfg = rk.RegistrationConfig()
    tsdf = TsdfRunner(D["tintr"], rank, world, dist, TSDF_VOXEL[args.tsdf_config],
                      TSDF_CAPACITY[args.tsdf_config])
    grid = tsdf.grid
    stream = torch.cuda.current_stream()
    pt_iters = torch.zeros(1, dtype=torch.int64, device=device)
    updated = torch.zeros(1, dtype=torch.int64, device=device)

    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for k in ("normals", "icp", "tsdf")}
    acc = {k: 0.0 for k in ev}

    def step(timed):
        e = ev["normals"]
        e[0].record(stream)
        surf = normals_cross_batch(intr, D["dst"], strides=[s for s, _ in cfg.schedule])
        e[1].record(stream)
        ev["icp"][0].record(stream)
        res = rk.register_batch(intr, D["src"], D["dst"], surf, pair_src=D["pair_idx"],
                                pair_dst=D["pair_dst"], config=cfg, pt_iters=pt_iters if timed else None)
        ev["icp"][1].record(stream)
        ev["tsdf"][0].record(stream)
        # one counter for warm-up and timed steps: the TSDF CUDA graphs are keyed
        # by their buffers, so all recording happens in the warm-up
        tsdf.run(D["frames"], D["poses_w"], D["inv_w"], updated)
        ev["tsdf"][1].record(stream)
        return res

    for _ in range(args.warmup):
        res = step(False)
    torch.cuda.synchronize()
    n_blocks, cap, overflow, _ = grid.info()
    if overflow:
        raise RuntimeError("TSDF pool overflow in warm-up; raise capacity")
    # correctness spot check on the bench's own output: recovered gt poses
    poses = res.poses.cpu().numpy()
    gts = D["gts"][D["pair_idx"].cpu().numpy()]
    terr = np.linalg.norm(poses[:, 9:] - gts[:, 9:], axis=1)
    ok_frac = float(np.mean(terr < 0.05))

    updated.zero_()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step(True)
            torch.cuda.synchronize()
            for k, (a, b) in ev.items():
                acc[k] += a.elapsed_time(b)
        t1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = t0.elapsed_time(t1)
    if dist is not None:
        t = torch.tensor([elapsed_ms, acc["icp"] + acc["normals"], acc["tsdf"]], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, icp_ms, tsdf_ms = t.tolist()
        pt = pt_iters.clone()
        dist.all_reduce(pt)
        upd = updated.clone()
        dist.all_reduce(upd)
        total_pairs = args.pairs
    else:
        icp_ms, tsdf_ms = acc["icp"] + acc["normals"], acc["tsdf"]
        pt, upd = pt_iters, updated
        total_pairs = D["n_pairs"]
    K = args.steps
    # roofline quantities are per GPU: this rank's work over this rank's kernel time
    pt_local, upd_local = pt_iters.item() / K, updated.item() / K
    reg_per_s = total_pairs * K / (icp_ms / 1e3)
    # the ranks share one sequence (hash-sharded blocks): strong scaling
    tsdf_fps = args.frames * K / (tsdf_ms / 1e3)
    pt_per_launch = pt.item() / K
    icp_kernel_ms = acc["icp"] / K
    achieved = ICP_BYTES_PER_PT_IT * pt_local / (icp_kernel_ms / 1e3) / 1e9
    upd_per_step = upd.item() / K
    tin = D["tintr"]
    tsdf_bytes = TSDF_BYTES_PER_VOXEL * upd_local + TSDF_BYTES_PER_PIXEL * tin.height * tin.width * args.frames
    tsdf_achieved = tsdf_bytes / (acc["tsdf"] / K / 1e3) / 1e9
    coarse = len({s for s, _ in cfg.schedule if s > 1})
    launches = K * (1 + coarse + 1 + pipeline.LAUNCHES_CLEAR + pipeline.LAUNCHES_PER_FRAME * args.frames)
    # single-pair latency through the public API (host numpy in, pose out):
    # the online-odometry use (the paper's "registration at 100 Hz")
    latency = None
    if dist is None:
        src0 = D["src"][D["pair_idx"][0]].cpu().numpy()
        dst0 = D["dst"][D["pair_idx"][0]].cpu().numpy()
        for _ in range(3):
            rk.register(rk.RangeImage(src0, intr), rk.RangeImage(dst0, intr))
        torch.cuda.synchronize()
        t_l = time.perf_counter()
        n_l = 20
        for _ in range(n_l):
            res1 = rk.register(rk.RangeImage(src0, intr), rk.RangeImage(dst0, intr))
        latency = {"ms": 1e3 * (time.perf_counter() - t_l) / n_l, "iterations": len(res1.stats),
                   "what": "register() of one 64x1024 pair from host arrays: H2D, K1 normals, "
                           "K3 schedule, pose D2H"}
    # K6 on the sequence's final grid (outside the timed region), wall clock
    # incl. its syncs: extract_mesh through the public API on one GPU; at N > 1
    # the distributed form (halo all-to-all, per-shard MC, mesh gather + merge)
    if dist is None:
        from paper_2112_02779_b200.mesh_extract import extract_mesh_device
        extract_mesh_device(grid)
        mc_ms = []
        for _ in range(3):
            torch.cuda.synchronize()
            t_mc = time.perf_counter()
            v, tri, _ = extract_mesh_device(grid)
            torch.cuda.synchronize()
            mc_ms.append(1e3 * (time.perf_counter() - t_mc))
        mesh = {"ms": float(np.median(mc_ms)), "vertices": int(v.shape[0]),
                "triangles": int(tri.shape[0]), "blocks": int(n_blocks)}
    else:
        tsdf.sharded.extract_mesh()
        dist.barrier()
        torch.cuda.synchronize()
        t_mc = time.perf_counter()
        m = tsdf.sharded.extract_mesh(root=0)
        torch.cuda.synchronize()
        mesh = {"ms": 1e3 * (time.perf_counter() - t_mc), "blocks_this_rank": int(n_blocks),
                "distributed": True, "what": "halo all-to-all, per-rank MC, gather to rank 0, "
                                             "device merge by exact position"}
        if m is not None:
            mesh.update(vertices=int(m.vertices.shape[0]), triangles=int(m.triangles.shape[0]))
    # C2 end to end (outside the timed region, wall clock incl. its one host
    # sync): frame-to-frame odometry of the sequence (one register_batch of
    # F-1 pairs + the host pose prefix product, cli.py:248-263) and the
    # sequence integrated at the ESTIMATED poses (cli.py:267-283)
    odo = None
    if dist is None:
        traj = D["traj"]
        og = rk.VoxelBlockGrid(voxel_size=TSDF_VOXEL[args.tsdf_config],
                               capacity=TSDF_CAPACITY[args.tsdf_config])
        od_ms = []
        for _ in range(4):
            pipeline.clear_grid(og)
            torch.cuda.synchronize()
            t_od = time.perf_counter()
            wposes, _, od_upd = pipeline.odometry_integrate(og, D["tintr"], D["frames"], cfg,
                                                            clip_max=30.0)
            od_upd.item()
            od_ms.append(1e3 * (time.perf_counter() - t_od))
        od = float(np.median(od_ms[1:]))
        drift = max(float(np.linalg.norm(wposes[k].t - (traj[0].inverse() @ traj[k]).t))
                    for k in range(len(traj)))
        odo = {"value": args.frames / (od / 1e3), "unit": "frames/s", "ms": od,
               "max_translation_drift_m": drift,
               "what": f"C2 end to end: odometry of {args.frames} frames (one batched launch of "
                       f"{args.frames - 1} frame-to-frame pairs + host pose chain) and TSDF "
                       "integration at the estimated poses, wall clock incl. one host sync"}
    return dict(reg_per_s=reg_per_s, tsdf_fps=tsdf_fps, elapsed_ms=elapsed_ms, icp_ms=icp_ms,
                tsdf_ms=tsdf_ms, achieved=achieved, pt_per_launch=pt_per_launch,
                icp_kernel_ms=icp_kernel_ms, normals_ms=acc["normals"] / K, pt_local=pt_local,
                upd_local=upd_local,
                tsdf_achieved=tsdf_achieved, tsdf_updated=upd_per_step, n_blocks=n_blocks,
                clocks=clocks.summary(), launches=launches, ok_frac=ok_frac, D=D, tsdf=tsdf, cfg=cfg,
                mesh=mesh, latency=latency, odometry=odo)


def run_e2e(args, rank, world, dist, D, tsdf, cfg):
    """Same step through the public API with host buffers: every step copies
    its input images from pinned host memory (H2D) and reads back poses,
    status and the voxel count (D2H).  Two device staging buffers let the
    copy of step k+1 run on a copy stream while step k computes; the host
    reads step k's results once step k+1 is enqueued."""
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200.range_image import normals_cross_batch
    src_h = D["src"].cpu().pin_memory()
    dst_h = D["dst"].cpu().pin_memory()
    frames_h = D["frames"].cpu().pin_memory()
    bufs = [dict(src=torch.empty_like(D["src"]), dst=torch.empty_like(D["dst"]),
                 frames=torch.empty_like(D["frames"])) for _ in range(2)]
    upd = torch.zeros(1, dtype=torch.int64, device="cuda")
    intr = D["intr"]
    main = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream()
    ev_ready = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    h2d = src_h.numel() * 4 + dst_h.numel() * 4 + frames_h.numel() * 4
    d2h = 0

    def issue_copy(b):
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev_free[b])      # no earlier step still reads buffer b
            bufs[b]["src"].copy_(src_h, non_blocking=True)
            bufs[b]["dst"].copy_(dst_h, non_blocking=True)
            bufs[b]["frames"].copy_(frames_h, non_blocking=True)
            ev_ready[b].record(copy_stream)

    # step results land in pinned host buffers (two sets); the host reads
    # step k's after step k+1 is enqueued, so the GPU never idles on the host
    out_h = [None, None]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def read_back(b):
        nonlocal d2h
        ev_out[b].synchronize()
        poses, status, n_upd = out_h[b]
        d2h = poses.numel() * 8 + status.numel() * 4 + n_upd.numel() * 8
        return poses, status, n_upd

    def run(n):
        issue_copy(0)
        for k in range(n):
            b = k % 2
            if k + 1 < n:
                issue_copy(1 - b)
            main.wait_event(ev_ready[b])
            src, dst, frames = bufs[b]["src"], bufs[b]["dst"], bufs[b]["frames"]
            surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
            res = rk.register_batch(intr, src, dst, surf, pair_src=D["pair_idx"],
                                    pair_dst=D["pair_idx"], config=cfg)
            upd.zero_()
            tsdf.run(frames, D["poses_w"], D["inv_w"], upd)
            ev_free[b].record(main)
            if out_h[b] is None:
                out_h[b] = (torch.empty(res.poses.shape, dtype=res.poses.dtype, pin_memory=True),
                            torch.empty(res.status.shape, dtype=res.status.dtype, pin_memory=True),
                            torch.empty(upd.shape, dtype=upd.dtype, pin_memory=True))
            for h, d in zip(out_h[b], (res.poses, res.status, upd)):
                h.copy_(d, non_blocking=True)
            ev_out[b].record(main)
            if k > 0:
                read_back(1 - b)
        read_back((n - 1) % 2)

    run(2)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    run(args.steps)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([el], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = t.item()
    total_pairs = args.pairs if dist is not None else D["n_pairs"]
    return dict(value=total_pairs * args.steps / el, unit="registrations/s",
                h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                tsdf_frames_in_step=args.frames, seconds=el,
                note="every step's inputs copied H2D inside the timed region; the copy of step "
                     "k+1 overlaps step k (two staging buffers, copy stream); step k's results "
                     "are read on the host after step k+1 is enqueued")


# ------------------------------------------------------------------ extra lines (one GPU)

def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run_math_modes(args, D, cfg, modes=("fast", "cr")):
    """The same ICP + TSDF step in the other projection-arithmetic modes
    (MATH_NP is the headline): registrations/s and TSDF frames/s, one warm-up
    and two timed repetitions each, CUDA events."""
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import lidar_model as lm, pipeline
    from paper_2112_02779_b200.range_image import normals_cross_batch
    intr = D["intr"]
    out = {}
    grid = rk.VoxelBlockGrid(voxel_size=TSDF_VOXEL[args.tsdf_config], capacity=TSDF_CAPACITY[args.tsdf_config])
    for name in modes:
        mode = {"fast": lm.MATH_FAST, "cr": lm.MATH_CR, "np": lm.MATH_NP}[name]
        with lm.math_mode(mode):
            pt = torch.zeros(1, dtype=torch.int64, device="cuda")
            upd = torch.zeros(1, dtype=torch.int64, device="cuda")
            ms_icp = ms_tsdf = 0.0
            for rep in range(3):
                a, b = _events()
                c, d = _events()
                a.record()
                surf = normals_cross_batch(intr, D["dst"], strides=[s for s, _ in cfg.schedule])
                rk.register_batch(intr, D["src"], D["dst"], surf, pair_src=D["pair_idx"], pair_dst=D["pair_dst"],
                                  config=cfg, pt_iters=pt if rep else None)
                b.record()
                pipeline.clear_grid(grid)
                c.record()
                pipeline.integrate_sequence(grid, D["tintr"], D["frames"], D["poses_w"], D["inv_w"],
                                            clip_max=30.0, updated=upd, graph=True)
                d.record()
                torch.cuda.synchronize()
                if rep:
                    ms_icp += a.elapsed_time(b)
                    ms_tsdf += c.elapsed_time(d)
            out[name] = {"registrations_per_s": D["n_pairs"] * 2 / (ms_icp / 1e3),
                         "tsdf_frames_per_s": args.frames * 2 / (ms_tsdf / 1e3),
                         "point_iterations_per_step": pt.item() / 2}
    return out


def run_k1_per_pair(args, D, cfg, icp_kernel_ms):
    """``value`` with K1 charged per pair: the bench's pool computes the
    destination normals once per pool image (2,048) and reuses them across
    the 65,536 pairs; truly independent pairs need one K1 per pair.  K1 over
    the pool is timed and scaled to one image per pair."""
    import torch

    from paper_2112_02779_b200.range_image import normals_cross_batch
    intr = D["intr"]
    normals_cross_batch(intr, D["dst"], strides=[s for s, _ in cfg.schedule])
    a, b = _events()
    a.record()
    reps = 5
    for _ in range(reps):
        normals_cross_batch(intr, D["dst"], strides=[s for s, _ in cfg.schedule])
    b.record()
    torch.cuda.synchronize()
    k1_ms_per_image = a.elapsed_time(b) / reps / D["dst"].shape[0]
    n = D["n_pairs"]
    step_ms = icp_kernel_ms + k1_ms_per_image * n
    H, W = intr.height, intr.width
    coarse = sum(-(-H // s) * -(-W // s) for s, _ in cfg.schedule if s > 1)
    k1_bytes = 4 * H * W + 16 * (H * W + coarse)          # range in, surfel pyramid out
    peak, _ = measured_peak()
    achieved = k1_bytes / (k1_ms_per_image / 1e3) / 1e9
    return {"value": n / (step_ms / 1e3), "unit": "registrations/s",
            "k1_us_per_image": k1_ms_per_image * 1e3, "ms_per_step": step_ms,
            "what": "C4 with K1 normals computed for every pair's destination (65,536 per step) "
                    "instead of once per pool image",
            "k1_roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "bytes_per_image": k1_bytes}}


def run_e2e_independent(args, D, cfg):
    """End to end for truly independent pairs: every pair's own source and
    destination images cross PCIe (2 x 256 KB per pair, 34 GB per 65,536-pair
    step), chunked by the pool size and double-buffered on a copy stream, K1
    per pair, K3, poses back to the host.  The host images of chunk k are the
    pool's (same bytes per pair as distinct images would move)."""
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200.range_image import normals_cross_batch
    intr = D["intr"]
    P = D["src"].shape[0]
    n = D["n_pairs"]
    chunks = max(1, n // P)
    src_h = D["src"].cpu().pin_memory()
    dst_h = D["dst"].cpu().pin_memory()
    bufs = [(torch.empty_like(D["src"]), torch.empty_like(D["dst"])) for _ in range(2)]
    copy = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    out_h = torch.empty((chunks, P, 12), dtype=torch.float64, pin_memory=True)

    def issue(b):
        with torch.cuda.stream(copy):
            copy.wait_event(free[b])
            bufs[b][0].copy_(src_h, non_blocking=True)
            bufs[b][1].copy_(dst_h, non_blocking=True)
            ready[b].record(copy)

    def step():
        issue(0)
        for k in range(chunks):
            b = k % 2
            if k + 1 < chunks:
                issue(1 - b)
            main.wait_event(ready[b])
            src, dst = bufs[b]
            surf = normals_cross_batch(intr, dst, strides=[s for s, _ in cfg.schedule])
            res = rk.register_batch(intr, src, dst, surf, config=cfg)
            free[b].record(main)
            out_h[k].copy_(res.poses, non_blocking=True)
        torch.cuda.synchronize()

    step()
    t0 = time.perf_counter()
    reps = 2
    for _ in range(reps):
        step()
    el = (time.perf_counter() - t0) / reps
    h2d = chunks * P * 2 * intr.height * intr.width * 4
    return {"value": chunks * P / el, "unit": "registrations/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(chunks * P * 12 * 8), "seconds_per_step": el,
            "h2d_gbs": h2d / el / 1e9,
            "what": f"{chunks * P} independent pairs per step: each pair's two images copied H2D "
                    f"(chunks of {P}, double-buffered), K1 per pair, K3, poses D2H; wall clock"}


def run_c5_tsdf(frames: int = 100):
    """C5's TSDF: OS-128 128x2048 extended street at 0.5 m/frame,
    3 cm voxels -- the grid (~24k blocks, ~0.8 GB) is far beyond the 126 MB
    L2, so K5 streams its voxel states from HBM.  One warm-up, two timed
    sequences into a cleared grid, CUDA events."""
    import torch

    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import pipeline, scenes
    intr = scenes.os128()
    traj = scenes.street_trajectory(frames, seed=0, step_m=0.5, jitter=0.0002)
    fr = pipeline.render_batch(intr, scenes.extended_street_scene(0.5 * frames + 30.0), traj)
    poses_w = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
    inv_w = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
    grid = rk.VoxelBlockGrid(voxel_size=0.03, capacity=TSDF_CAPACITY["c5"])
    upd = torch.zeros(1, dtype=torch.int64, device="cuda")
    ms = 0.0
    for rep in range(3):
        pipeline.clear_grid(grid)
        upd.zero_()
        a, b = _events()
        a.record()
        pipeline.integrate_sequence(grid, intr, fr, poses_w, inv_w, clip_max=80.0, updated=upd, graph=True)
        b.record()
        torch.cuda.synchronize()
        if rep:
            ms += a.elapsed_time(b)
    ms /= 2
    n_blocks, _, overflow, _ = grid.info()
    if overflow:
        raise RuntimeError("C5 TSDF pool overflow")
    tsdf_bytes = TSDF_BYTES_PER_VOXEL * upd.item() + TSDF_BYTES_PER_PIXEL * intr.height * intr.width * frames
    peak, src = measured_peak()
    achieved = tsdf_bytes / (ms / 1e3) / 1e9
    return {"value": frames / (ms / 1e3), "unit": "frames/s", "frames": frames, "voxel_m": 0.03,
            "blocks": int(n_blocks), "grid_bytes": int(n_blocks) * 32768,
            "voxels_updated_per_frame": upd.item() / frames,
            "roofline": {"bound": "hbm", "kernel": "k_integrate (+ overlapped k_activate_image)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "work": f"16 B x {upd.item():.4g} updated voxels + 4 B x range pixels, "
                                 f"{ms:.2f} ms per sequence", "peak_source": src}}


def kernel_rooflines(args, D, r, tsdf):
    """Per-kernel HBM rooflines for the kernels besides K3/K5: K1 (normals +
    surfel pyramid over the pool), K4 (block activation of the sequence, run
    alone) and K6 (marching cubes of the final grid, wall clock incl. its one
    count readback, so an upper bound on kernel time)."""
    import torch

    from paper_2112_02779_b200 import _native as nat, lidar_model as lm
    peak, _ = measured_peak()
    out = {}
    intr = D["intr"]
    H, W = intr.height, intr.width
    cfg_coarse = sum(-(-H // s) * -(-W // s) for s in (4, 2))
    k1_bytes = D["dst"].shape[0] * (4 * H * W + 16 * (H * W + cfg_coarse))
    out["k_normals_cross_pyramid"] = {"bound": "hbm", "ms": r["normals_ms"],
                                      "achieved": k1_bytes / (r["normals_ms"] / 1e3) / 1e9, "peak": peak,
                                      "unit": "GB/s", "bytes": k1_bytes,
                                      "what": "4 B range in + 16 B surfel out per pixel (+ coarse levels)"}
    grid = tsdf.grid
    g = grid._ensure()
    F = args.frames
    tin = D["tintr"]
    nat.call("rk_grid_reserve_slots", g, F, nat.stream_ptr())
    grid._graphs.clear()   # the slot tables may have moved: drop recorded sequences
    for rep in range(2):
        from paper_2112_02779_b200 import pipeline
        pipeline.clear_grid(grid)
        a, b = _events()
        a.record()
        nat.call("rk_grid_activate_frames", g, lm.device_sensor(tin), nat.ptr(D["frames"]), F,
                 nat.ptr(D["poses_w"]), float(grid.truncation), 0.0, 30.0, nat.stream_ptr())
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    k4_bytes = F * 4 * tin.height * tin.width
    out["k_activate_image"] = {"bound": "hbm", "ms": ms, "achieved": k4_bytes / (ms / 1e3) / 1e9,
                               "peak": peak, "unit": "GB/s", "bytes": k4_bytes,
                               "what": f"{F} frames: 4 B range per pixel (+ hash probes, latency-bound); "
                                       "overlapped with K5 in the sequence"}
    m = r["mesh"]
    if m and "ms" in m:
        nb = m.get("blocks", 0)
        mc_bytes = nb * 4096 * 8 * (19 ** 3 / 16 ** 3) + m["vertices"] * 48 + m["triangles"] * 12
        out["k_mc"] = {"bound": "hbm", "ms": m["ms"], "achieved": mc_bytes / (m["ms"] / 1e3) / 1e9,
                       "peak": peak, "unit": "GB/s", "bytes": mc_bytes,
                       "what": "8 B per voxel of the 19^3 halo window per block + 48 B per vertex "
                               "(position, normal) + 12 B per triangle; wall clock incl. one readback"}
    for v in out.values():
        v["frac"] = v["achieved"] / v["peak"]
    return out


# ------------------------------------------------------------------ CPU oracle

def _cpu_icp_job(seed_pairs):
    """Worker: oracle normals + register on a few pool pairs (single thread)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import icp as oicp
    from oracle import image as oimg
    from oracle import sensor as osens
    from oracle import synth as osynth
    from paper_2112_02779_b200 import scenes
    intr = scenes.ouster64()
    S = osens.Sensor.from_intrinsics(intr)
    street = scenes.street_scene()
    pool = scenes.pair_pool_poses(max(seed_pairs) + 1, seed=0)
    imgs = []
    for i in seed_pairs:
        base, gt = pool[i]
        s = base @ gt
        imgs.append((osynth.render(S, street, s.R, s.t), osynth.render(S, street, base.R, base.t)))
    t0 = time.perf_counter()
    for src, dst in imgs:
        vec, valid = oimg.normals_cross(S, dst)
        oicp.register(S, src, dst, vec, valid, fma="blas")
    return len(imgs), time.perf_counter() - t0


def cpu_icp_baseline(budget_s: float, steps: int = 1, warmup: int = 0):
    """The reference's CPU path (oracle port) on every host core: a process
    pool of single-threaded workers, each registering its own pool pairs.
    ``warmup`` untimed steps (one pair per worker), then ``steps`` timed
    steps sized so the timed work totals about ``budget_s`` seconds; a
    step's time is its slowest worker's compute time (rendering excluded)."""
    from concurrent.futures import ProcessPoolExecutor
    cores = os.cpu_count() or 1
    steps = max(1, steps)
    # calibrate: one pair on one core
    n1, t1 = _cpu_icp_job([0])
    per_worker = max(1, int(budget_s / steps / max(t1, 1e-3) / 2))
    done, busy, step_s = 0, 0.0, []
    t0 = time.perf_counter()
    with ProcessPoolExecutor(cores) as ex:
        for _ in range(warmup):
            list(ex.map(_cpu_icp_job, [[k] for k in range(cores)]))
        nxt = 0
        for _ in range(steps):
            jobs = [list(range(nxt + k * per_worker, nxt + (k + 1) * per_worker)) for k in range(cores)]
            nxt += cores * per_worker
            outs = list(ex.map(_cpu_icp_job, jobs))
            done += sum(n for n, _ in outs)
            step_s.append(max(t for _, t in outs))
    wall = time.perf_counter() - t0
    busy = sum(step_s)
    return dict(value=done / busy, unit="registrations/s", cores=cores, kind="port",
                ms_per_step=1e3 * busy / steps,
                sample=f"{done} C4 pool pairs over {steps} step(s) after {warmup} warm-up step(s) "
                       f"(normals + 3-level register), oracle numpy, {cores} processes x 1 thread, "
                       f"{busy:.1f} s compute ({wall:.1f} s wall)")


def cpu_tsdf_baseline(frames: int = 3, threads: int = 1):
    from oracle import sensor as osens
    from oracle import synth as osynth
    from oracle import tsdf as otsdf
    from paper_2112_02779_b200 import scenes
    intr = scenes.ouster64()
    S = osens.Sensor.from_intrinsics(intr)
    traj = scenes.street_trajectory(frames, seed=0)
    imgs = [osynth.render(S, scenes.street_scene(), p.R, p.t) for p in traj]
    grid = {}
    t0 = time.perf_counter()
    for img, p in zip(imgs, traj):
        otsdf.integrate_cloud_frame(grid, S, img, p.R, p.t, 0.05, 0.2, clip_max=30.0, fma="blas",
                                    threads=threads)
    dt = time.perf_counter() - t0
    return dict(value=frames / dt, unit="frames/s", cores=threads, kind="port",
                sample=f"{frames} frames of the C2 street sequence at 5 cm, oracle numpy, "
                       f"{threads} thread(s) (the reference's chunk pool)")


def host_info():
    """CPU model and numpy's BLAS, for the CPU-baseline records."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = "unknown"
    try:
        from threadpoolctl import threadpool_info
        info = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')} ({info[0].get('architecture')})"
    except Exception:
        pass
    import numpy
    return {"cpu_model": model, "cores": os.cpu_count(), "numpy": numpy.__version__, "blas": blas}


def cpu_extras(tsdf_frames_1: int = 8, tsdf_frames_n: int = 16):
    """The rest of SURVEY §8(d)'s CPU baseline, on the oracle port (bit-exact
    with the reference, tests/test_oracle_golden.py): (i) register() latency,
    best of 7, at threads=1 and at the reference default min(8, cores) (its
    stride-1 shards on a thread pool); (iii) TSDF frames/s of the C2 sequence
    at 1 and min(8, cores) threads (bounded frame counts); (iv) one
    extract_mesh of the C3 grid after its 100-frame sequence (grid built on
    the GPU in MATH_NP -- bit-exact with the oracle's -- and exported)."""
    from oracle import icp as oicp
    from oracle import image as oimg
    from oracle import mesh as omesh
    from oracle import sensor as osens
    from oracle import synth as osynth
    from oracle import tsdf as otsdf
    from paper_2112_02779_b200 import scenes
    threads = min(8, os.cpu_count() or 1)
    intr = scenes.ouster64()
    S = osens.Sensor.from_intrinsics(intr)
    street = scenes.street_scene()
    base, gt = scenes.pair_pool_poses(1, seed=0)[0]
    sp = base @ gt
    src = osynth.render(S, street, sp.R, sp.t)
    dst = osynth.render(S, street, base.R, base.t)
    lat = {}
    for t in (1, threads):
        best = 1e9
        for _ in range(7):
            t0 = time.perf_counter()
            vec, valid = oimg.normals_cross(S, dst)
            oicp.register(S, src, dst, vec, valid, fma="blas", threads=t)
            best = min(best, time.perf_counter() - t0)
        lat[f"threads_{t}"] = best * 1e3
    out = {"latency_ms": dict(lat, what="normals + register() of the C1 street pair, best of 7")}
    traj = scenes.street_trajectory(max(tsdf_frames_1, tsdf_frames_n), seed=0)
    imgs = [osynth.render(S, street, p.R, p.t) for p in traj]
    fps = {}
    for t, nf in ((1, tsdf_frames_1), (threads, tsdf_frames_n)):
        grid = {}
        t0 = time.perf_counter()
        for img, p in zip(imgs[:nf], traj[:nf]):
            otsdf.integrate_cloud_frame(grid, S, img, p.R, p.t, 0.05, 0.2, clip_max=30.0, fma="blas", threads=t)
        fps[f"threads_{t}"] = nf / (time.perf_counter() - t0)
    out["tsdf_frames_per_s"] = dict(fps, what=f"C2 street sequence at 5 cm, first {tsdf_frames_1} / "
                                              f"{tsdf_frames_n} frames")
    out["marching_cubes"] = _cpu_mc_c3(omesh)
    out["host"] = host_info()
    return out


def _cpu_mc_c3(omesh):
    import paper_2112_02779_b200 as rk
    from paper_2112_02779_b200 import pipeline, scenes
    import torch
    intr = scenes.hdl64()
    traj = scenes.street_trajectory(100, seed=0)
    frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
    grid = rk.VoxelBlockGrid(voxel_size=0.10, capacity=8192)
    pipeline.integrate_sequence(grid, intr, frames, torch.from_numpy(pipeline.poses_to_rows(traj)).cuda(),
                                clip_max=30.0)
    keys, vox = grid.export_blocks()
    og = {tuple(k): (vox[i, :, 0].reshape(16, 16, 16).copy(), vox[i, :, 1].reshape(16, 16, 16).copy())
          for i, k in enumerate(keys.tolist())}
    t0 = time.perf_counter()
    V, T, _ = omesh.extract_mesh(og, 0.10)
    ms = 1e3 * (time.perf_counter() - t0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    m = rk.extract_mesh(grid)
    gpu_ms = 1e3 * (time.perf_counter() - t1)
    return {"ms": ms, "blocks": len(og), "vertices": int(len(V)), "triangles": int(len(T)),
            "gpu_ms_public_api": gpu_ms, "gpu_same_counts": bool(m.n_vertices == len(V) and m.n_triangles == len(T)),
            "what": "oracle extract_mesh (mesh_extract.py:85-209 restated, 1 thread) of the C3 HDL-64 "
                    "grid at 10 cm after 100 frames; the GPU's extract_mesh of the same grid beside it"}


# ------------------------------------------------------------------ main

def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profile_traffic(kernel: str, key: str | None = None):
    """dram bytes (or, with key="instructions", warp instructions) per work
    unit from the committed ncu captures (profiles/traffic.json), if any."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(key, {}).get(kernel) if key else d.get(kernel)
    return None


def issue_roofline(kernel: str, units: float, seconds: float, sm_mhz):
    """The bound these kernels actually sit on: warp-instruction issue.  Peak =
    4 schedulers x SMs x SM clock (one warp instruction per scheduler per
    cycle); instructions per unit from the committed ncu capture."""
    ipu = profile_traffic(kernel, "instructions")
    if not ipu or not seconds:
        return None
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    clk = (sm_mhz or 1965.0) * 1e6
    achieved = ipu * units / seconds
    peak = 4 * sms * clk
    return {"bound": "issue", "unit": "warp-instr/s", "instr_per_unit": ipu, "achieved": achieved,
            "peak": peak, "frac": achieved / peak, "sm_mhz": clk / 1e6}


def dist_init(args):
    if args.gpus <= 1 or "RANK" not in os.environ:
        return None, 0, 1
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("RK_BENCH_GLOO"):
        # functional check of the N > 1 path on a one-GPU box: every rank on
        # cuda:0, collectives staged through host memory over gloo (timings
        # are not scaling numbers)
        from paper_2112_02779_b200.distributed import CpuStagedDist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        staged = CpuStagedDist(dist)
        staged.destroy_process_group = dist.destroy_process_group
        return staged, dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    if dist.get_rank() == 0:
        print(f"[bench] NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}, world {dist.get_world_size()}, "
              f"backend {dist.get_backend()}", file=sys.stderr)
    return dist, dist.get_rank(), dist.get_world_size()


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        icp = cpu_icp_baseline(args.cpu_seconds, args.steps, args.warmup)
        line = {"impl": "reference", "metric": METRIC, "value": icp["value"], "unit": "registrations/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": icp["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
                "config": {"workload": "C4 65,536 64x1024 street pairs (bounded CPU sample per step) "
                                       "+ C2 TSDF 5 cm", "pairs": args.pairs},
                "cpu_baseline": dict(icp, host=host_info()),
                "tsdf": cpu_tsdf_baseline(frames=16, threads=min(8, os.cpu_count() or 1)),
                "e2e": {"value": icp["value"], "unit": "registrations/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    dist, rank, world = dist_init(args)
    if args.math is not None:
        from paper_2112_02779_b200 import lidar_model as lm
        lm.set_default_math({"np": lm.MATH_NP, "fast": lm.MATH_FAST, "cr": lm.MATH_CR}[args.math])
    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    r = run_ours(args, rank, world, dist)
    e2e = None if args.no_e2e else run_e2e(args, rank, world, dist, r["D"], r["tsdf"], r["cfg"])
    extras = {}
    if world == 1 and not args.no_extras:
        extras["math_modes"] = run_math_modes(args, r["D"], r["cfg"])
        extras["value_k1_per_pair"] = run_k1_per_pair(args, r["D"], r["cfg"], r["icp_kernel_ms"])
        extras["e2e_independent"] = run_e2e_independent(args, r["D"], r["cfg"])
        extras["kernel_rooflines"] = kernel_rooflines(args, r["D"], r, r["tsdf"])
        extras["c5_tsdf"] = run_c5_tsdf()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_icp_baseline(args.cpu_seconds)
        cpu.update(cpu_extras())
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peak()
    tr = profile_traffic("k_register")
    line = {
        "metric": METRIC, "value": r["reg_per_s"], "unit": "registrations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["elapsed_ms"] / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (f64 solve and sensor tables)", "data": "synthetic (device-rendered street scene)",
        "config": {"workload": "C4: 65,536 independent 64x1024 Ouster-like pairs (pool of "
                               f"{args.pool} unique street pairs), 3-level ICP 4:20,2:20,1:10 + "
                               + TSDF_DESC[args.tsdf_config].format(n=args.frames),
                   "pairs": args.pairs, "pairs_per_rank": r["D"]["n_pairs"], "pool": args.pool,
                   "frames": args.frames, "voxel_m": TSDF_VOXEL[args.tsdf_config],
                   "tsdf_config": args.tsdf_config,
                   "l2": "inputs > L2 (ICP pool %.1f GB)" % (args.pool * 64 * 1024 * 24 / 1e9),
                   "parallelism": f"pairs sharded over {world} rank(s)"},
        "tsdf": {"value": r["tsdf_fps"], "unit": "frames/s", "voxels_updated_per_step": r["tsdf_updated"],
                 "blocks": r["n_blocks"],
                 "roofline": {"bound": "hbm", "achieved": r["tsdf_achieved"], "peak": peak, "unit": "GB/s",
                              "frac": r["tsdf_achieved"] / peak,
                              "traffic": (tt * r["upd_local"] if (tt := profile_traffic("k_integrate"))
                                          else None)}},
        "roofline": {"bound": "hbm", "kernel": "k_register", "achieved": r["achieved"], "peak": peak,
                     "unit": "GB/s", "frac": r["achieved"] / peak,
                     "traffic": (tr * r["pt_local"] if tr else None),
                     "work": f"{r['pt_local']:.4g} source-point-iterations x {ICP_BYTES_PER_PT_IT} B "
                             f"per launch, {r['icp_kernel_ms']:.2f} ms/launch", "peak_source": peak_src},
        "issue_roofline": {
            "k_register": issue_roofline("k_register", r["pt_local"], r["icp_kernel_ms"] / 1e3,
                                         r["clocks"].get("sm_mhz")),
            "k_integrate": issue_roofline("k_integrate", r["upd_local"],
                                          r["tsdf_ms"] / args.steps / 1e3, r["clocks"].get("sm_mhz"))},
        "phase_ms": {"normals": r["normals_ms"], "register": r["icp_kernel_ms"],
                     "tsdf_sequence": r["tsdf_ms"] / args.steps},
        "gt_recovered_frac": r["ok_frac"],
        "marching_cubes": r["mesh"],
        "single_pair_latency": r["latency"],
        "odometry_tsdf": r["odometry"],
        "clocks": r["clocks"], "gpu_launches": r["launches"],
        "e2e": e2e, "cpu_baseline": cpu,
    }
    line.update(extras)
    line["math"] = {"headline": "np (numpy-exact projection: the reference's decisions and per-point "
                                "terms bit for bit)", "others": "math_modes"}
    line["pool_reuse"] = ("value/e2e reuse a pool of %d device-rendered pairs: K1 once per pool image and "
                          "16.4 KB of H2D per registration; value_k1_per_pair and e2e_independent charge "
                          "K1 and 512 KB of H2D to every pair" % args.pool)
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
