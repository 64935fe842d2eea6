"""Diagnostic: per-frame time of the C2 TSDF sequence (100 frames, 5 cm)
(a) through the overlapped pipeline (rk_grid_integrate_frames), and
(b) split: all activations first (rk_grid_activate_frames into F slots),
then the F integrations back to back (rk_grid_integrate_activated) -- (b)'s
second phase is the K5-only time per frame."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2112_02779_b200 as rk  # noqa: E402
from paper_2112_02779_b200 import _native as nat, lidar_model as lm, pipeline, scenes  # noqa: E402

F = 100
intr = scenes.ouster64()
traj = scenes.street_trajectory(F, seed=0)
frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
inv = torch.from_numpy(np.stack([p.inverse().as_row12() for p in traj])).cuda()
sensor = lm.device_sensor(intr)
st = nat.stream_ptr()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

g = rk.VoxelBlockGrid(voxel_size=0.05, capacity=65536)
upd = nat.zeros((1,), np.int64)
for rep in range(4):
    pipeline.clear_grid(g)
    ev[0].record()
    pipeline.integrate_sequence(g, intr, frames, poses, inv, clip_max=30.0, updated=upd, graph=True)
    ev[1].record()
    torch.cuda.synchronize()
print(f"(a) overlapped pipeline: {ev[0].elapsed_time(ev[1]) / F * 1e3:.1f} us/frame")

h = g._ensure()
nat.call("rk_grid_reserve_slots", h, F, st)
for rep in range(4):
    pipeline.clear_grid(g)
    ev[0].record()
    nat.call("rk_grid_activate_frames", h, sensor, nat.ptr(frames), F, nat.ptr(poses), float(g.truncation),
             0.0, 30.0, st)
    ev[1].record()
    nat.call("rk_grid_integrate_activated", h, sensor, nat.ptr(frames), F, nat.ptr(inv), None, 0.0, 30.0,
             lm.default_math(), nat.ptr(upd), st)
    ev[2].record()
    torch.cuda.synchronize()
print(f"(b) activations {ev[0].elapsed_time(ev[1]) / F * 1e3:.1f} us/frame, "
      f"integrations back to back {ev[1].elapsed_time(ev[2]) / F * 1e3:.1f} us/frame")
