import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
from paper_2112_02779_b200.mesh_extract import extract_mesh_device
intr = scenes.ouster64()
traj = scenes.street_trajectory(100, seed=0)
frames = pipeline.render_batch(intr, scenes.street_scene(), traj)
poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
for cap in (32768, 65536):
    grid = rk.VoxelBlockGrid(voxel_size=0.05, capacity=cap)
    pipeline.integrate_sequence(grid, intr, frames, poses, clip_max=30.0)
    torch.cuda.synchronize()
    ts = []
    for i in range(5):
        t = time.perf_counter(); v, tri, n = extract_mesh_device(grid); torch.cuda.synchronize(); ts.append(1e3*(time.perf_counter()-t))
    print(cap, grid.info()[0], [round(x, 2) for x in ts], v.shape[0])
