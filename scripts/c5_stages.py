import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2112_02779_b200 as rk
from paper_2112_02779_b200 import pipeline, scenes
from paper_2112_02779_b200.mesh_extract import extract_mesh_device
F = int(sys.argv[1])
intr = scenes.os128()
t = time.perf_counter()
traj = scenes.street_trajectory(F, seed=0, step_m=0.5, jitter=float(__import__('os').environ.get('JITTER', '0.0002')))
frames = pipeline.render_batch(intr, scenes.extended_street_scene(0.5 * F + 30.0), traj); torch.cuda.synchronize()
print('render', time.perf_counter() - t, flush=True); t = time.perf_counter()
g = rk.VoxelBlockGrid(voxel_size=0.03, capacity=262144)
poses = torch.from_numpy(pipeline.poses_to_rows(traj)).cuda()
upd = pipeline.integrate_sequence(g, intr, frames, poses, clip_max=30.0); torch.cuda.synchronize()
print('tsdf', time.perf_counter() - t, g.info(), flush=True); t = time.perf_counter()
v, tri, _ = extract_mesh_device(g); torch.cuda.synchronize()
print('mc', time.perf_counter() - t, v.shape, tri.shape, flush=True); t = time.perf_counter()
w, res = pipeline.odometry(intr, frames); torch.cuda.synchronize()
print('odometry', time.perf_counter() - t, flush=True)
