"""Generate golden input/output vectors by running the UNMODIFIED reference.

Runs only in the build container (needs /root/reference); the resulting
``tests/golden/*.npz`` files are committed and travel to the GPU box.

    PYTHONDONTWRITEBYTECODE=1 RANGEKIT_THREADS=1 python tests/golden/make_golden.py

RANGEKIT_THREADS=1 makes register() use one shard (registration.py:292-296),
the schedule the oracle restates.  Inputs are rendered by the reference's own
synth.render_scene from the seeded definitions in paper_2112_02779_b200/scenes.py.
"""

from __future__ import annotations

import os
import sys
from itertools import product
from pathlib import Path

os.environ.setdefault("RANGEKIT_THREADS", "1")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))

import numpy as np  # noqa: E402

import rangekit as rk  # noqa: E402  (the reference)
from rangekit import mc_tables, mesh_extract, registration, sdf_volume  # noqa: E402
from rangekit.range_image import compute_normal_map, points_at_stride, to_point_cloud  # noqa: E402
from rangekit.synth import Box, Plane, Sphere, render_scene  # noqa: E402

from paper_2112_02779_b200 import scenes  # noqa: E402  (input definitions only)


def ref_intr(intr):
    """Rebuild a package LidarIntrinsics as the reference's class."""
    return rk.LidarIntrinsics(width=intr.width, height=intr.height,
                              receiver_radius=intr.receiver_radius,
                              azimuth_lut=intr.azimuth_lut, elevation_lut=intr.elevation_lut,
                              mode=intr.mode)


def ref_scene(prims):
    out = []
    for p in prims:
        if p[0] == "box":
            out.append(Box(center=p[1], size=p[2]) if p[3] is None else
                       Box(center=p[1], size=p[2], rotation=p[3]))
        elif p[0] == "sphere":
            out.append(Sphere(center=p[1], radius=p[2]))
        else:
            out.append(Plane(normal=p[1], offset=p[2]))
    return out


def ref_pose(pose):
    return rk.RigidTransform(pose.R, pose.t)


def sensors():
    return {"small": scenes.small_calib(), "synth": scenes.synth_intr(),
            "ouster": scenes.ouster64()}


def gen_sensor_and_projection():
    out = {}
    g = np.random.default_rng(100)
    for name, intr in sensors().items():
        ri = ref_intr(intr)
        out[f"{name}/inv_rows"] = ri.inv_elevation_lut.rows
        out[f"{name}/fov"] = np.array(ri.fov_bounds)
        if name != "ouster":
            out[f"{name}/dirs"] = ri.ray_dirs
            out[f"{name}/origins"] = ri.ray_origins
        # points in a shell around the sensor, some inside r0 / outside fov
        n = 20000
        d = g.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        d[:, 2] *= 0.4
        r = g.uniform(0.01, 40.0, n)
        pts = d * r[:, None]
        pts[:50] *= 1e-3  # degenerate (inside the receiver cylinder)
        pts32 = pts.astype(np.float32)
        u, v, rr, st = rk.project_many(pts32, ri, single=True, refine=False)
        out[f"{name}/p32_in"], out[f"{name}/p32_u"], out[f"{name}/p32_v"] = pts32, u, v
        out[f"{name}/p32_r"], out[f"{name}/p32_st"] = rr, st
        u, v, rr, st = rk.project_many(pts[:5000], ri)
        out[f"{name}/p64_in"], out[f"{name}/p64_u"], out[f"{name}/p64_v"] = pts[:5000], u, v
        out[f"{name}/p64_r"], out[f"{name}/p64_st"] = rr, st
        lo, hi = ri.fov_bounds
        phi = g.uniform(lo - 0.05, hi + 0.05, 5000)
        out[f"{name}/phi64"] = phi
        out[f"{name}/row64"] = ri.row_from_elevation(phi)
        out[f"{name}/phi32"] = phi.astype(np.float32)
        out[f"{name}/row32"] = ri.row_from_elevation(phi.astype(np.float32))
        out[f"{name}/lookup64"] = ri.inv_elevation_lut.lookup(phi)
    np.savez_compressed(OUT / "sensor_projection.npz", **out)


def render_pairs():
    """dst at identity, src at a seeded perturbation (the reference convention)."""
    pairs = {}
    small = sensors()["small"]
    rs = ref_intr(small)
    room = ref_scene(scenes.room_scene())
    gt = scenes.perturbation_pose(np.random.default_rng(3), 2.0, 0.2)
    pairs["room"] = (small, rs, render_scene(room, rs, ref_pose(gt)).data,
                     render_scene(room, rs).data, gt)
    ous = sensors()["ouster"]
    ro = ref_intr(ous)
    street = ref_scene(scenes.street_scene())
    gt2 = scenes.perturbation_pose(np.random.default_rng(1), 2.0, 0.3)
    pairs["street"] = (ous, ro, render_scene(street, ro, ref_pose(gt2)).data,
                       render_scene(street, ro).data, gt2)
    syn = sensors()["synth"]
    ry = ref_intr(syn)
    gt3 = scenes.perturbation_pose(np.random.default_rng(12), 5.0, 0.5)
    noisy = render_scene(room, ry, noise_std=0.01, seed=4).data
    pairs["synth"] = (syn, ry, render_scene(room, ry, ref_pose(gt3)).data, noisy, gt3)
    return pairs


def gen_images_icp(pairs):
    out = {}
    for name, (intr, ri, src, dst, gt) in pairs.items():
        out[f"{name}/src"], out[f"{name}/dst"] = src, dst
        out[f"{name}/gt"] = gt.matrix()
        dimg, simg = rk.RangeImage(dst, ri), rk.RangeImage(src, ri)
        nm = compute_normal_map(dimg)
        out[f"{name}/nrm"], out[f"{name}/nvalid"] = nm.vectors, nm.valid
        big = name == "street"  # keep the committed fixtures small
        if not big:
            out[f"{name}/cloud"] = to_point_cloud(simg, clip_min=0.5, clip_max=20.0)
            for s in (1, 2, 4):
                out[f"{name}/pts_s{s}"] = points_at_stride(simg, s)
        pose = rk.RigidTransform(gt.R, gt.t * 0.9)
        src_pts = to_point_cloud(simg)
        out[f"{name}/corr_pose"] = pose.matrix()
        for s in ((4,) if big else (1, 2, 4)):
            c = registration.projective_correspondences(src_pts, dimg, nm, pose, 0.5 * s, s,
                                                        single=True)
            out[f"{name}/c32_s{s}_sel"] = rows_of(src_pts, c.source)
            out[f"{name}/c32_s{s}_tgt"] = c.target
            out[f"{name}/c32_s{s}_nrm"] = c.normal
        sub = src_pts[::7] if big else src_pts[::2]
        c = registration.projective_correspondences(sub, dimg, nm, pose, 0.5, 1)
        out[f"{name}/c64_sel"] = rows_of(sub, c.source)
        out[f"{name}/c64_tgt"], out[f"{name}/c64_nrm"] = c.target, c.normal
        res = registration.register(simg, dimg, dst_normals=nm)
        out[f"{name}/reg_pose"] = res.pose.matrix()
        out[f"{name}/reg_converged"] = np.array(res.converged)
        out[f"{name}/reg_stats"] = np.array([[s.stride, s.iteration, s.n_correspondences, s.cost,
                                              s.inlier_rmse] for s in res.stats])
        init = registration.initial_translation_by_centroids(to_point_cloud(simg), to_point_cloud(dimg))
        out[f"{name}/centroid_t"] = init.t
    np.savez_compressed(OUT / "images_icp.npz", **out)


def rows_of(cloud, subset):
    """Indices of subset's rows inside cloud (rows are unique; order kept)."""
    index = {tuple(r): i for i, r in enumerate(cloud.tolist())}
    return np.array([index[tuple(r)] for r in subset.tolist()], dtype=np.int32)


def grid_arrays(grid):
    keys = sorted(grid.blocks)
    vox = np.stack([np.stack([grid.blocks[k].tsdf.reshape(-1), grid.blocks[k].weight.reshape(-1)], -1)
                    for k in keys]) if keys else np.zeros((0, 4096, 2), np.float32)
    return np.array(keys, dtype=np.int32).reshape(-1, 3), vox.astype(np.float32)


def gen_tsdf(pairs):
    out = {}
    g = np.random.default_rng(21)
    pts = g.uniform(-4.0, 4.0, size=(50, 3))
    grid = sdf_volume.VoxelBlockGrid(voxel_size=0.1)
    keys = sdf_volume.activate_blocks(pts, grid, 0.55)
    out["act_pts"], out["act_keys"] = pts, np.array(sorted(keys), dtype=np.int32)
    # a short posed sequence on the small sensor (room scene), 3 frames, 0.2 m voxels
    small, rs = sensors()["small"], ref_intr(sensors()["small"])
    room = ref_scene(scenes.room_scene())
    poses = [scenes.perturbation_pose(np.random.default_rng(40 + i), 3.0, 0.3) for i in range(3)]
    frames = [render_scene(room, rs, ref_pose(p)).data for p in poses]
    grid = sdf_volume.VoxelBlockGrid(voxel_size=0.2)
    counts = []
    for f, p in zip(frames, poses):
        counts.append(sdf_volume.integrate_cloud_frame(grid, rk.RangeImage(f, rs), ref_pose(p),
                                                       clip_max=12.0))
    k, v = grid_arrays(grid)
    out["seq_frames"] = np.stack(frames)
    out["seq_poses"] = np.stack([p.matrix() for p in poses])
    out["seq_counts"], out["seq_keys"], out["seq_vox"] = np.array(counts), k, v
    # one Ouster street frame at 5 cm: key set + per-block checksums + sample blocks
    _, ro, _, dst, _ = pairs["street"]
    grid = sdf_volume.VoxelBlockGrid(voxel_size=0.05)
    n = sdf_volume.integrate_cloud_frame(grid, rk.RangeImage(dst, ro), rk.RigidTransform.identity(),
                                         clip_max=30.0)
    k, v = grid_arrays(grid)
    out["street_count"], out["street_keys"] = np.array(n), k
    out["street_tsdf_sum"] = v[..., 0].astype(np.float64).sum(axis=1)
    out["street_weight_sum"] = v[..., 1].astype(np.float64).sum(axis=1)
    pick = np.random.default_rng(5).choice(len(k), size=min(24, len(k)), replace=False)
    out["street_pick"], out["street_pick_vox"] = pick, v[pick]
    # queries on the small sequence grid
    q = g.uniform(-3, 3, size=(400, 3))
    gseq = sdf_volume.VoxelBlockGrid(voxel_size=0.2)
    for f, p in zip(frames, poses):
        sdf_volume.integrate_cloud_frame(gseq, rk.RangeImage(f, rs), ref_pose(p), clip_max=12.0)
    s, w, ok = sdf_volume.query_sdf_many(gseq, q)
    out["q_pts"], out["q_sdf"], out["q_w"], out["q_ok"] = q, s, w, ok
    np.savez_compressed(OUT / "tsdf.npz", **out)


def gen_mesh():
    out = {"tri_table": mc_tables.TRI_TABLE, "edge_table": mc_tables.EDGE_TABLE}
    grid = sdf_volume.VoxelBlockGrid(voxel_size=0.05, truncation=0.2)
    ext = grid.block_extent
    for key in product(range(int(np.floor(-0.8 / ext)), int(np.floor(0.8 / ext)) + 1), repeat=3):
        blk = sdf_volume.VoxelBlock()
        c = grid.voxel_centers(key)
        vals = np.clip(np.linalg.norm(c, axis=1) - 0.6, -0.2, 0.2)
        blk.tsdf = vals.reshape(16, 16, 16).astype(np.float32)
        blk.weight = np.full((16, 16, 16), 1.0, np.float32)
        grid.blocks[key] = blk
    k, v = grid_arrays(grid)
    m = mesh_extract.extract_mesh(grid)
    out["sphere_keys"], out["sphere_vox"] = k, v
    out["sphere_V"], out["sphere_T"], out["sphere_N"] = m.vertices, m.triangles, m.normals
    np.savez_compressed(OUT / "mesh.npz", **out)


def gen_next(pairs):
    """N1 from_point_cloud, N2 SDFG / PLY bytes, N3 PCA normals."""
    import tempfile

    from rangekit import io_formats
    from rangekit.range_image import from_point_cloud
    out = {}
    g = np.random.default_rng(77)
    for name in ("room", "street"):
        intr, ri, src, dst, gt = pairs[name]
        cloud = to_point_cloud(rk.RangeImage(dst, ri))
        pick = g.choice(cloud.shape[0], size=min(12000, cloud.shape[0]), replace=False)
        pts = cloud[pick] + g.normal(scale=0.004, size=(len(pick), 3))
        dup = pts[:1500] + g.normal(scale=0.002, size=(1500, 3))      # pixel collisions
        extra = np.array([[0.0, 0.0, 0.0], [1e-3, 0.0, 0.0], [0.0, 0.0, 5.0], [0.1, 0.0, -8.0],
                          [3.0, 2.0, 40.0]])                             # degenerate / out of FoV
        pts = np.concatenate([pts, dup, extra])
        img, st = from_point_cloud(pts, ri)
        out[f"{name}/fpc_in"], out[f"{name}/fpc_img"] = pts, img.data
        out[f"{name}/fpc_stats"] = np.array([st.kept, st.collisions, st.out_of_fov, st.degenerate])
    for name in ("room", "synth"):
        intr, ri, src, dst, gt = pairs[name]
        nm = compute_normal_map(rk.RangeImage(dst, ri), "pca")
        out[f"{name}/pca_nrm"], out[f"{name}/pca_valid"] = nm.vectors, nm.valid
        nm3 = compute_normal_map(rk.RangeImage(dst, ri), "pca", radius=1, discontinuity_abs=0.1,
                                 discontinuity_rel=0.02)
        out[f"{name}/pca1_nrm"], out[f"{name}/pca1_valid"] = nm3.vectors, nm3.valid
        res = registration.register(rk.RangeImage(src, ri), rk.RangeImage(dst, ri),
                                    config=registration.RegistrationConfig(normal_method="pca"))
        out[f"{name}/pca_reg_pose"] = res.pose.matrix()
        out[f"{name}/pca_reg_stats"] = np.array([[s.stride, s.iteration, s.n_correspondences]
                                                 for s in res.stats])
    # N2: on-disk formats, byte for byte
    small, rs = sensors()["small"], ref_intr(sensors()["small"])
    room = ref_scene(scenes.room_scene())
    poses = [scenes.perturbation_pose(np.random.default_rng(40 + i), 3.0, 0.3) for i in range(3)]
    grid = sdf_volume.VoxelBlockGrid(voxel_size=0.2)
    for p in poses:
        sdf_volume.integrate_cloud_frame(grid, rk.RangeImage(render_scene(room, rs, ref_pose(p)).data, rs),
                                         ref_pose(p), clip_max=12.0)
    with tempfile.TemporaryDirectory() as d:
        io_formats.write_grid(Path(d) / "g.sdfg", grid)
        out["sdfg_bytes"] = np.frombuffer((Path(d) / "g.sdfg").read_bytes(), np.uint8)
        m = np.load(OUT / "mesh.npz")
        mesh = mesh_extract.TriangleMesh(m["sphere_V"], m["sphere_T"], m["sphere_N"])
        io_formats.write_ply(Path(d) / "m.ply", mesh)
        out["ply_bytes"] = np.frombuffer((Path(d) / "m.ply").read_bytes(), np.uint8)
    np.savez_compressed(OUT / "next.npz", **out)


def main():
    gen_sensor_and_projection()
    pairs = render_pairs()
    gen_images_icp(pairs)
    gen_tsdf(pairs)
    gen_mesh()
    gen_next(pairs)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
