"""Seeded synthetic workload definitions (sensors, scenes, trajectories).

These are *input definitions* shared by the tests, ``bench.py`` and
``__graft_entry__.smoke()`` -- not algorithms on the hot path.  They follow
SURVEY.md §8(d):

* ``ouster64`` -- the Ouster-like 64x1024 sensor (r0 = 0.015806 m, 4-column
  stagger azimuth table + U(+-1e-3) jitter seed 7, non-uniform 33.2 deg span);
* ``hdl64`` -- KITTI-shaped 64x2048 ``synthetic_intrinsics`` (r0 = 0 path);
* ``os128`` -- 128x2048, r0 = 0.05, U(+-0.01) azimuth seed 7, 45 deg span;
* the reference test fixtures ``small_calib`` (32x256), ``synth_intr`` (64x512)
  and ``calib128`` (128x1024) (reference pkg/tests/conftest.py:17-38);
* ``street_scene`` (reference test_acceptance.py:41-47), ``room_scene``
  (conftest.py:41-52) and ``wall_scene``.

Primitives are tuples ``("box", centre, size, R|None)``, ``("sphere", c, r)``,
``("plane", normal, offset)``.
"""

from __future__ import annotations

import numpy as np

from .lidar_model import LidarIntrinsics, synthetic_intrinsics
from .se3 import RigidTransform


def nonuniform_elevation_lut(height, span_deg=45.0, skew=0.15, top_deg=None):
    """Decreasing, mildly non-uniform elevation table (conftest.py:9-14)."""
    s = np.linspace(0.0, 1.0, height)
    top = span_deg / 2 if top_deg is None else top_deg
    return np.deg2rad(top) - np.deg2rad(span_deg) * (s + skew * s * (1.0 - s))


def ouster64(width=1024):
    az = np.resize(np.deg2rad([3.1, 0.9, -1.3, -3.4]), 64)
    az = az + np.random.default_rng(7).uniform(-1e-3, 1e-3, 64)
    return LidarIntrinsics(width=width, height=64, receiver_radius=0.015806,
                           azimuth_lut=az,
                           elevation_lut=nonuniform_elevation_lut(64, span_deg=33.2, skew=0.10))


def hdl64():
    return synthetic_intrinsics(64, 2048, np.deg2rad(-24.8), np.deg2rad(2.0))


def os128():
    g = np.random.default_rng(7)
    return LidarIntrinsics(width=2048, height=128, receiver_radius=0.05,
                           azimuth_lut=g.uniform(-0.01, 0.01, 128),
                           elevation_lut=nonuniform_elevation_lut(128))


def calib128():
    g = np.random.default_rng(7)
    return LidarIntrinsics(width=1024, height=128, receiver_radius=0.05,
                           azimuth_lut=g.uniform(-0.01, 0.01, 128),
                           elevation_lut=nonuniform_elevation_lut(128))


def small_calib():
    g = np.random.default_rng(11)
    return LidarIntrinsics(width=256, height=32, receiver_radius=0.04,
                           azimuth_lut=g.uniform(-0.008, 0.008, 32),
                           elevation_lut=nonuniform_elevation_lut(32, span_deg=40.0))


def synth_intr():
    return synthetic_intrinsics(64, 512, np.deg2rad(-15.75), np.deg2rad(16.25))


def street_scene():
    return [("box", (8.0, 0.0, 2.0), (0.5, 30.0, 8.0), None),
            ("box", (-8.0, 3.0, 2.0), (0.5, 30.0, 8.0), None),
            ("box", (0.0, 16.0, 2.0), (18.0, 0.5, 8.0), None),
            ("box", (0.0, -14.0, 2.0), (18.0, 0.5, 8.0), None),
            ("box", (0.0, 1.0, -2.05), (17.0, 31.0, 0.5), None),
            ("box", (4.0, 6.0, -1.0), (2.0, 3.0, 2.0), None),
            ("sphere", (-3.0, -6.0, -0.3), 1.5)]


def extended_street_scene(length_m: float, y0: float = -14.0):
    """C5's extended street: the street's two façades and ground
    slab run ``length_m`` along +y from ``y0``, with a box and a sphere
    repeated every 10 m (street_scene's kerb-side objects) and a cross wall
    closing each end."""
    L = float(length_m)
    yc = y0 + 0.5 * L
    prims = [("box", (8.0, yc, 2.0), (0.5, L, 8.0), None),
             ("box", (-8.0, yc, 2.0), (0.5, L, 8.0), None),
             ("box", (0.0, yc, -2.05), (17.0, L + 1.0, 0.5), None),
             ("box", (0.0, y0, 2.0), (18.0, 0.5, 8.0), None),
             ("box", (0.0, y0 + L, 2.0), (18.0, 0.5, 8.0), None)]
    for k in range(int(L // 10.0)):
        y = y0 + 10.0 * k
        prims.append(("box", (4.0, y + 6.0, -1.0), (2.0, 3.0, 2.0), None))
        prims.append(("sphere", (-3.0, y + 2.0, -0.3), 1.5))
    return prims


def room_scene():
    return [("box", (6.0, 0.0, 1.0), (0.4, 16.0, 6.0), None),
            ("box", (0.0, 7.0, 1.0), (16.0, 0.4, 6.0), None),
            ("box", (-6.5, -1.0, 1.5), (0.4, 14.0, 6.0), None),
            ("box", (1.0, -7.5, 1.0), (14.0, 0.4, 6.0), None),
            ("plane", (0.0, 0.0, 1.0), -1.2),
            ("sphere", (3.0, -2.0, 0.2), 1.2),
            ("box", (-2.5, 3.5, -0.4), (1.6, 1.2, 1.6), None)]


def wall_scene():
    return [("box", (4.5, 0.0, 0.0), (1.0, 12.0, 6.0), None)]


def perturbation_pose(rng, rot_deg, trans_m):
    """Random-axis rotation of rot_deg and translation of length trans_m
    (conftest.py:65-70)."""
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    t = rng.normal(size=3)
    t *= trans_m / np.linalg.norm(t)
    return RigidTransform.exp(np.concatenate([axis * np.deg2rad(rot_deg), t]))


def street_trajectory(n, seed=0, step_m=0.2, jitter=0.002):
    """C2 sequence: drive along the street's +y axis from (0, -10, 0) with
    step_m per frame plus U(+-jitter) twist noise; world-from-frame poses."""
    g = np.random.default_rng(seed)
    c, s = np.cos(np.pi / 2), np.sin(np.pi / 2)
    pose = RigidTransform(np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]]),
                          np.array([0.0, -10.0, 0.0]))
    poses = []
    for _ in range(n):
        poses.append(pose)
        step = np.concatenate([g.uniform(-jitter, jitter, 3),
                               np.array([step_m, 0.0, 0.0]) + g.uniform(-jitter, jitter, 3)])
        pose = pose @ RigidTransform.exp(step)
    return poses


def pair_pool_poses(n_pairs, seed=0, rot_deg=2.0, trans_m=0.3):
    """C4 pool: dst sensor placed at a seeded spot in the street, src at
    dst @ perturbation; returns [(dst_pose_world, gt_src_to_dst)]."""
    g = np.random.default_rng(seed)
    out = []
    for i in range(n_pairs):
        yaw = g.uniform(-np.pi, np.pi)
        c, s = np.cos(yaw), np.sin(yaw)
        base = RigidTransform(np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]]),
                              np.array([g.uniform(-4.0, 4.0), g.uniform(-9.0, 9.0), 0.0]))
        gt = perturbation_pose(np.random.default_rng(1000 + i), rot_deg, trans_m)
        out.append((base, gt))
    return out
