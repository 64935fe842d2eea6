"""Oracle: Marching Cubes over the sparse block grid.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
``rangekit/mc_tables.py`` (case-table generation) and
``rangekit/mesh_extract.py`` (extraction); citations are to those files.
"""

from __future__ import annotations

import numpy as np

from .tsdf import EDGE

CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
           (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))          # mc_tables.py:28-31
EDGES = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
         (0, 4), (1, 5), (2, 6), (3, 7))                         # mc_tables.py:33-37
FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4),
         (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5))               # mc_tables.py:40-47


def build_tri_table():
    """Face-segment loops, fan-triangulated (mc_tables.py:55-111).

    On each face, walking the boundary ccw, every sign change is a crossing;
    an inside->outside crossing is joined to the crossing just before it.  The
    directed segments are chained into loops starting from the smallest edge
    id, and each loop (l0, l1, ..., lk) becomes triangles (l0, l_{i+1}, l_i).
    """
    edge_id = {}
    for e, (a, b) in enumerate(EDGES):
        edge_id[(a, b)] = edge_id[(b, a)] = e
    table = np.full((256, 16), -1, dtype=np.int8)
    for case in range(256):
        inside = [bool((case >> i) & 1) for i in range(8)]
        nxt = {}
        for face in FACES:
            xs = []
            for i in range(4):
                a, b = face[i], face[(i + 1) % 4]
                if inside[a] != inside[b]:
                    xs.append((edge_id[(a, b)], inside[a]))
            for i, (e, leaving) in enumerate(xs):
                if leaving:
                    nxt[e] = xs[i - 1][0]
        tris = []
        done = set()
        for start in sorted(nxt):
            if start in done:
                continue
            loop = [start]
            done.add(start)
            e = nxt[start]
            while e != start:
                loop.append(e)
                done.add(e)
                e = nxt[e]
            for i in range(1, len(loop) - 1):
                tris += [loop[0], loop[i + 1], loop[i]]
        table[case, :len(tris)] = tris
    return table


TRI_TABLE = build_tri_table()

# canonical (lower corner, upper corner) per edge and its axis (mesh_extract.py:25-34)
CANON = [(a, b) if CORNERS[a] <= CORNERS[b] else (b, a) for a, b in EDGES]
AXIS = [int(np.nonzero(np.subtract(CORNERS[b], CORNERS[a]))[0][0]) for a, b in CANON]


def halo(grid, key):
    """(tsdf, weight) over local -1..17 on each axis; missing voxels weight 0 (58-82)."""
    n = EDGE + 3
    d = np.zeros((n, n, n), np.float32)
    w = np.zeros((n, n, n), np.float32)
    # each halo index h covers local voxel h-1 of block key + floor((h-1)/16)
    for ox in (-1, 0, 1):
        for oy in (-1, 0, 1):
            for oz in (-1, 0, 1):
                blk = grid.get((key[0] + ox, key[1] + oy, key[2] + oz))
                if blk is None:
                    continue
                src, dst = [], []
                for o in (ox, oy, oz):
                    lo = max(o * EDGE, -1)
                    hi = min(o * EDGE + EDGE, EDGE + 2)
                    dst.append(slice(lo + 1, hi + 1))
                    src.append(slice(lo - o * EDGE, hi - o * EDGE))
                d[tuple(dst)] = blk[0][tuple(src)]
                w[tuple(dst)] = blk[1][tuple(src)]
    return d, w


def corner_gradients(d, w, voxel):
    """Central (else one-sided, else 0) differences at local corners 0..16 (181-199)."""
    g = np.zeros((3, EDGE + 1, EDGE + 1, EDGE + 1))
    core = slice(1, EDGE + 2)
    for ax in range(3):
        up = np.roll(d, -1, axis=ax)
        dn = np.roll(d, 1, axis=ax)
        up_ok = np.roll(w, -1, axis=ax) > 0
        dn_ok = np.roll(w, 1, axis=ax) > 0
        val = np.where(up_ok & dn_ok, (up - dn) / (2 * voxel),
                       np.where(up_ok, (up - d) / voxel,
                                np.where(dn_ok, (d - dn) / voxel, 0.0)))
        g[ax] = val[core, core, core]
    return g


def extract_mesh(grid, voxel, min_weight=1.0):
    """Sequential MC with global edge-key and exact-position vertex merging (85-209).

    Returns (vertices (V,3) f64, triangles (T,3) int32, normals (V,3) f64).
    """
    E = EDGE
    by_edge, by_pos = {}, {}
    verts, vnorm, tris = [], [], []
    corner_arr = np.array(CORNERS)
    for key in sorted(grid):
        d32, w = halo(grid, key)
        d = d32.astype(np.float64)
        seen = w >= min_weight
        vals = np.empty((8, E, E, E))
        full = np.ones((E, E, E), bool)
        for ci, (cx, cy, cz) in enumerate(CORNERS):
            sl = (slice(1 + cx, 1 + cx + E), slice(1 + cy, 1 + cy + E), slice(1 + cz, 1 + cz + E))
            vals[ci] = d[sl]
            full &= seen[sl]
        case = np.zeros((E, E, E), np.int32)
        for ci in range(8):
            case |= (vals[ci] < 0).astype(np.int32) << ci
        active = full & (case > 0) & (case < 255)
        if not active.any():
            continue
        base = np.asarray(key, dtype=np.int64) * E
        grads = corner_gradients(d, w, voxel)
        for cell in zip(*np.nonzero(active)):
            cell = np.array(cell, dtype=np.int64)
            cv = vals[:, cell[0], cell[1], cell[2]]
            row = TRI_TABLE[case[tuple(cell)]]
            local = {}
            for e in (int(x) for x in row if x >= 0):
                if e in local:
                    continue
                a, b = CANON[e]
                ca, cb = cell + corner_arr[a], cell + corner_arr[b]
                ek = (int(base[0] + ca[0]), int(base[1] + ca[1]), int(base[2] + ca[2]), AXIS[e])
                vid = by_edge.get(ek)
                if vid is None:
                    da, db = cv[a], cv[b]
                    t = 0.5 if abs(da - db) < 1e-9 else da / (da - db)
                    if t < 1e-6:
                        t = 0.0
                    elif t > 1.0 - 1e-6:
                        t = 1.0
                    pos = ((base + ca + 0.5) * voxel) * (1.0 - t) + ((base + cb + 0.5) * voxel) * t
                    pk = (pos[0], pos[1], pos[2])
                    vid = by_pos.get(pk)
                    if vid is None:
                        vid = len(verts)
                        by_pos[pk] = vid
                        verts.append(pos)
                        vnorm.append(grads[:, ca[0], ca[1], ca[2]] * (1.0 - t)
                                     + grads[:, cb[0], cb[1], cb[2]] * t)
                    by_edge[ek] = vid
                local[e] = vid
            for i in range(0, 16, 3):
                if row[i] < 0:
                    break
                tri = (local[int(row[i])], local[int(row[i + 1])], local[int(row[i + 2])])
                if len(set(tri)) == 3:
                    tris.append(tri)
    if not verts:
        return np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros((0, 3))
    V = np.asarray(verts)
    T = np.asarray(tris, dtype=np.int32).reshape(-1, 3)
    N = np.asarray(vnorm)
    nn = np.linalg.norm(N, axis=1)
    good = nn > 1e-12
    N[good] /= nn[good, None]
    N[~good] = (0.0, 0.0, 1.0)
    if T.shape[0]:
        a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
        T = T[np.linalg.norm(np.cross(b - a, c - a), axis=1) > 2e-12]
    return V, T, N
