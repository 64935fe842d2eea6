"""Marching Cubes case tables -- drop-in for rangekit/mc_tables.py.

The reference *generates* its table (it is not the classic published listing):
on each cube face the sign changes are walked counter-clockwise and every
inside->outside crossing is joined to the crossing before it; the directed
face segments are chained into loops (started from the smallest edge id) and
each loop (l0, l1, ..., lk) is fanned into triangles (l0, l_{i+1}, l_i)
(mc_tables.py:55-111).  The same construction is restated here so the device
kernel receives an identical ``TRI_TABLE``.
"""

from __future__ import annotations

import numpy as np

CORNER_POS = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                       (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)], dtype=np.int64)

EDGE_CORNERS = np.array([(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
                         (0, 4), (1, 5), (2, 6), (3, 7)], dtype=np.int64)

# faces, corners counter-clockwise seen from outside
_FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5))


def _edge_lookup():
    table = {}
    for e, (a, b) in enumerate(EDGE_CORNERS.tolist()):
        table[(a, b)] = table[(b, a)] = e
    return table


def _case_loops(case: int, edge_of) -> list[list[int]]:
    inside = [(case >> i) & 1 == 1 for i in range(8)]
    successor = {}
    for face in _FACES:
        ring = [(edge_of[(face[i], face[(i + 1) % 4])], inside[face[i]])
                for i in range(4) if inside[face[i]] != inside[face[(i + 1) % 4]]]
        for i, (edge, leaving) in enumerate(ring):
            if leaving:
                successor[edge] = ring[i - 1][0]
    loops, used = [], set()
    for start in sorted(successor):
        if start in used:
            continue
        loop, e = [start], successor[start]
        used.add(start)
        while e != start:
            loop.append(e)
            used.add(e)
            e = successor[e]
        loops.append(loop)
    return loops


def _generate():
    edge_of = _edge_lookup()
    tri = np.full((256, 16), -1, dtype=np.int8)
    for case in range(256):
        flat = []
        for loop in _case_loops(case, edge_of):
            for i in range(1, len(loop) - 1):
                flat += (loop[0], loop[i + 1], loop[i])
        tri[case, :len(flat)] = flat
    edge = np.zeros(256, dtype=np.int32)
    for case in range(256):
        for e in tri[case][tri[case] >= 0]:
            edge[case] |= 1 << int(e)
    return edge, tri


EDGE_TABLE, TRI_TABLE = _generate()
