"""CPU oracle for marching cubes -- TEST INFRASTRUCTURE ONLY (imported by
tests/ as the checker; never by the product).

A numpy restatement of /root/reference/pkg/src/refusion/meshing.py:112-245
(`_padded_grids`, `_block_cells`, `marching_cubes`) over a plain exported
block set (keys [n] packed as volume.py:137-141, data [n][5][512] = D, W,
C0, C1, C2).  The triangle table is the canonical one (mc_tables.py:44-302);
it is read from the packed copy in csrc/rf_mesh.cuh, itself checked against
the reference's table by tests/test_mesh.py, and the whole restatement is
pinned by golden meshes the reference produced (tests/golden/mesh_golden.npz,
tests/golden/gen_mesh_golden.py).
"""

import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HEADER = os.path.join(os.path.dirname(_HERE), "paper_1709_03763_b200", "csrc", "rf_mesh.cuh")

CORNERS = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                    (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)], dtype=np.int64)  # meshing.py:23-35
EDGES = np.array([(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
                  (0, 4), (1, 5), (2, 6), (3, 7)], dtype=np.int64)                  # mc_tables.py:10-23
NEIGHBOURS = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)]
BIAS = 1 << 20


def _tables():
    text = open(_HEADER).read()
    body = text[text.index("kMcTriangles[256]"):]
    words = [int(w, 16) for w in re.findall(r"0x([0-9a-f]{16})ull", body)[:256]]
    tri = -np.ones((256, 16), dtype=np.int64)
    for c, w in enumerate(words):
        n = 3 * (w >> 60)
        for i in range(n):
            tri[c, i] = (w >> (4 * i)) & 0xF
    edges = np.zeros(256, dtype=np.int64)
    for c in range(256):
        for e, (a, b) in enumerate(EDGES):
            if ((c >> a) ^ (c >> b)) & 1:
                edges[c] |= 1 << e
    return edges, tri


CASE_EDGES, CASE_TRIANGLES = _tables()


def _coords(key):
    key = int(key)
    return ((key >> 42) - BIAS, ((key >> 21) & ((1 << 21) - 1)) - BIAS,
            (key & ((1 << 21) - 1)) - BIAS)


def _pack(x, y, z):
    return ((x + BIAS) << 42) | ((y + BIAS) << 21) | (z + BIAS)


def _grids(index, data, coord):
    """meshing.py:112-146: 9x9x9 D, W and 9x9x9x3 C in [z, y, x] order."""
    d9, w9, c9 = np.zeros((9, 9, 9)), np.zeros((9, 9, 9)), np.zeros((9, 9, 9, 3))

    def planes(i):
        blk = data[i]
        return (blk[0].reshape(8, 8, 8), blk[1].reshape(8, 8, 8),
                np.stack([blk[2], blk[3], blk[4]], axis=1).reshape(8, 8, 8, 3))

    d, w, c = planes(index[_pack(*coord)])
    d9[:8, :8, :8], w9[:8, :8, :8], c9[:8, :8, :8] = d, w, c
    for dx, dy, dz in NEIGHBOURS:
        j = index.get(_pack(coord[0] + dx, coord[1] + dy, coord[2] + dz))
        if j is None:
            continue
        d, w, c = planes(j)
        dst = (8 if dz else slice(0, 8), 8 if dy else slice(0, 8), 8 if dx else slice(0, 8))
        src = (0 if dz else slice(0, 8), 0 if dy else slice(0, 8), 0 if dx else slice(0, 8))
        d9[dst], w9[dst], c9[dst] = d[src], w[src], c[src]
    return d9, w9, c9


def _cells(index, data, coord, vs):
    """meshing.py:149-213 for one block."""
    d9, w9, c9 = _grids(index, data, coord)
    cd = np.stack([d9[oz:oz + 8, oy:oy + 8, ox:ox + 8] for ox, oy, oz in CORNERS])
    cw = np.stack([w9[oz:oz + 8, oy:oy + 8, ox:ox + 8] for ox, oy, oz in CORNERS])
    cube = np.zeros((8, 8, 8), dtype=np.int64)
    for i in range(8):
        cube |= (cd[i] < 0.0).astype(np.int64) << i
    live = (cw > 0.0).all(axis=0) & (CASE_EDGES[cube] != 0)
    if not live.any():
        return None
    z, y, x = np.nonzero(live)
    cube = cube[live]
    dcell = cd[:, live].T
    ccell = np.stack([c9[oz:oz + 8, oy:oy + 8, ox:ox + 8][live] for ox, oy, oz in CORNERS], axis=1)
    a, b = EDGES[:, 0], EDGES[:, 1]
    da, db = dcell[:, a], dcell[:, b]
    den = da - db
    t = np.where(den == 0.0, 0.5, da / np.where(den == 0.0, 1.0, den))
    anchor = np.stack([x + coord[0] * 8, y + coord[1] * 8, z + coord[2] * 8], axis=1)
    base = (anchor[:, None, :] + 0.5) * vs
    offs = CORNERS.astype(np.float64) * vs
    pa, pb = base + offs[a][None], base + offs[b][None]
    pos = pa + t[:, :, None] * (pb - pa)
    col = ccell[:, a] + t[:, :, None] * (ccell[:, b] - ccell[:, a])
    used = ((CASE_EDGES[cube][:, None] >> np.arange(12)) & 1).astype(bool)
    rank = np.cumsum(used, axis=1) - 1
    first = np.concatenate([[0], np.cumsum(used.sum(axis=1))[:-1]])
    tl = CASE_TRIANGLES[cube]
    slot = tl >= 0
    cell = np.broadcast_to(np.arange(len(cube))[:, None], slot.shape)[slot]
    tri = (first[cell] + rank[cell, tl[slot]]).reshape(-1, 3)
    return pos[used], col[used], tri


def marching_cubes(keys, data, voxel_size):
    """meshing.py:216-245: (vertices, colors, triangles) of an exported volume."""
    keys = np.asarray(keys, dtype=np.int64)
    data = np.asarray(data, dtype=np.float64).reshape(len(keys), 5, 512)
    index = {int(k): i for i, k in enumerate(keys)}
    vs, cs, ts, n = [], [], [], 0
    for k in np.sort(keys):
        out = _cells(index, data, _coords(k), voxel_size)
        if out is None:
            continue
        v, c, t = out
        vs.append(v)
        cs.append(c)
        ts.append(t + n)
        n += len(v)
    if not vs:
        return np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)
    return np.concatenate(vs), np.concatenate(cs), np.concatenate(ts)


def nn_min_d2(q, pts):
    """_kernels_cy.pyx:111-129 / _kernels_py.py:107-120: per query the minimum
    of (dx*dx + dy*dy) + dz*dz over the points (+inf without points)."""
    q = np.asarray(q, dtype=np.float64)
    pts = np.asarray(pts, dtype=np.float64)
    out = np.full(len(q), np.inf)
    for lo in range(0, len(pts), 4096):
        p = pts[lo:lo + 4096]
        dx = q[:, None, 0] - p[None, :, 0]
        dy = q[:, None, 1] - p[None, :, 1]
        dz = q[:, None, 2] - p[None, :, 2]
        d2 = dx * dx + dy * dy
        d2 = d2 + dz * dz
        np.minimum(out, d2.min(axis=1), out=out)
    return out
