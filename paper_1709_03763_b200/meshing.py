"""Triangle mesh extraction from the device volume.

Mirrors /root/reference/pkg/src/refusion/meshing.py: the same TriangleMesh
container, ``marching_cubes(store, cfg)`` and ``weld(mesh, tol)`` names and
results.  Marching cubes runs on the GPU (rf_marching_cubes, csrc/rf_mesh.cuh)
over every block of the store -- both tiers live in HBM -- and returns the
reference's vertex / triangle order bit for bit.  Welding and the file
writers are host post-processing of the returned arrays (meshing.py:248-321).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


def _zeros3(dtype=np.float64):
    return np.zeros((0, 3), dtype=dtype)


@dataclass
class TriangleMesh:
    """meshing.py:72-109: (N, 3) f64 vertices, (N, 3) f64 colours on the
    0..255 scale, (M, 3) int64 triangles."""

    vertices: np.ndarray = field(default_factory=_zeros3)
    colors: np.ndarray = field(default_factory=_zeros3)
    triangles: np.ndarray = field(default_factory=lambda: _zeros3(np.int64))

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_triangles(self):
        return self.triangles.shape[0]

    def validate(self):
        n = self.n_vertices
        if self.vertices.shape != (n, 3):
            raise ValueError("vertices must be (N, 3)")
        if self.colors.shape != self.vertices.shape:
            raise ValueError("colors must match vertices shape")
        if self.triangles.shape != (self.n_triangles, 3):
            raise ValueError("triangles must be (M, 3)")
        if np.isnan(self.vertices).any():
            raise ValueError("vertices contain NaN")
        if self.n_triangles and (self.triangles.min() < 0 or self.triangles.max() >= n):
            raise ValueError("triangle indices out of range")


def marching_cubes(store, cfg):
    """meshing.py:216-245 -- the D = 0 iso-surface of every block (both tiers),
    cells with all eight corners observed; vertices are not shared between
    cells (see weld)."""
    store._bind(cfg)  # raises if the store serves another config
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    store._call("rf_marching_cubes", None, None, None, 0, 0, ctypes.byref(nv), ctypes.byref(nt))
    if nv.value == 0:
        return TriangleMesh()
    v = np.empty((nv.value, 3), dtype=np.float64)
    c = np.empty((nv.value, 3), dtype=np.float64)
    t = np.empty((max(nt.value, 1), 3), dtype=np.int64)
    store._call("rf_marching_cubes", v.ctypes.data_as(L.c_double_p), c.ctypes.data_as(L.c_double_p),
                t.ctypes.data_as(L.c_int64_p), nv.value, nt.value, ctypes.byref(nv),
                ctypes.byref(nt))
    return TriangleMesh(vertices=v, colors=c, triangles=t[: nt.value])


def mesh_blocks(store, cfg):
    """The per-block layout of marching_cubes(store, cfg): (sorted block
    keys, vertices per block, triangles per block)."""
    store._bind(cfg)
    n = ctypes.c_int64()
    store._call("rf_mesh_blocks", None, None, None, 0, ctypes.byref(n))
    k = np.empty(n.value, dtype=np.int64)
    nv = np.empty(n.value, dtype=np.int64)
    nt = np.empty(n.value, dtype=np.int64)
    if n.value:
        store._call("rf_mesh_blocks", k.ctypes.data_as(L.c_int64_p), nv.ctypes.data_as(L.c_int64_p),
                    nt.ctypes.data_as(L.c_int64_p), n.value, ctypes.byref(n))
    return k, nv, nt


def merge_shard_meshes(parts):
    """Interleave the shards' meshes into the unsharded mesh's order (blocks
    by sorted coordinate, meshing.py:229-231).  ``parts``: per shard
    (TriangleMesh, keys, vertices per block, triangles per block) -- each
    shard's own blocks, meshed with its cross-shard neighbours."""
    rows = []
    for si, (m, k, nv, nt) in enumerate(parts):
        vo = np.concatenate([[0], np.cumsum(nv)])
        to = np.concatenate([[0], np.cumsum(nt)])
        rows += [(int(k[b]), si, vo[b], vo[b + 1], to[b], to[b + 1]) for b in range(len(k))]
    rows.sort()
    vs, cs, ts, base = [], [], [], 0
    for _, si, v0, v1, t0, t1 in rows:
        m = parts[si][0]
        vs.append(m.vertices[v0:v1])
        cs.append(m.colors[v0:v1])
        ts.append(m.triangles[t0:t1] - v0 + base)
        base += v1 - v0
    if not rows or base == 0:
        return TriangleMesh()
    return TriangleMesh(vertices=np.concatenate(vs), colors=np.concatenate(cs),
                        triangles=np.concatenate(ts).astype(np.int64))


def marching_cubes_sharded(stores, cfg):
    """marching_cubes over a hash-sharded volume (stores connected by
    volume.connect_shards): every shard meshes its own blocks on its device,
    reading +x/+y/+z neighbours owned by other shards from their pools, and
    the parts are merged in block order -- the unsharded mesh, bit for bit."""
    stores = sorted(stores, key=lambda s: s.shard_rank)
    G = len(stores)
    if G < 2 or [s.shard_rank for s in stores] != list(range(G)) or \
            any(s.shard_count != G for s in stores):
        raise ValueError("marching_cubes_sharded needs one store per shard rank 0..G-1")
    for s in stores:
        s._bind(cfg)
    vols = (ctypes.c_void_p * G)(*[s._ptr.value for s in stores])
    for s in stores:  # idempotent (connect_shards does it too)
        s._call("rf_mesh_connect", vols, G)
    parts = []
    for s in stores:
        parts.append((marching_cubes(s, cfg), *mesh_blocks(s, cfg)))
    return merge_shard_meshes(parts)


def welded_mesh(store, cfg, tol=1e-7):
    """weld(marching_cubes(store, cfg), tol) with both steps on the device
    (rf_marching_cubes_welded): only the welded mesh crosses to the host."""
    if tol <= 0.0:
        raise ValueError(f"tol must be > 0, got {tol}")
    store._bind(cfg)
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    store._call("rf_marching_cubes_welded", float(tol), None, None, None, 0, 0,
                ctypes.byref(nv), ctypes.byref(nt))
    if nv.value == 0:
        return TriangleMesh()
    v = np.empty((nv.value, 3), dtype=np.float64)
    c = np.empty((nv.value, 3), dtype=np.float64)
    t = np.empty((max(nt.value, 1), 3), dtype=np.int64)
    store._call("rf_marching_cubes_welded", float(tol), v.ctypes.data_as(L.c_double_p),
                c.ctypes.data_as(L.c_double_p), t.ctypes.data_as(L.c_int64_p), nv.value,
                nt.value, ctypes.byref(nv), ctypes.byref(nt))
    return TriangleMesh(vertices=v, colors=c, triangles=t[: nt.value])


def weld(mesh, tol=1e-7):
    """meshing.py:248-276 -- merge vertices on the same tol-grid point (the
    lowest index keeps its position and colour); drop triangles that collapse."""
    if tol <= 0.0:
        raise ValueError(f"tol must be > 0, got {tol}")
    if mesh.n_vertices == 0:
        return TriangleMesh()
    grid = np.round(mesh.vertices / tol).astype(np.int64)
    _, first, remap = np.unique(grid, axis=0, return_index=True, return_inverse=True)
    tri = remap.reshape(-1)[mesh.triangles]
    ok = (tri[:, 0] != tri[:, 1]) & (tri[:, 1] != tri[:, 2]) & (tri[:, 0] != tri[:, 2])
    return TriangleMesh(vertices=mesh.vertices[first], colors=mesh.colors[first],
                        triangles=tri[ok])


def save_ply(mesh, path):
    """meshing.py:279-311: binary little-endian PLY, xyz f32 + rgb u8."""
    mesh.validate()
    head = ("ply\nformat binary_little_endian 1.0\n"
            f"element vertex {mesh.n_vertices}\n"
            "property float x\nproperty float y\nproperty float z\n"
            "property uchar red\nproperty uchar green\nproperty uchar blue\n"
            f"element face {mesh.n_triangles}\n"
            "property list uchar int vertex_indices\nend_header\n")
    vt = np.dtype([("p", "<f4", (3,)), ("rgb", "u1", (3,))])
    vr = np.empty(mesh.n_vertices, dtype=vt)
    vr["p"] = mesh.vertices.astype(np.float32)
    vr["rgb"] = np.clip(np.rint(mesh.colors), 0, 255).astype(np.uint8)
    ft = np.dtype([("n", "u1"), ("idx", "<i4", (3,))])
    fr = np.empty(mesh.n_triangles, dtype=ft)
    fr["n"] = 3
    fr["idx"] = mesh.triangles.astype(np.int32)
    with open(path, "wb") as fh:
        fh.write(head.encode("ascii"))
        fh.write(vr.tobytes())
        fh.write(fr.tobytes())


def save_obj(mesh, path):
    """meshing.py:314-321: Wavefront OBJ, positions only."""
    mesh.validate()
    out = [f"v {float(x)!r} {float(y)!r} {float(z)!r}" for x, y, z in mesh.vertices]
    out += [f"f {int(a)} {int(b)} {int(c)}" for a, b, c in mesh.triangles + 1]
    with open(path, "w") as fh:
        fh.write("\n".join(out + [""]))
