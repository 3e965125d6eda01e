"""Marching cubes + weld (refusion/meshing.py:112-276).

CPU: the packed triangle table equals the reference's, the numpy oracle
(oracle/mesh_oracle.py) reproduces the reference's golden meshes bit for bit
and the host weld reproduces the reference's welded meshes.  GPU: the device
marching cubes (rf_marching_cubes) equals the golden meshes and the oracle,
bit for bit, on imported and on integrated volumes."""

import os
import re
import sys

import numpy as np
import pytest

import scenarios as S

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = np.load(os.path.join(HERE, "golden", "mesh_golden.npz"))
CASES = (("a", 5, 0.01), ("b", 11, 0.004))


def oracle():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import mesh_oracle

    return mesh_oracle


def test_packed_table_matches_reference():
    ref = None
    for p in (os.path.join(REPO, "oracle", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "refusion")):
            sys.path.insert(0, p)
            from refusion import mc_tables as ref
            break
    if ref is None:
        pytest.skip("reference package not present (GPU box)")
    O = oracle()
    assert np.array_equal(O.CASE_TRIANGLES, ref.CASE_TRIANGLES)
    assert np.array_equal(O.CASE_EDGES, ref.CASE_EDGES)
    assert np.array_equal(O.EDGES, ref.EDGE_VERTEX_PAIRS)


@pytest.mark.parametrize("name,seed,voxel", CASES)
def test_oracle_matches_reference_golden(name, seed, voxel):
    keys, data, _ = S.mesh_volume(seed, voxel)
    v, c, t = oracle().marching_cubes(keys, data, voxel)
    assert np.array_equal(v, GOLDEN[f"{name}_vertices"])
    assert np.array_equal(c, GOLDEN[f"{name}_colors"])
    assert np.array_equal(t, GOLDEN[f"{name}_triangles"])


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_weld_matches_reference_golden(name):
    from paper_1709_03763_b200 import meshing as M

    mesh = M.TriangleMesh(GOLDEN[f"{name}_vertices"], GOLDEN[f"{name}_colors"],
                          GOLDEN[f"{name}_triangles"])
    mesh.validate()
    w = M.weld(mesh, 1e-7)
    assert np.array_equal(w.vertices, GOLDEN[f"{name}_weld_vertices"])
    assert np.array_equal(w.triangles, GOLDEN[f"{name}_weld_triangles"])
    with pytest.raises(ValueError):
        M.weld(mesh, 0.0)
    assert M.weld(M.TriangleMesh(), 1e-7).n_vertices == 0


def test_mesh_writers(tmp_path):
    from paper_1709_03763_b200 import meshing as M

    mesh = M.TriangleMesh(GOLDEN["a_vertices"], GOLDEN["a_colors"], GOLDEN["a_triangles"])
    M.save_ply(mesh, tmp_path / "m.ply")
    raw = (tmp_path / "m.ply").read_bytes()
    head = raw[: raw.index(b"end_header\n") + len(b"end_header\n")]
    assert f"element vertex {mesh.n_vertices}".encode() in head
    assert len(raw) - len(head) == mesh.n_vertices * 15 + mesh.n_triangles * 13
    M.save_obj(mesh, tmp_path / "m.obj")
    lines = (tmp_path / "m.obj").read_text().splitlines()
    assert len(lines) == mesh.n_vertices + mesh.n_triangles


# ---------------------------------------------------------------------------
# device


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed,voxel", CASES)
def test_device_mc_matches_reference_golden(V, name, seed, voxel):
    from paper_1709_03763_b200 import meshing as M

    keys, data, _ = S.mesh_volume(seed, voxel)
    cfg = V.VolumeConfig(voxel_size=voxel, hash_buckets=1 << 12)
    store = V.TwoTierStore(block_capacity=4096)
    store._bind(cfg)
    store._import(keys, data)
    mesh = M.marching_cubes(store, cfg)
    mesh.validate()
    assert np.array_equal(mesh.vertices, GOLDEN[f"{name}_vertices"])
    assert np.array_equal(mesh.colors, GOLDEN[f"{name}_colors"])
    assert np.array_equal(mesh.triangles, GOLDEN[f"{name}_triangles"])
    w = M.weld(mesh, 1e-7)
    assert np.array_equal(w.triangles, GOLDEN[f"{name}_weld_triangles"])


@pytest.mark.gpu
def test_device_mc_matches_oracle_on_integrated_volume(V):
    """A volume the device fused from noisy wall frames (negative and positive
    coordinates, holes): device mesh == oracle mesh of the exported blocks."""
    from paper_1709_03763_b200 import meshing as M

    rng = np.random.default_rng(8)
    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.03, stream_radius=6.0, hash_buckets=1 << 14)
    store = V.TwoTierStore(block_capacity=1 << 15)
    V.stream(store, np.zeros(3), cfg)
    for i in range(3):
        f = S.wall_frame(S.QVGA_INTR, 0.9 + 0.1 * i, rng=rng, tilt=0.3 * i, noise=0.002,
                         holes=0.05)
        V.integrate(store, f, S.SPose(S.rot_y(0.1 * i), [0.05 * i - 0.05, 0.02, -0.1]), cfg)
    keys, d, w, c = store.export()
    data = np.concatenate([d[:, None], w[:, None], np.transpose(c, (0, 2, 1))], axis=1)
    v, col, t = oracle().marching_cubes(keys, data, cfg.voxel_size)
    mesh = M.marching_cubes(store, cfg)
    assert mesh.n_triangles > 1000
    assert np.array_equal(mesh.vertices, v)
    assert np.array_equal(mesh.colors, col)
    assert np.array_equal(mesh.triangles, t)


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed,voxel", CASES)
def test_device_weld_matches_reference_golden(V, name, seed, voxel):
    from paper_1709_03763_b200 import meshing as M

    keys, data, _ = S.mesh_volume(seed, voxel)
    cfg = V.VolumeConfig(voxel_size=voxel, hash_buckets=1 << 12)
    store = V.TwoTierStore(block_capacity=4096)
    store._bind(cfg)
    store._import(keys, data)
    w = M.welded_mesh(store, cfg, 1e-7)
    assert np.array_equal(w.vertices, GOLDEN[f"{name}_weld_vertices"])
    assert np.array_equal(w.triangles, GOLDEN[f"{name}_weld_triangles"])
    host = M.weld(M.marching_cubes(store, cfg), 1e-7)
    assert np.array_equal(w.colors, host.colors)
    # a coarse tolerance merges more (and collapses triangles): still numpy's result
    coarse = M.welded_mesh(store, cfg, 2e-3)
    want = M.weld(M.marching_cubes(store, cfg), 2e-3)
    for a in ("vertices", "colors", "triangles"):
        assert np.array_equal(getattr(coarse, a), getattr(want, a))
    assert coarse.n_triangles < w.n_triangles


@pytest.mark.gpu
def test_device_mc_empty(V):
    from paper_1709_03763_b200 import meshing as M

    cfg = V.VolumeConfig(voxel_size=0.01, hash_buckets=1 << 10)
    store = V.TwoTierStore(block_capacity=64)
    mesh = M.marching_cubes(store, cfg)
    assert mesh.n_vertices == 0 and mesh.n_triangles == 0
    assert M.welded_mesh(store, cfg).n_vertices == 0
    store.put_block((0, 0, 0), d=np.ones(512), w=np.ones(512))  # no sign change
    assert M.marching_cubes(store, cfg).n_triangles == 0
    assert M.welded_mesh(store, cfg).n_triangles == 0


# ---------------------------------------------------------------------------
# nn_min_d2: the plugin's evaluation kernel (_kernels_cy.pyx:111-129)


def _nn_case(seed, n, m):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 3)) * rng.choice([1e-3, 1.0, 50.0], size=(n, 1))
    pts = rng.normal(size=(m, 3))
    if m and n > 4:
        q[:3] = pts[rng.integers(0, m, 3)]  # exact hits: d2 = 0
    return np.ascontiguousarray(q), np.ascontiguousarray(pts)


def test_nn_oracle_matches_reference_python():
    ref = None
    for p in (os.path.join(REPO, "oracle", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "refusion")):
            sys.path.insert(0, p)
            from refusion import _kernels_py as ref
            break
    if ref is None:
        pytest.skip("reference package not present")
    q, pts = _nn_case(1, 300, 5000)
    want = np.empty(len(q))
    ref.nn_min_d2(q, pts, want)
    assert np.array_equal(oracle().nn_min_d2(q, pts), want)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(1, 1), (513, 1), (1000, 3000), (4097, 1025), (7, 0), (0, 5)])
def test_device_nn_min_d2_matches_oracle(V, n, m):
    from paper_1709_03763_b200 import kernels as K

    q, pts = _nn_case(n + m, n, m)
    out = np.empty(n)
    K.nn_min_d2(q, pts, out)
    assert np.array_equal(out, oracle().nn_min_d2(q, pts))
    with pytest.raises((TypeError, ValueError)):
        K.nn_min_d2(q.astype(np.float32), pts, out)


def test_merge_shard_meshes_restores_block_order():
    """Host merge of the shards' meshes (meshing.merge_shard_meshes): blocks
    interleave by key, triangle indices are re-based -- the unsharded mesh."""
    from paper_1709_03763_b200 import meshing as M

    rng = np.random.default_rng(2)
    keys = np.sort(rng.choice(10_000, size=40, replace=False)).astype(np.int64)
    nv = rng.integers(0, 9, size=40)
    nt = np.where(nv >= 3, rng.integers(0, 5, size=40), 0)
    verts = rng.normal(size=(nv.sum(), 3))
    cols = rng.uniform(0, 255, size=(nv.sum(), 3))
    vo = np.concatenate([[0], np.cumsum(nv)])
    tris = np.concatenate([vo[b] + rng.integers(0, nv[b], size=(nt[b], 3)) for b in range(40)]
                          + [np.zeros((0, 3), np.int64)]).astype(np.int64)
    whole = M.TriangleMesh(verts, cols, tris)
    to = np.concatenate([[0], np.cumsum(nt)])
    owner = rng.integers(0, 3, size=40)
    parts = []
    for s in range(3):
        bs = np.flatnonzero(owner == s)
        sv = [verts[vo[b]:vo[b + 1]] for b in bs]
        sc = [cols[vo[b]:vo[b + 1]] for b in bs]
        st, base = [], 0
        for b in bs:
            st.append(tris[to[b]:to[b + 1]] - vo[b] + base)
            base += nv[b]
        m = M.TriangleMesh(np.concatenate(sv + [np.zeros((0, 3))]),
                           np.concatenate(sc + [np.zeros((0, 3))]),
                           np.concatenate(st + [np.zeros((0, 3), np.int64)]).astype(np.int64))
        parts.append((m, keys[bs], nv[bs], nt[bs]))
    got = M.merge_shard_meshes(parts)
    assert np.array_equal(got.vertices, whole.vertices)
    assert np.array_equal(got.colors, whole.colors)
    assert np.array_equal(got.triangles, whole.triangles)
