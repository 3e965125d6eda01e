"""SURVEY §8 f1 on a hash-sharded volume: marching cubes borrows the +x/+y/+z
neighbour blocks (reference meshing.py:112-147), which on a sharded store
may belong to another shard.  Each shard meshes its own blocks reading
those neighbours from their owners' pools (rf_mesh_connect); merged in
block order the shards' meshes must equal the unsharded mesh bit for bit.
Shards are emulated on the one device (like tests/test_sharding_gpu.py)."""

import numpy as np
import pytest

import scenarios as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import meshing, volume

    return volume, meshing


def _same(a, b):
    return (np.array_equal(a.vertices, b.vertices) and np.array_equal(a.colors, b.colors)
            and np.array_equal(a.triangles, b.triangles))


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_marching_cubes_equals_single(mods, G):
    V, M = mods
    rng = np.random.default_rng(41 + G)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames = [S.wall_frame(S.QVGA_INTR, 1.1 + 0.15 * i, rng=rng, tilt=0.25 * i, noise=0.001,
                           holes=0.02) for i in range(3)]
    poses = [S.SPose(S.rot_z(0.07 * i), [0.03 * i, -0.02, 0.1]) for i in range(3)]
    single = V.TwoTierStore(block_capacity=1 << 15)
    shards = [V.TwoTierStore(block_capacity=1 << 15, shard_rank=r, shard_count=G)
              for r in range(G)]
    for s in [single] + shards:
        for f, p in zip(frames, poses):
            V.stream(s, p.translation, cfg)
            V.integrate(s, f, p, cfg)
    want = M.marching_cubes(single, cfg)
    assert want.n_triangles > 1000
    # without the other shards' neighbours the seams lose their cells
    alone = M.merge_shard_meshes([(M.marching_cubes(s, cfg), *M.mesh_blocks(s, cfg))
                                  for s in shards])
    assert alone.n_vertices < want.n_vertices
    got = M.marching_cubes_sharded(shards, cfg)
    assert _same(got, want)
    # welded on the host from the merged mesh == welded single mesh
    assert _same(M.weld(got), M.weld(want))
    # per-block layout adds up
    k, nv, nt = M.mesh_blocks(single, cfg)
    assert nv.sum() == want.n_vertices and nt.sum() == want.n_triangles
    assert np.all(np.diff(k) > 0)
