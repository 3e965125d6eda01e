"""Hash-sharded volume emulated with G shards on one device:
the union of the shards must be the single-volume result, block for block
and bit for bit, each shard must hold exactly the blocks it owns, and the
streaming counters must add up.  (Only one GPU exists in this run; the
ownership function and the per-shard kernels are what is under test.)"""

import numpy as np
import pytest

import scenarios as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


def union_export(stores):
    parts = [s.export() for s in stores]
    keys = np.concatenate([p[0] for p in parts])
    order = np.argsort(keys, kind="stable")
    return [keys[order]] + [np.concatenate([p[i] for p in parts])[order] for i in (1, 2, 3)]


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_union_equals_single(V, G):
    from paper_1709_03763_b200 import _lib as L

    rng = np.random.default_rng(99 + G)
    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames = [S.wall_frame(S.QVGA_INTR, 1.2 + 0.2 * i, rng=rng, tilt=0.2 * i, noise=0.0015,
                           holes=0.05) for i in range(3)]
    old = [S.SPose(S.rot_z(0.05 * i), [0.02 * i, 0.0, 0.1]) for i in range(3)]
    new = [S.SPose(S.rot_z(0.05 * i + 0.01), [0.02 * i + 0.02, 0.01, 0.1]) for i in range(3)]
    single = V.TwoTierStore(block_capacity=1 << 16)
    shards = [V.TwoTierStore(block_capacity=1 << 16, shard_rank=r, shard_count=G)
              for r in range(G)]
    stores = [single] + shards
    recs = []
    for f, p in zip(frames, old):
        rr = []
        for s in stores:
            V.stream(s, p.translation, cfg)
            rr.append(V.integrate(s, f, p, cfg))
        recs.append(rr)
    for rr in recs:
        assert sum(r.voxels_updated for r in rr[1:]) == rr[0].voxels_updated
        assert sum(r.blocks_touched for r in rr[1:]) == rr[0].blocks_touched
        assert set().union(*[r.new_blocks for r in rr[1:]]) == rr[0].new_blocks
    for s in stores:
        ents = [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)]
        V.correct_entries(s, ents, cfg, np.array([0.3, 0.0, 0.0]))
    want = single.export()
    got = union_export(shards)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    lib = L.lib()
    for r, s in enumerate(shards):
        keys = s.export()[0]
        assert all(lib.rf_key_owner(int(k), G) == r for k in keys)
    c1 = single.counters()
    cs = [s.counters() for s in shards]
    assert sum(c.blocks_streamed_in for c in cs) == c1.blocks_streamed_in
    assert sum(c.blocks_streamed_out for c in cs) == c1.blocks_streamed_out
    assert all(c.sphere_relocations == c1.sphere_relocations for c in cs)


def test_sharded_contract_error_is_global(V):
    """A footprint block outside the sphere raises on EVERY shard, even the
    shards that do not own it, and the partial allocation matches."""
    from paper_1709_03763_b200.errors import StreamingContractError

    rng = np.random.default_rng(17)
    frame = S.random_frame(rng)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.08, stream_radius=1.2)
    G = 3
    single = V.TwoTierStore(block_capacity=1 << 12)
    shards = [V.TwoTierStore(block_capacity=1 << 12, shard_rank=r, shard_count=G)
              for r in range(G)]
    for s in [single] + shards:
        V.stream(s, np.array([-1.0, 0.0, 1.5]), cfg)
        with pytest.raises(StreamingContractError):
            V.integrate(s, frame, S.identity(), cfg)
    want = single.export()
    got = union_export(shards)
    assert len(want[0]) > 0
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
