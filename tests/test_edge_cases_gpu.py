"""Edge cases of the volume path against the CPU oracle (bit for bit): keyframes
with no valid pixel, non-finite / non-positive depths, a one-pixel image,
windows with no entries, and a de-integration of a keyframe that touched
nothing.  (volume.py:151-338, reintegration.py:156-181.)"""

import numpy as np
import pytest

import oracle as O
import scenarios as S

pytestmark = pytest.mark.gpu

ONE_PX = S.Intr(1.0, 1.0, 0.0, 0.0, 1, 1)


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


def both(V, cfg, cap=1 << 12):
    store = V.TwoTierStore(block_capacity=cap)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    return store, ref


def assert_equal(store, ref):
    got, want = store.export(), ref.export()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_keyframe_without_valid_pixels(V):
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    store, ref = both(V, cfg)
    rng = np.random.default_rng(1)
    f = S.random_frame(rng)
    f.weight[:] = 0.0  # volume.py:163: weight > 0 required
    pose = S.SPose(np.eye(3), [0.0, 0.0, 0.0])
    V.stream(store, pose.translation, cfg)
    ref.stream(pose.translation)
    rec = V.integrate(store, f, pose, cfg)
    _, touched, updated = ref.integrate(f, pose)
    assert (rec.blocks_touched, rec.voxels_updated, len(rec.new_blocks)) == (touched, updated, 0)
    V.deintegrate(store, f, pose, cfg)
    ref.deintegrate(f, pose)
    assert store.block_count() == 0
    assert_equal(store, ref)


def test_nonfinite_and_nonpositive_depths_are_skipped(V):
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    store, ref = both(V, cfg)
    rng = np.random.default_rng(2)
    f = S.random_frame(rng, holes=0.0)
    f.depth[0, :] = np.nan
    f.depth[1, :] = np.inf
    f.depth[2, :] = -1.0
    f.depth[3, :] = 0.0
    pose = S.SPose(S.rot_y(0.1), [0.02, 0.0, 0.0])
    V.stream(store, pose.translation, cfg)
    ref.stream(pose.translation)
    rec = V.integrate(store, f, pose, cfg)
    _, touched, updated = ref.integrate(f, pose)
    assert (rec.blocks_touched, rec.voxels_updated) == (touched, updated)
    assert touched > 0
    assert_equal(store, ref)


def test_one_pixel_image(V):
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    store, ref = both(V, cfg)
    f = S.Frame(np.array([[1.5]]), np.array([[2.0]]), np.array([[[10.0, 20.0, 30.0]]]), ONE_PX)
    pose = S.SPose(np.eye(3), [0.0, 0.0, 0.0])
    V.stream(store, pose.translation, cfg)
    ref.stream(pose.translation)
    rec = V.integrate(store, f, pose, cfg)
    _, touched, updated = ref.integrate(f, pose)
    assert (rec.blocks_touched, rec.voxels_updated) == (touched, updated)
    assert updated > 0
    assert_equal(store, ref)
    assert V.keyframe_block_footprint(f, pose, cfg) == ref.footprint(f, pose)


def test_empty_windows(V):
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    store, ref = both(V, cfg)
    rng = np.random.default_rng(3)
    f = S.random_frame(rng)
    pose = S.SPose(np.eye(3), [0.0, 0.0, 0.0])
    V.stream(store, pose.translation, cfg)
    ref.stream(pose.translation)
    V.integrate(store, f, pose, cfg)
    ref.integrate(f, pose)
    assert V.correct_windows(store, [], cfg) == 0
    assert V.correct_windows(store, [[], []], cfg) == 0
    # an empty window list with a next centre only streams
    assert V.correct_windows(store, [[]], cfg, next_center=np.array([0.5, 0.0, 0.0])) == 0
    ref.stream(np.array([0.5, 0.0, 0.0]))
    assert store.last_center[0] == 0.5
    assert_equal(store, ref)
