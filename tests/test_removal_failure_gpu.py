"""De-integration against the CPU oracle, bit for bit, on memo-resolved and
sampled footprints: the success path, a removal that fails part-way
(removing a keyframe twice: blocks sorted before the first failing block
removed and re-added, the rest untouched -- volume.py:315-338), and a
correction window that rolls back (reintegration.py:156-181).  The
per-operation profile counters are checked on the way."""

import ctypes

import numpy as np
import pytest

import oracle as O
import scenarios as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


def _same(store, ref):
    got, want = store.export(), ref.export()
    assert np.array_equal(got[0], want[0]), "block sets differ"
    for name, a, b in zip("dwc", got[1:], want[1:]):
        assert np.array_equal(a, b), f"{name}: {int((a != b).sum())} values differ"


class _Prof:
    """rf_profile around a few calls."""

    def __init__(self, store):
        self.s = store

    def __enter__(self):
        self.s._call("rf_profile_begin")
        return self

    def __exit__(self, *exc):
        from paper_1709_03763_b200 import _lib as L

        self.p = L.RfProfile()
        self.s._call("rf_profile_end", ctypes.byref(self.p))


def _scene(seed, vs=0.005, n=3):
    rng = np.random.default_rng(seed)
    frames = [S.wall_frame(S.VGA_INTR, 1.3 + 0.1 * i, rng=rng, tilt=0.15 * i, noise=0.0015,
                           holes=0.05) for i in range(n)]
    poses = [S.SPose(S.rot_z(0.04 * i) @ S.rot_y(0.02 * i), [0.03 * i, 0.01, 0.1])
             for i in range(n)]
    return frames, poses


def _build(V, cfg, frames, poses):
    store = V.TwoTierStore(block_capacity=1 << 16)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    for f, p in zip(frames, poses):
        V.stream(store, p.translation, cfg)
        V.integrate(store, f, p, cfg)
        ref.stream(p.translation)
        ref.integrate(f, p)
    return store, ref


@pytest.mark.parametrize("vs", [0.01, 0.005])
def test_removal_bitexact(V, vs):
    cfg = V.VolumeConfig(voxel_size=vs, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    frames, poses = _scene(11, vs)
    store, ref = _build(V, cfg, frames, poses)
    with _Prof(store) as pr:
        for i in (1, 0):
            V.deintegrate(store, frames[i], poses[i], cfg)
            ref.deintegrate(frames[i], poses[i])
    assert pr.p.removal_ops == 2 and pr.p.removal_voxels > 0
    assert pr.p.integrate_launches == 0 and pr.p.removal_ms > 0
    _same(store, ref)
    assert V.garbage_collect(store) == ref.garbage_collect()
    _same(store, ref)


def test_removal_failure_restores_like_reference(V):
    """Removing a keyframe twice: the second removal fails part-way; the blocks sorted before the first failing one are
    removed and re-added, the rest untouched."""
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    frames, poses = _scene(23)
    store, ref = _build(V, cfg, frames, poses)
    V.deintegrate(store, frames[1], poses[1], cfg)
    ref.deintegrate(frames[1], poses[1])
    with _Prof(store) as pr:
        with pytest.raises(VolumeInconsistencyError):
            V.deintegrate(store, frames[1], poses[1], cfg)
    with pytest.raises(O.VolumeInconsistencyError):
        ref.deintegrate(frames[1], poses[1])
    assert pr.p.removal_ops == 1
    _same(store, ref)
    # still consistent afterwards
    V.deintegrate(store, frames[0], poses[0], cfg)
    ref.deintegrate(frames[0], poses[0])
    _same(store, ref)


def test_window_rollback_matches_oracle(V):
    """A window whose second entry fails (its keyframe was already removed):
    entry 0's removal is rolled back by re-integration."""
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    frames, poses = _scene(31)
    store, ref = _build(V, cfg, frames, poses)
    V.deintegrate(store, frames[2], poses[2], cfg)
    ref.deintegrate(frames[2], poses[2])
    new = [S.SPose(S.rot_z(0.04 * i + 0.01), [0.03 * i + 0.01, 0.0, 0.1]) for i in range(3)]
    ents = [S.Entry(frames[i], poses[i].copy(), new[i].copy()) for i in (0, 2)]
    rents = [S.Entry(frames[i], poses[i].copy(), new[i].copy()) for i in (0, 2)]
    with pytest.raises(VolumeInconsistencyError):
        V.correct_entries(store, ents, cfg, np.array([0.1, 0.0, 0.1]))
    with pytest.raises(O.VolumeInconsistencyError):
        ref.correct_entries(rents)
    _same(store, ref)
    for e in ents:
        assert np.array_equal(e.integrated_pose.translation, e.target_pose.translation) is False


def test_sampled_footprint_removal_matches_oracle(V):
    """Without the memo every footprint is sampled (same result)."""
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    frames, poses = _scene(41)
    store, ref = _build(V, cfg, frames, poses)
    store._call("rf_set_memo_budget", 0)  # no memo: every footprint is sampled
    with _Prof(store) as pr:
        V.deintegrate(store, frames[0], poses[0], cfg)
    ref.deintegrate(frames[0], poses[0])
    assert pr.p.removal_ops == 1
    _same(store, ref)
