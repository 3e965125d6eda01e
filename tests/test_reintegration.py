"""Correction scheduler: host selection logic (CPU) and device corrections
(GPU), following the reference's tests/test_reintegration.py."""

import numpy as np
import pytest

import oracle as O
import scenarios as S
from paper_1709_03763_b200 import reintegration as R
from paper_1709_03763_b200.errors import MalformedEventError, VolumeInconsistencyError
from paper_1709_03763_b200.geometry import Pose, compose, pose_distance, rotation_z

INTR = S.SMALL_INTR


def x_pose(x):
    return Pose(np.eye(3), np.array([float(x), 0.0, 0.0]))


def ledger_with_distances(dvec):
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, Pose.identity())
    for i, d in enumerate(dvec):
        e = ledger.add(None, i + 1, 0, x_pose(0.0), x_pose(0.0))
        e.target_pose = x_pose(d)
    return ledger


FIG_DISTANCES = [0.05, 0.05, 0.5, 0.45, 0.55, 0.40, 0.42, 0.70,
                 0.05, 0.05, 0.05, 0.90, 0.60, 0.05, 0.05]


# ---------------------------------------------------------------------------
# host logic (CPU)


def brute_window(d, m):
    k = len(d)
    length = min(m, k)
    best, arg = -1.0, None
    for j in range(k - length + 1):
        s = 0.0
        for off in range(length):
            s += d[j + off]
        if s > best:
            best, arg = s, j
    return None if best < R.EPS_MOVE else arg + 1


def test_select_window_fig4():
    ledger = ledger_with_distances(FIG_DISTANCES)
    assert R.select_window(ledger, 6) == 3
    assert R.select_topk(ledger, 3) == [12, 8, 13]


def test_select_window_matches_brute_force():
    rng = np.random.default_rng(99)
    for _ in range(300):
        k = int(rng.integers(1, 30))
        d = rng.uniform(0.0, 1.0, k)
        d[rng.random(k) < 0.3] = 0.0
        ledger = ledger_with_distances(d)
        m = int(rng.integers(1, 12))
        assert R.select_window(ledger, m) == brute_window(ledger.distances(), m)


def test_select_window_nothing_moved():
    assert R.select_window(ledger_with_distances([0.0, 0.0]), 2) is None
    assert R.select_window(R.IntegrationLedger(), 3) is None
    with pytest.raises(ValueError):
        R.select_window(ledger_with_distances([1.0]), 0)


def test_topk_stable_ties():
    ledger = ledger_with_distances([0.3, 0.5, 0.3, 0.5])
    assert R.select_topk(ledger, 4) == [2, 4, 1, 3]


def test_apply_pose_update_anchor_relative():
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, Pose.identity())
    ledger.declare_anchor(1, x_pose(1.0))
    ledger.add(None, 1, 0, x_pose(0.0), x_pose(0.0))
    ledger.add(None, 2, 1, x_pose(0.0), x_pose(1.0))
    ev = R.PoseUpdateEvent(at_frame=3, anchor_poses={1: x_pose(1.3)})
    assert R.apply_pose_update(ledger, ev) == 1
    d = ledger.distances()
    assert d[0] == 0.0 and abs(d[1] - 0.3) < 1e-12
    assert R.apply_pose_update(ledger, ev) == 0


def test_event_validation():
    with pytest.raises(MalformedEventError):
        R.PoseUpdateEvent(at_frame=0)
    with pytest.raises(MalformedEventError):
        R.PoseUpdateEvent(at_frame=1, anchor_poses={0: "not a pose"})
    ledger = R.IntegrationLedger()
    with pytest.raises(MalformedEventError):
        ledger.anchor_pose(7)


# ---------------------------------------------------------------------------
# device corrections (GPU)


def make_volume_ledger(V, cfg, rng, n_entries=3):
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, Pose.identity())
    store = V.TwoTierStore(block_capacity=1 << 14)
    V.stream(store, np.zeros(3), cfg)
    for i in range(n_entries):
        kf = S.random_frame(rng)
        pose = x_pose(0.05 * i)
        V.stream(store, pose.translation, cfg)
        rec = V.integrate(store, kf, pose, cfg)
        ledger.add(kf, i + 1, 0, pose.copy(), rec.pose)
    return store, ledger


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


CFG_ARGS = dict(voxel_size=0.01, mu=0.06, stream_radius=4.0)


@pytest.mark.gpu
def test_identity_window_correction_is_noop(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    store, ledger = make_volume_ledger(V, cfg, np.random.default_rng(23))
    before = dict(store.iter_blocks())
    assert R.correct_window(store, ledger, 1, 3, cfg) == 3
    for coord, blk in store.iter_blocks():
        assert np.abs(blk.d - before[coord].d).max() <= 1e-9
        assert np.abs(blk.w - before[coord].w).max() <= 1e-12


@pytest.mark.gpu
def test_single_entry_correction_matches_fresh_integration(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    rng = np.random.default_rng(29)
    kf = S.random_frame(rng)
    old, new = x_pose(0.0), Pose(np.eye(3), np.array([0.15, 0.05, 0.0]))
    store = V.TwoTierStore(block_capacity=1 << 14)
    V.stream(store, old.translation, cfg)
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, Pose.identity())
    rec = V.integrate(store, kf, old, cfg)
    entry = ledger.add(kf, 1, 0, old, rec.pose)
    entry.target_pose = new.copy()
    assert R.correct_window(store, ledger, 1, 1, cfg) == 1
    assert pose_distance(entry.integrated_pose, entry.target_pose) < R.EPS_MOVE
    fresh = V.TwoTierStore(block_capacity=1 << 14)
    V.stream(fresh, new.translation, cfg)
    V.integrate(fresh, kf, new, cfg)
    dd, dc, dw = V.compare_volumes(store, fresh)
    assert dd <= 1e-9 and dc <= 1e-9 and dw <= 1e-12


@pytest.mark.gpu
def test_correction_abort_restores_volume(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    store, ledger = make_volume_ledger(V, cfg, np.random.default_rng(31), n_entries=2)
    ledger.entries[1].integrated_pose = x_pose(2.5)
    ledger.entries[1].target_pose = x_pose(2.6)
    ledger.entries[0].target_pose = x_pose(0.02)
    before = dict(store.iter_blocks())
    with pytest.raises(VolumeInconsistencyError):
        R.correct_window(store, ledger, 1, 2, cfg)
    for coord, blk in store.iter_blocks():
        old = before.get(coord)
        if old is None:
            assert not blk.w.any()
            continue
        assert np.abs(blk.d - old.d).max() <= 1e-9
        assert np.abs(blk.w - old.w).max() <= 1e-12
    assert np.array_equal(ledger.entries[0].integrated_pose.translation, np.zeros(3))


@pytest.mark.gpu
def test_correct_window_returns_sphere_to_next_center(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    store, ledger = make_volume_ledger(V, cfg, np.random.default_rng(37), n_entries=2)
    nxt = np.array([0.5, 0.0, 0.0])
    R.correct_window(store, ledger, 1, 2, cfg, next_center=nxt)
    assert np.array_equal(store.last_center, nxt)


@pytest.mark.gpu
def test_finalize_all_moved_matches_rebuild(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    store, ledger = make_volume_ledger(V, cfg, np.random.default_rng(43), n_entries=4)
    assert R.finalize(store, ledger, cfg) == 0
    shift = Pose(np.eye(3), np.array([0.0, 0.12, 0.0]))
    R.apply_pose_update(ledger, R.PoseUpdateEvent(at_frame=99, anchor_poses={0: shift}))
    assert R.finalize(store, ledger, cfg, m=2) == 4
    assert all(d < R.EPS_MOVE for d in ledger.distances())
    fresh = V.TwoTierStore(block_capacity=1 << 14)
    V.stream(fresh, np.zeros(3), cfg)
    for e in ledger.entries:
        V.stream(fresh, e.target_pose.translation, cfg)
        V.integrate(fresh, e.kf, e.target_pose, cfg)
    dd, dc, dw = V.compare_volumes(store, fresh)
    assert dd <= 1e-9 and dc <= 1e-9 and dw <= 1e-12


@pytest.mark.gpu
def test_topk_batch_equals_sequential_oracle_bitexact(V):
    """correct_topk runs all picks in one native batch; the result must be
    bit-identical to the reference's one-_correct_entries-per-pick order."""
    cfg = V.VolumeConfig(**CFG_ARGS)
    rng = np.random.default_rng(47)
    frames = [S.random_frame(rng) for _ in range(5)]
    old = [S.SPose(rotation_z(0.02 * i), [0.04 * i, 0.0, 0.0]) for i in range(5)]
    new = [S.SPose(rotation_z(0.02 * i + 0.01), [0.04 * i + 0.03, 0.01, 0.0]) for i in range(5)]
    store = V.TwoTierStore(block_capacity=1 << 14)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, Pose.identity())
    for i, (f, p) in enumerate(zip(frames, old)):
        V.stream(store, p.translation, cfg)
        V.integrate(store, f, p, cfg)
        ref.stream(p.translation)
        ref.integrate(f, p)
        e = ledger.add(f, i + 1, 0, Pose(p.rotation, p.translation), Pose(p.rotation, p.translation))
        e.target_pose = Pose(new[i].rotation, new[i].translation)
    picks = [4, 1, 3]
    nxt = np.array([0.1, 0.2, 0.0])
    assert R.correct_topk(store, ledger, picks, cfg, next_center=nxt) == 3
    for j in picks:
        ref.correct_entries([S.Entry(frames[j - 1], old[j - 1].copy(), new[j - 1].copy())])
    ref.stream(nxt)
    got, want = store.export(), ref.export()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    c = store.counters()
    assert (c.blocks_streamed_in, c.blocks_streamed_out, c.sphere_relocations) == (
        ref.blocks_streamed_in, ref.blocks_streamed_out, ref.sphere_relocations)


@pytest.mark.gpu
def test_weight_conserved_through_correction(V):
    cfg = V.VolumeConfig(**CFG_ARGS)
    store, ledger = make_volume_ledger(V, cfg, np.random.default_rng(53))
    shift = Pose(np.eye(3), np.array([0.03, 0.0, 0.0]))
    R.apply_pose_update(ledger, R.PoseUpdateEvent(at_frame=9, anchor_poses={0: shift}))
    j = R.select_window(ledger, 3)
    assert j == 1
    R.correct_window(store, ledger, j, 3, cfg)
    fresh = V.TwoTierStore(block_capacity=1 << 14)
    V.stream(fresh, np.zeros(3), cfg)
    for e in ledger.entries:
        V.stream(fresh, e.integrated_pose.translation, cfg)
        V.integrate(fresh, e.kf, e.integrated_pose, cfg)
    total, want = V.total_weight(store), V.total_weight(fresh)
    assert abs(total - want) <= 1e-9 * max(want, 1.0)
