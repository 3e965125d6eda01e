"""Routed footprints for hash-sharded volumes (rf_route):
shard r samples 1/G of every keyframe's pixel tiles and k_route stores each
distinct block key straight into its owner's inbox.  Emulated with G shard
stores on the one device of this run, each driven from its own thread as a
rank would be (connect_shards): the union of the shards must equal the
single-volume result bit for bit, errors must be raised on every shard, and
the inbox contract (route first, exactly the call's ops) must hold."""

import ctypes
import threading

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


def lockstep(stores, fn):
    """fn(rank, store) on every shard at once (one thread per shard); returns
    the per-shard results, re-raising nothing: exceptions are returned."""
    import torch

    out = [None] * len(stores)

    def run(r):
        torch.cuda.set_device(0)
        try:
            out[r] = fn(r, stores[r])
        except Exception as e:  # noqa: BLE001 -- compared by the test
            out[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(len(stores))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "shard thread hung"
    return out


def union_export(stores):
    parts = [s.export() for s in stores]
    keys = np.concatenate([p[0] for p in parts])
    order = np.argsort(keys, kind="stable")
    return [keys[order]] + [np.concatenate([p[i] for p in parts])[order] for i in (1, 2, 3)]


def assert_same(single, shards):
    want = single.export()
    got = union_export(shards)
    assert len(want[0]) > 0
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def scene(seed, n=3):
    rng = np.random.default_rng(seed)
    frames = [S.wall_frame(S.QVGA_INTR, 1.2 + 0.2 * i, rng=rng, tilt=0.2 * i, noise=0.0015,
                           holes=0.05) for i in range(n)]
    old = [S.SPose(S.rot_z(0.05 * i), [0.02 * i, 0.0, 0.1]) for i in range(n)]
    new = [S.SPose(S.rot_z(0.05 * i + 0.01), [0.02 * i + 0.02, 0.01, 0.1]) for i in range(n)]
    return frames, old, new


def make(V, G, cfg, cap=1 << 16, **kw):
    single = V.TwoTierStore(block_capacity=cap)
    shards = [V.TwoTierStore(block_capacity=cap, shard_rank=r, shard_count=G) for r in range(G)]
    V.connect_shards(shards, cfg, image=(320, 240), **kw)
    return single, shards


@pytest.mark.parametrize("G", [2, 3])
def test_routed_union_equals_single(V, G):
    from paper_1709_03763_b200 import _lib as L

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames, old, new = scene(99 + G)
    single, shards = make(V, G, cfg)
    want = []
    for f, p in zip(frames, old):
        V.stream(single, p.translation, cfg)
        want.append(V.integrate(single, f, p, cfg))

    def build(r, s):
        recs = []
        for f, p in zip(frames, old):
            V.stream(s, p.translation, cfg)
            recs.append(V.integrate(s, f, p, cfg))
        return recs

    recs = lockstep(shards, build)
    for rr in recs:
        assert not isinstance(rr, Exception), rr
    for k, w in enumerate(want):
        assert sum(r[k].voxels_updated for r in recs) == w.voxels_updated
        assert sum(r[k].blocks_touched for r in recs) == w.blocks_touched
        assert set().union(*[r[k].new_blocks for r in recs]) == w.new_blocks
    assert_same(single, shards)

    nc = np.array([0.3, 0.0, 0.0])
    V.correct_entries(single, [S.Entry(f, o.copy(), n.copy())
                               for f, o, n in zip(frames, old, new)], cfg, nc)
    out = lockstep(shards, lambda r, s: V.correct_entries(
        s, [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)], cfg, nc))
    assert out == [len(frames)] * G
    assert_same(single, shards)
    lib = L.lib()
    for r, s in enumerate(shards):
        assert all(lib.rf_key_owner(int(k), G) == r for k in s.export()[0])
    c1 = single.counters()
    cs = [s.counters() for s in shards]
    assert sum(c.blocks_streamed_in for c in cs) == c1.blocks_streamed_in
    assert sum(c.blocks_streamed_out for c in cs) == c1.blocks_streamed_out


def test_routed_windows_split_across_calls(V):
    """More windows than one routed call holds: the store splits them over
    several native calls (same on every shard); the result is unchanged."""
    G = 2
    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames, old, new = scene(5, n=4)
    single, shards = make(V, G, cfg, max_ops=4)  # two entries per call

    def run(s, lock):
        for f, p in zip(frames, old):
            V.stream(s, p.translation, cfg)
            V.integrate(s, f, p, cfg)
        ents = [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)]
        # correct_topk's shape: one window per entry, then finalize's runs
        n1 = V.correct_windows(s, [[e] for e in ents], cfg, np.array([0.1, 0.0, 0.1]))
        back = [S.Entry(f, n.copy(), o.copy()) for f, o, n in zip(frames, old, new)]
        n2 = V.correct_windows(s, [back[:2], back[2:]], cfg)
        return n1 + n2

    assert run(single, None) == 8
    assert lockstep(shards, lambda r, s: run(s, None)) == [8] * G
    assert_same(single, shards)
    with pytest.raises(ValueError):  # a window larger than the inboxes
        V.correct_windows(shards[0], [[S.Entry(frames[0], old[0], new[0])] * 3], cfg)


def test_routed_contract_error_is_global(V):
    """A footprint block outside the sphere raises on every shard; the partial
    allocation (keys below the violating one) matches the single volume."""
    from paper_1709_03763_b200.errors import StreamingContractError

    rng = np.random.default_rng(17)
    frame = S.random_frame(rng)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.08, stream_radius=1.2)
    single, shards = make(V, 3, cfg, cap=1 << 12)
    c = np.array([-1.0, 0.0, 1.5])
    V.stream(single, c, cfg)
    with pytest.raises(StreamingContractError):
        V.integrate(single, frame, S.identity(), cfg)

    def run(r, s):
        V.stream(s, c, cfg)
        V.integrate(s, frame, S.identity(), cfg)

    out = lockstep(shards, run)
    assert all(isinstance(e, StreamingContractError) for e in out), out
    assert_same(single, shards)


def test_routed_inbox_overflow_is_a_capacity_error(V):
    from paper_1709_03763_b200.errors import CapacityError

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames, old, _ = scene(3, n=1)
    _, shards = make(V, 2, cfg, cap_keys=64)

    def run(r, s):
        V.stream(s, old[0].translation, cfg)
        V.integrate(s, frames[0], old[0], cfg)

    out = lockstep(shards, run)
    assert all(isinstance(e, CapacityError) for e in out), out


def test_routed_call_without_route_is_rejected(V):
    """The native op of a connected shard refuses to run on stale inboxes."""
    from paper_1709_03763_b200 import _lib as L

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames, old, _ = scene(4, n=1)
    _, shards = make(V, 2, cfg)
    s = shards[0]
    view, keep = V.kf_view(frames[0], s.device)
    ps = V.pose_struct(old[0])
    res = L.RfOpResult()
    st = s._call_status("rf_integrate", ctypes.byref(view), ctypes.byref(ps), ctypes.byref(res),
                        None, 0)
    assert st == L.RF_INVALID_ARG
    del keep


@pytest.mark.parametrize("route", [True, False])
def test_shard_local_inconsistency_raises_everywhere(V, route):
    """A de-integration at a pose the keyframe was never integrated at fails
    on the shards owning the failing blocks; with the shards connected, every
    shard raises VolumeInconsistencyError (routed or replicated sampling)."""
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames, old, _ = scene(13, n=1)
    G = 2
    shards = [V.TwoTierStore(block_capacity=1 << 16, shard_rank=r, shard_count=G)
              for r in range(G)]
    V.connect_shards(shards, cfg, image=(320, 240), route=route)
    wrong = S.SPose(S.rot_z(0.3), [0.05, 0.02, 0.1])

    def run(r, s):
        V.stream(s, old[0].translation, cfg)
        V.integrate(s, frames[0], old[0], cfg)
        V.deintegrate(s, frames[0], wrong, cfg)

    out = lockstep(shards, run)
    assert all(isinstance(e, VolumeInconsistencyError) for e in out), out
