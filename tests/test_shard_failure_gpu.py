"""All-or-nothing de-integration across hash shards (VERDICT r1 item 2,
ADVICE r1 high): a removal that fails on the shards owning the failing
blocks must leave the UNION of the shards exactly where one volume would be
-- blocks sorted before the globally first failing block removed and
re-added, the rest untouched (volume.py:315-338), and inside a correction
window the already-removed entries re-integrated (reintegration.py:
166-174).  G shards emulated on the one device, each driven from its own
thread, replicated and routed footprints; the single volume is the
reference (itself bit-exact vs the oracle, tests/test_volume_gpu.py)."""

import numpy as np
import pytest

import scenarios as S
from test_routing_gpu import lockstep, union_export

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


def _scene(seed, n=3):
    rng = np.random.default_rng(seed)
    frames = [S.wall_frame(S.QVGA_INTR, 1.2 + 0.2 * i, rng=rng, tilt=0.2 * i, noise=0.0015,
                           holes=0.05) for i in range(n)]
    old = [S.SPose(S.rot_z(0.05 * i), [0.02 * i, 0.0, 0.1]) for i in range(n)]
    new = [S.SPose(S.rot_z(0.05 * i + 0.01), [0.02 * i + 0.02, 0.01, 0.1]) for i in range(n)]
    return frames, old, new


def _setup(V, G, route, cfg, frames, old):
    single = V.TwoTierStore(block_capacity=1 << 16)
    shards = [V.TwoTierStore(block_capacity=1 << 16, shard_rank=r, shard_count=G)
              for r in range(G)]
    V.connect_shards(shards, cfg, image=(320, 240), route=route)
    for f, p in zip(frames, old):
        V.stream(single, p.translation, cfg)
        V.integrate(single, f, p, cfg)

    def build(r, s):
        for f, p in zip(frames, old):
            V.stream(s, p.translation, cfg)
            V.integrate(s, f, p, cfg)

    assert all(o is None for o in lockstep(shards, build))
    return single, shards


def _assert_union(single, shards):
    want = single.export()
    got = union_export(shards)
    assert len(want[0]) > 0
    assert np.array_equal(got[0], want[0]), "block sets differ"
    for name, a, b in zip("dwc", got[1:], want[1:]):
        assert np.array_equal(a, b), f"{name}: {int((a != b).sum())} voxels differ"


CFG = dict(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)


@pytest.mark.parametrize("G,route", [(2, False), (3, False), (2, True), (3, True)])
def test_failed_deintegration_union_equals_single(V, G, route):
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    cfg = V.VolumeConfig(**CFG)
    frames, old, _ = _scene(31 + G)
    single, shards = _setup(V, G, route, cfg, frames, old)
    wrong = S.SPose(S.rot_z(0.02), [0.015, 0.004, 0.1])  # overlaps, never integrated
    with pytest.raises(VolumeInconsistencyError):
        V.deintegrate(single, frames[0], wrong, cfg)
    out = lockstep(shards, lambda r, s: V.deintegrate(s, frames[0], wrong, cfg))
    assert all(isinstance(e, VolumeInconsistencyError) for e in out), out
    _assert_union(single, shards)
    # the volume stays usable: a consistent correction afterwards agrees too
    V.deintegrate(single, frames[1], old[1], cfg)
    lockstep(shards, lambda r, s: V.deintegrate(s, frames[1], old[1], cfg))
    _assert_union(single, shards)


@pytest.mark.parametrize("G,route", [(2, False), (3, False), (2, True)])
@pytest.mark.parametrize("bad", [0, 1, 2])
def test_failed_window_union_equals_single(V, G, route, bad):
    """A correction window whose entry `bad` holds a pose it was never
    integrated at: every shard raises at the same entry, re-integrates the
    entries removed before it, and the ledger is untouched -- the union of
    the shards equals the single volume bit for bit."""
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    cfg = V.VolumeConfig(**CFG)
    frames, old, new = _scene(41 + G + 7 * bad)
    single, shards = _setup(V, G, route, cfg, frames, old)
    claimed = [p.copy() for p in old]
    claimed[bad] = S.SPose(S.rot_z(0.05 * bad + 0.02), [0.02 * bad + 0.012, 0.004, 0.1])

    def entries():
        return [S.Entry(f, c.copy(), n.copy()) for f, c, n in zip(frames, claimed, new)]

    e1 = entries()
    with pytest.raises(VolumeInconsistencyError):
        V.correct_entries(single, e1, cfg, np.array([0.3, 0.0, 0.0]))
    ents = [entries() for _ in shards]
    out = lockstep(shards, lambda r, s: V.correct_entries(s, ents[r], cfg,
                                                          np.array([0.3, 0.0, 0.0])))
    assert all(isinstance(e, VolumeInconsistencyError) for e in out), out
    _assert_union(single, shards)
    for es in ents:
        for a, b in zip(es, e1):
            assert np.array_equal(a.integrated_pose.translation, b.integrated_pose.translation)
    c1 = single.counters()
    cs = [s.counters() for s in shards]
    assert sum(c.blocks_streamed_in for c in cs) == c1.blocks_streamed_in
    assert sum(c.blocks_streamed_out for c in cs) == c1.blocks_streamed_out


def test_failed_topk_batch_union_equals_single(V):
    """correct_topk's back-to-back single-entry windows in one native batch:
    the second pick fails; the first stays corrected on every shard."""
    from paper_1709_03763_b200.errors import VolumeInconsistencyError

    G = 2
    cfg = V.VolumeConfig(**CFG)
    frames, old, new = _scene(77)
    single, shards = _setup(V, G, False, cfg, frames, old)
    claimed = [p.copy() for p in old]
    claimed[1] = S.SPose(S.rot_z(0.07), [0.032, 0.004, 0.1])

    def windows():
        return [[S.Entry(frames[i], claimed[i].copy(), new[i].copy())] for i in range(3)]

    w1 = windows()
    with pytest.raises(VolumeInconsistencyError):
        V.correct_windows(single, w1, cfg)
    ws = [windows() for _ in shards]
    out = lockstep(shards, lambda r, s: V.correct_windows(s, ws[r], cfg))
    assert all(isinstance(e, VolumeInconsistencyError) for e in out), out
    _assert_union(single, shards)
    for w in ws:
        assert np.array_equal(w[0][0].integrated_pose.translation, new[0].translation)
        assert np.array_equal(w[1][0].integrated_pose.translation, claimed[1].translation)
