"""Keyframes held in host memory (pinned torch tensors and plain numpy): the
library stages them through a ring of device slots on its copy stream and the
kernels wait on per-slot upload flags (no stream event waits).  A correction
batch with more keyframes than the ring's 16 slots (the ring and its flags
grow), followed by smaller batches that refill the slots, must give the same
volume, bit for bit, as the same corrections on resident (device) keyframes."""

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


class _KF:
    def __init__(self, f, depth, weight, color):
        self.depth, self.weight, self.color, self.intrinsics = depth, weight, color, f.intrinsics


def _frames(n):
    rng = np.random.default_rng(123)
    return [S.wall_frame(S.QVGA_INTR, 1.1 + 0.04 * i, rng=rng, tilt=0.05 * (i % 7), noise=0.001,
                         holes=0.03) for i in range(n)]


def _run(V, kfs, cfg):
    n = len(kfs)
    old = [S.SPose(S.rot_z(0.01 * i), [0.004 * i, 0.0, 0.1]) for i in range(n)]
    new = [S.SPose(S.rot_z(0.01 * i + 0.003), [0.004 * i + 0.002, 0.001, 0.1]) for i in range(n)]
    store = V.TwoTierStore(block_capacity=1 << 16)
    for kf, p in zip(kfs, old):
        V.stream(store, p.translation, cfg)
        V.integrate(store, kf, p, cfg)
    ents = [S.Entry(kf, o.copy(), nw.copy()) for kf, o, nw in zip(kfs, old, new)]
    # one batch of 20 single-entry windows (> 16 staging slots), then two
    # smaller batches back to the old poses
    V.correct_windows(store, [[e] for e in ents], cfg)
    back = [S.Entry(e.kf, e.integrated_pose.copy(), o.copy()) for e, o in zip(ents, old)]
    V.correct_windows(store, [[e] for e in back[:5]], cfg)
    V.correct_windows(store, [back[5:12]], cfg)
    return store.export()


def test_staged_host_keyframes_match_resident(V):
    import torch

    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    frames = _frames(20)
    dev = [_KF(f, torch.from_numpy(f.depth).cuda(), torch.from_numpy(f.weight).cuda(),
               torch.from_numpy(f.color).cuda()) for f in frames]
    pinned = [_KF(f, torch.from_numpy(f.depth).pin_memory(), torch.from_numpy(f.weight).pin_memory(),
                  torch.from_numpy(f.color).pin_memory()) for f in frames]
    pageable = [_KF(f, f.depth.copy(), f.weight.copy(), f.color.copy()) for f in frames]
    want = _run(V, dev, cfg)
    for kfs in (pinned, pageable):
        got = _run(V, kfs, cfg)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
