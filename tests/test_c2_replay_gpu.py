"""Parity at BASELINE scale: the bench's own C2 workload
-- corridor keyframes fused on the device from 5 rendered frames each, 5 mm
voxels, mu 0.06, stream radius 7 m -- replayed through top-k pose-graph
corrections (reintegration.select_topk + correct_topk, m = 4) on the device
and, from the same starting volume, in the CPU oracle (oracle/oracle.py,
the reference's algorithm restated; checker only).  The final volumes must
agree bit for bit (block set, D, W, C) and so must the streaming counters.

The starting volume is the device's (exported and loaded into the oracle):
the oracle cannot afford to build it, and the device build is itself
bit-exact against the reference (tests/test_volume_gpu.py, tools/bench_c4.py).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

N_KF = 8
EVENTS = 3
M = 4


class _Entry:
    def __init__(self, kf, integrated_pose, target_pose):
        self.kf, self.integrated_pose, self.target_pose = kf, integrated_pose, target_pose


class _HostKF:
    def __init__(self, kf):
        self.depth = kf.depth.cpu().numpy()
        self.weight = kf.weight.cpu().numpy()
        self.color = kf.color.cpu().numpy()
        self.intrinsics = kf.intrinsics


def _oracle_from(store, cfg):
    keys, d, w, c = store.export()
    st = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    st.last_center = store.last_center.copy()
    coords = O.keys_to_coords(keys)
    if coords:
        centers = (np.asarray(coords, dtype=np.float64) + 0.5) * st.span
        dist = np.linalg.norm(centers - st.last_center, axis=1)  # volume.py:341-348
        for i, cc in enumerate(coords):
            b = O.Block.__new__(O.Block)
            b.d, b.w, b.c = d[i], w[i], c[i]
            (st.active if dist[i] <= cfg.stream_radius else st.host)[cc] = b
    return st


def _oracle_export(st):
    blocks = dict(st.active)
    blocks.update(st.host)
    coords = sorted(blocks)
    keys = np.asarray([int(O.pack_coords(*cc)) for cc in coords], dtype=np.int64)
    order = np.argsort(keys, kind="stable")
    return (keys[order], np.stack([blocks[coords[j]].d for j in order]),
            np.stack([blocks[coords[j]].w for j in order]),
            np.stack([blocks[coords[j]].c for j in order]))


def test_c2_topk_replay_matches_oracle():
    import torch

    import bench as B
    from paper_1709_03763_b200 import geometry as G
    from paper_1709_03763_b200 import reintegration as R
    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    gt, gt_kf, drifted = B.kf_poses(B.N_FRAMES // B.KAPPA)  # the bench trajectory
    gt_kf, drifted = gt_kf[:N_KF], drifted[:N_KF]
    kfs = B.build_keyframes(N_KF, gt, drifted)
    cfg = V.VolumeConfig(voxel_size=B.VOXEL, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << 20)
    store = V.TwoTierStore(block_capacity=400_000)
    for kf, p in zip(kfs, drifted):
        V.stream(store, p.translation, cfg)
        V.integrate(store, kf, p, cfg)
    ost = _oracle_from(store, cfg)
    c0 = store.counters()
    host = {id(kf): _HostKF(kf) for kf in kfs}
    # anchors every 4 keyframes, events pull random anchors toward the truth
    saved = B.EVENT_EVERY_KF
    B.EVENT_EVERY_KF = 4
    try:
        scen = B.Scenario(R, G, SY, gt_kf, drifted, kfs,
                          B.make_events(-(-N_KF // 4), EVENTS, seed=5))
        scen.frac = 0.6
        for s in range(EVENTS):
            R.apply_pose_update(scen.ledger, scen.event(s))
            picks = R.select_topk(scen.ledger, M)
            ents = [scen.ledger.entries[j - 1] for j in picks]
            work = [_Entry(host[id(e.kf)], e.integrated_pose.copy(), e.target_pose.copy())
                    for e in ents]
            nxt = ents[0].target_pose.translation.copy()
            assert R.correct_topk(store, scen.ledger, picks, cfg, next_center=nxt) == len(picks)
            for e in work:  # correct_topk: one _correct_entries per pick
                ost.correct_entries([e])
            ost.stream(nxt)
    finally:
        B.EVENT_EVERY_KF = saved
    got, want = store.export(), _oracle_export(ost)
    assert len(want[0]) > 10_000
    assert np.array_equal(got[0], want[0])
    for a, b in zip(got[1:], want[1:]):
        assert np.array_equal(a, b)
    c1 = store.counters()
    assert c1.blocks_streamed_in - c0.blocks_streamed_in == ost.blocks_streamed_in
    assert c1.blocks_streamed_out - c0.blocks_streamed_out == ost.blocks_streamed_out
    assert c1.sphere_relocations - c0.sphere_relocations == ost.sphere_relocations
    store.close()
