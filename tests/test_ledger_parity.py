"""Host scheduler parity (no GPU): the memoised apply_pose_update / distances
give the reference's targets, change counts, distances and picks bit for
bit, over 1,000 random ledgers with repeated events and corrections
(reference: reintegration.py:95-153, run from oracle/_ref)."""

import numpy as np
import pytest

from paper_1709_03763_b200 import geometry as G
from paper_1709_03763_b200 import reintegration as R
from refimport import REF, reference

pytestmark = pytest.mark.skipif(reference() is None, reason="oracle/_ref not built")


def _ref():
    reference()
    import refusion.geometry as RG
    import refusion.reintegration as RR
    return RG, RR


def _rand_pose(rng, scale=1.0):
    ax = rng.normal(size=3)
    R_ = G.Pose.identity().rotation
    from paper_1709_03763_b200.synth import axis_angle_rotation
    R_ = axis_angle_rotation(ax, rng.uniform(-np.pi, np.pi) * scale)
    return R_, rng.normal(size=3) * 3.0 * scale


@pytest.mark.parametrize("chunk", range(10))
def test_random_ledgers_match_reference(chunk):
    RG, RR = _ref()
    for case in range(100):
        rng = np.random.default_rng(1000 * chunk + case)
        n_anchor = int(rng.integers(1, 8))
        n_entry = int(rng.integers(1, 40))
        mine, ref = R.IntegrationLedger(), RR.IntegrationLedger()
        for a in range(n_anchor):
            Ra, ta = _rand_pose(rng)
            mine.declare_anchor(a, G.Pose(Ra, ta))
            ref.declare_anchor(a, RG.Pose(Ra, ta))
        for k in range(n_entry):
            a = int(rng.integers(0, n_anchor))
            Rr, tr = _rand_pose(rng, 0.3)
            Ri, ti = _rand_pose(rng)
            mine.add(object(), k + 1, a, G.Pose(Rr, tr), G.Pose(Ri, ti))
            ref.add(object(), k + 1, a, RG.Pose(Rr, tr), RG.Pose(Ri, ti))
        for ev in range(4):
            upd_m, upd_r = {}, {}
            for a in rng.choice(n_anchor, size=int(rng.integers(0, n_anchor + 1)), replace=False):
                Ra, ta = _rand_pose(rng)
                upd_m[int(a)] = G.Pose(Ra, ta)
                upd_r[int(a)] = RG.Pose(Ra, ta)
            cm = R.apply_pose_update(mine, R.PoseUpdateEvent(at_frame=ev + 1, anchor_poses=upd_m))
            cr = RR.apply_pose_update(ref, RR.PoseUpdateEvent(at_frame=ev + 1, anchor_poses=upd_r))
            assert cm == cr
            for em, er in zip(mine.entries, ref.entries):
                assert np.array_equal(em.target_pose.rotation, er.target_pose.rotation)
                assert np.array_equal(em.target_pose.translation, er.target_pose.translation)
            dm, dr = mine.distances(), ref.distances()
            assert np.array_equal(dm, dr)
            m = int(rng.integers(1, 6))
            assert R.select_topk(mine, m) == RR.select_topk(ref, m)
            assert R.select_window(mine, m) == RR.select_window(ref, m)
            # a correction moves the picked entries to their targets
            for j in R.select_topk(mine, m):
                mine.entries[j - 1].integrated_pose = mine.entries[j - 1].target_pose.copy()
                ref.entries[j - 1].integrated_pose = ref.entries[j - 1].target_pose.copy()
            assert np.array_equal(mine.distances(), ref.distances())
