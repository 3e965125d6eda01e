"""the faithful port of the reference's synthetic generator
(/root/reference/pkg/src/refusion/synth.py:220-390).  The checker is the
unmodified reference compiled into oracle/_ref (tests/refimport.py), run on
the same host: depth, noisy depth, colour, blur, trajectories and events
must be bit-identical.  CPU tests cover the host-side trajectory and pose
algebra; the -m gpu tests render on the device."""

import numpy as np
import pytest

from refimport import reference

from paper_1709_03763_b200 import geometry as G
from paper_1709_03763_b200 import synth as S

REF = reference()
pytestmark = pytest.mark.skipif(REF is None, reason="oracle/_ref (reference build) absent")


def _rs():
    import refusion.synth as RS

    return RS


def _rpose(p):
    return REF["G"].Pose(p.rotation, p.translation)


def _rintr(i):
    return REF["G"].Intrinsics(fx=i.fx, fy=i.fy, cx=i.cx, cy=i.cy, width=i.width,
                               height=i.height)


def _same_pose(a, b):
    return np.array_equal(a.rotation, b.rotation) and np.array_equal(a.translation, b.translation)


def _ref_scene(scene):
    RS = _rs()
    prims = []
    for p in scene.prims():
        if p.kind == S.SPHERE:
            prims.append(RS.Sphere(center=p.center, radius=p.size[0], albedo=p.albedo))
        elif p.kind == S.BOX:
            prims.append(RS.BoxSolid(center=p.center, half_extents=p.size, albedo=p.albedo))
        else:
            prims.append(RS.RoomShell(center=p.center, half_extents=p.size, albedo=p.albedo))
    return RS.AnalyticScene(primitives=prims)


def _small_intr(w, h):
    s = w / 640.0
    return G.Intrinsics(fx=525.0 * s, fy=525.0 * s, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0,
                        width=w, height=h)


# ---------------------------------------------------------------------------
# host side (CPU)


def test_waypoints_and_pose_at_match_reference():
    RS = _rs()
    ours = S.orbit_waypoints(7)
    ref = RS.orbit_waypoints(7)
    assert all(_same_pose(a, b) for a, b in zip(ours, ref))
    inward = S.orbit_waypoints(4, outward=False, center=(0.3, -0.2))
    assert all(_same_pose(a, b) for a, b in
               zip(inward, RS.orbit_waypoints(4, outward=False, center=(0.3, -0.2))))
    spec = S.TrajectorySpec(waypoints=ours, frames_per_segment=5)
    rspec = RS.TrajectorySpec(waypoints=ref, frames_per_segment=5)
    assert spec.n_frames == rspec.n_frames
    for i in range(1, spec.n_frames + 1):
        assert _same_pose(spec.pose_at(i), rspec.pose_at(i)), i


def test_exact_pose_algebra_matches_reference():
    RG = REF["G"]
    rng = np.random.default_rng(5)
    for _ in range(50):
        ax = rng.normal(size=3)
        ang = rng.uniform(-3.2, 3.2)
        assert np.array_equal(G.rotation_from_axis_angle(ax, ang),
                              RG.rotation_from_axis_angle(ax, ang))
        R = RG.rotation_from_axis_angle(ax, ang)
        a1, t1 = G.axis_angle_from_rotation(R)
        a2, t2 = RG.axis_angle_from_rotation(R)
        assert t1 == t2 and np.array_equal(a1, a2)
    # the angle-pi branch
    R = RG.rotation_from_axis_angle([0.3, 0.4, 0.5], np.pi)
    assert np.array_equal(G.axis_angle_from_rotation(R)[0], RG.axis_angle_from_rotation(R)[0])


def test_add_noise_and_scene_sdf_match_reference():
    RS = _rs()
    rng = np.random.default_rng(3)
    d = rng.uniform(0.0, 4.0, size=(30, 40))
    d[d < 0.5] = 0.0
    for seed in [(0, 7, 1), (1, 7, 12), 5]:
        assert np.array_equal(S.add_noise(d, seed=seed), RS.add_noise(d, seed=seed))
    assert np.array_equal(S.add_noise(d, seed=1, sigma0=0.0), d)
    scene = S.AnalyticScene(S.corridor_scene())
    pts = rng.uniform(-1.0, 3.0, size=(500, 3)) + np.array([5.0, 0.0, 0.0])
    assert np.array_equal(scene.sdf(pts), _ref_scene(scene).sdf(pts))


def test_render_orders_are_calibrated():
    gemm, gemv = S.detect_render_orders()
    assert gemm in (0, 1, 2, 3) and gemv in (0, 1, 2, 3)


# ---------------------------------------------------------------------------
# device renderer (GPU) vs the reference renderer on the same host


def _views(n=4):
    return S.orbit_waypoints(n)[:n]


@pytest.mark.gpu
@pytest.mark.parametrize("w,h", [(96, 72), (160, 120)])
def test_render_depth_and_color_bitexact(w, h):
    RS = _rs()
    scene = S.reference_demo_scene()
    rscene = RS.demo_scene()
    intr = _small_intr(w, h)
    for k, pose in enumerate(_views(4)):
        ref_d = RS.render_depth(rscene, _rpose(pose), _rintr(intr))
        got_d = S.render_depth(scene, pose, intr)
        assert np.array_equal(got_d, ref_d), (k, int((got_d != ref_d).sum()))
        assert (ref_d > 0).mean() > 0.5
        noisy = RS.add_noise(ref_d, seed=(0, 7, k + 1), sigma0=0.0015)
        ref_c = RS.render_color(rscene, _rpose(pose), _rintr(intr), noisy)
        got_c = S.render_color(scene, pose, intr, noisy)
        assert np.array_equal(got_c, ref_c), (k, int((got_c != ref_c).any(axis=-1).sum()))


@pytest.mark.gpu
def test_render_corridor_many_primitives_bitexact():
    RS = _rs()
    scene = S.AnalyticScene(S.corridor_scene())
    rscene = _ref_scene(scene)
    intr = _small_intr(128, 96)
    for x in (2.0, 9.5, 21.0):
        pose = S.look_at_pose((x, 0.2, 1.5), (x + 1.0, 0.35, 1.4))
        ref_d = RS.render_depth(rscene, _rpose(pose), _rintr(intr), z_max=5.0)
        got_d = S.render_depth(scene, pose, intr, z_max=5.0)
        assert np.array_equal(got_d, ref_d), (x, int((got_d != ref_d).sum()))
        ref_c = RS.render_color(rscene, _rpose(pose), _rintr(intr), ref_d)
        got_c = S.render_color(scene, pose, intr, ref_d)
        assert np.array_equal(got_c, ref_c), x


@pytest.mark.gpu
def test_render_full_vga_frame_bitexact():
    RS = _rs()
    pose = _views(9)[2]
    intr = S.DEFAULT_INTRINSICS
    ref_d = RS.render_depth(RS.demo_scene(), _rpose(pose), _rintr(intr))
    got_d = S.render_depth(S.reference_demo_scene(), pose, intr)
    assert np.array_equal(got_d, ref_d), int((got_d != ref_d).sum())


@pytest.mark.gpu
def test_gaussian_blur_matches_scipy():
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(8)
    c = rng.uniform(0.0, 255.0, size=(37, 53, 3))
    for sigma in (0.3, 0.9, 1.7, 4.2):
        ref = gaussian_filter(c, sigma=(sigma, sigma, 0.0))
        got = S.gaussian_blur(c, sigma)
        assert np.array_equal(got, ref), sigma


@pytest.mark.gpu
def test_make_sequence_bitexact():
    RS = _rs()
    intr = _small_intr(64, 48)
    sched = [(4, 0.5), (7, 1.0)]
    spec = S.TrajectorySpec(waypoints=S.orbit_waypoints(3), frames_per_segment=3,
                            drift_rate=(0.002, 0.001), correction_schedule=sched)
    rspec = RS.TrajectorySpec(waypoints=RS.orbit_waypoints(3), frames_per_segment=3,
                              drift_rate=(0.002, 0.001), correction_schedule=sched)
    kw = dict(seed=1, noise_sigma0=0.0015, blur_sigma_max=1.2, anchor_interval=3)
    got = S.make_sequence(S.reference_demo_scene(), spec, intr, **kw)
    ref = RS.make_sequence(RS.demo_scene(), rspec, _rintr(intr), **kw)
    assert got.n_frames == ref.n_frames == 10
    for a, b in zip(got.frames, ref.frames):
        assert a.index == b.index
        assert np.array_equal(a.depth, b.depth), a.index
        assert np.array_equal(a.color, b.color), a.index
    for i in ref.gt_poses:
        assert _same_pose(got.gt_poses[i], ref.gt_poses[i])
        assert _same_pose(got.drifted_poses[i], ref.drifted_poses[i])
    assert len(got.events) == len(ref.events)
    for a, b in zip(got.events, ref.events):
        assert a.at_frame == b.at_frame and a.dvo_kf_flags == b.dvo_kf_flags
        assert sorted(a.anchor_poses) == sorted(b.anchor_poses)
        assert all(_same_pose(a.anchor_poses[k], b.anchor_poses[k]) for k in a.anchor_poses)
