"""Keyframe fusion on the device vs the reference's keyframe_fusion
(oracle/_ref, run on this host so both sides share the host BLAS)."""

import numpy as np
import pytest

from refimport import reference

pytestmark = pytest.mark.gpu

REF = reference()
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def KF():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import keyframe_fusion

    return keyframe_fusion


def scene_depth(h, w, fx, cx, cy, rng, jumps=True, noise=0.002):
    """A tilted plane + a sphere bump + holes: normals, grazing angles and
    depth discontinuities all occur."""
    u = np.arange(w, dtype=np.float64)[None, :]
    v = np.arange(h, dtype=np.float64)[:, None]
    xn, yn = (u - cx) / fx, (v - cy) / fx
    depth = 1.6 / (1.0 - 0.3 * xn + 0.2 * yn)
    r2 = (u - 0.6 * w) ** 2 + (v - 0.4 * h) ** 2
    bump = r2 < (0.15 * w) ** 2
    depth = np.where(bump, depth - 0.35 + 1e-6 * r2, depth)
    if jumps:
        depth[:, int(0.8 * w):] += 0.5
    depth = depth + rng.normal(0.0, noise, depth.shape) * depth * depth
    depth[rng.random(depth.shape) < 0.02] = 0.0
    return depth


def color_img(h, w, rng):
    u = np.arange(w, dtype=np.float64)[None, :]
    v = np.arange(h, dtype=np.float64)[:, None]
    c = np.empty((h, w, 3))
    c[..., 0] = 128 + 100 * np.sin(u / 7.0)
    c[..., 1] = (u * 3 + v * 2) % 255
    c[..., 2] = 40 + 0.5 * v
    return np.clip(c + rng.normal(0, 3, c.shape), 0, 255)


def ref_pair(KF, h, w):
    from paper_1709_03763_b200.geometry import Intrinsics

    f = 0.82 * w
    mine = Intrinsics(f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h)
    ref = REF["G"].Intrinsics(f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h)
    return mine, ref


@needs_ref
@pytest.mark.parametrize("hw", [(48, 64), (480, 640)])
def test_depth_weight_map_bitexact(KF, hw):
    h, w = hw
    rng = np.random.default_rng(h)
    intr, rintr = ref_pair(KF, h, w)
    depth = scene_depth(h, w, intr.fx, intr.cx, intr.cy, rng)
    depth[3, 5] = np.nan
    depth[7, 9] = np.inf
    want = REF["KF"].depth_sample_weight(depth, rintr)
    want[REF["KF"].discontinuity_mask(depth, 0.1)] = 0.0
    got = KF.depth_weight_map(depth, intr, 0.1).cpu().numpy()
    assert np.array_equal(got, want)
    mask = KF.discontinuity_mask(depth, 0.1).cpu().numpy()
    assert np.array_equal(mask, REF["KF"].discontinuity_mask(depth, 0.1))


def _poses(G, n, step=0.01):
    out = []
    for i in range(n):
        R = G.rotation_z(0.004 * i) @ G.rotation_y(-0.003 * i)
        out.append(G.Pose(R, np.array([step * i, -0.5 * step * i, 0.3 * step * i])))
    return out


@needs_ref
@pytest.mark.parametrize("hw,n", [((48, 64), 3), ((120, 160), 5), ((480, 640), 5)])
def test_fuse_depth_and_color_bitexact(KF, hw, n):
    from paper_1709_03763_b200 import geometry as MG

    h, w = hw
    rng = np.random.default_rng(w + n)
    intr, rintr = ref_pair(KF, h, w)
    RG, RK = REF["G"], REF["KF"]
    rposes = _poses(RG, n)
    mposes = [MG.Pose(p.rotation, p.translation) for p in rposes]
    frames = []
    for i in range(n):
        d = scene_depth(h, w, intr.fx, intr.cx, intr.cy, rng)
        frames.append((d, color_img(h, w, rng)))
    rkf = mkf = None
    for i, (d, c) in enumerate(frames):
        rf = RK.FrameObservation(i + 1, c, d, rposes[i])
        mf = KF.FrameObservation(i + 1, c, d, mposes[i])
        if rkf is None:
            rkf = RK.new_keyframe(rf, rintr)
            mkf = KF.new_keyframe(mf, intr)
        RK.fuse_depth(rkf, rf)
        KF.fuse_depth(mkf, mf)
    assert np.array_equal(mkf.depth.cpu().numpy(), rkf.depth)
    assert np.array_equal(mkf.weight.cpu().numpy(), rkf.weight)
    assert mkf.members == rkf.members
    for mo, ro in zip(mkf.observations, rkf.observations):
        assert float(mo.blur_weight.item()) == ro.blur_weight
        assert np.array_equal(mo.color.cpu().numpy(), ro.color)
    RK.fuse_color(rkf)
    KF.fuse_color(mkf)
    assert np.array_equal(mkf.color_valid.cpu().numpy(), rkf.color_valid)
    assert np.array_equal(mkf.color.cpu().numpy(), rkf.color)
    assert mkf.finalized
    with pytest.raises(ValueError):
        KF.fuse_color(mkf)


@needs_ref
def test_unsharp_blurriness_helpers(KF):
    rng = np.random.default_rng(5)
    img = rng.uniform(0, 255, (37, 53, 3))
    assert np.array_equal(KF.unsharp_mask(img).cpu().numpy(), REF["KF"].unsharp_mask(img))
    g2 = rng.uniform(0, 255, (40, 31))
    assert np.array_equal(KF.unsharp_mask(g2, gain=1.0).cpu().numpy(),
                          REF["KF"].unsharp_mask(g2, gain=1.0))
    assert np.array_equal(KF.unsharp_mask(img, gain=0.0).cpu().numpy(), img)
    gray = REF["KF"].grayscale(img)
    assert np.array_equal(KF.grayscale(img).cpu().numpy(), gray)
    assert KF.blurriness(gray) == REF["KF"].blurriness(gray)
    assert KF.blurriness(np.full((32, 32), 77.0)) == 1.0
    tile = np.indices((64, 64)).sum(axis=0) // 8 % 2 * 255.0
    assert KF.blurriness(tile) == REF["KF"].blurriness(tile)


def test_fusion_reference_test_cases(KF):
    """Reference tests/test_keyframe_fusion.py:135-163, 274-320 on the device."""
    from paper_1709_03763_b200.geometry import Intrinsics, Pose

    intr = Intrinsics(50.0, 50.0, 31.5, 23.5, 64, 48)

    def wall(i, z, color=None):
        return KF.FrameObservation(i, color, np.full((48, 64), float(z)), Pose.identity())

    kf = KF.new_keyframe(wall(1, 2.0), intr)
    KF.fuse_depth(kf, wall(1, 2.0))
    d, wt = kf.depth.cpu().numpy(), kf.weight.cpu().numpy()
    valid = wt > 0
    assert np.allclose(d[valid], 2.0, atol=1e-9) and not valid[0].any() and valid[10, 10]
    w1 = wt.copy()
    KF.fuse_depth(kf, wall(2, 2.0))
    assert np.array_equal(kf.weight.cpu().numpy(), 2.0 * w1)
    kf = None
    for i, level in enumerate((10.0, 200.0, 12.0)):
        f = wall(i + 1, 2.0, np.full((48, 64, 3), level))
        kf = kf or KF.new_keyframe(f, intr)
        KF.fuse_depth(kf, f)
    KF.fuse_color(kf)
    cv = kf.color_valid.cpu().numpy()
    assert cv.any() and np.allclose(kf.color.cpu().numpy()[cv], 12.0, atol=1e-9)
    assert KF.weighted_median([9, 5], [1, 1]) == 5
    assert KF.weighted_median([10, 200], [3, 1]) == 10


@needs_ref
def test_normal_map_and_weight_with_normals_bitexact(KF):
    """normal_map (keyframe_fusion.py:142-188) and depth_sample_weight with
    caller-supplied normals (:191-208) on the device."""
    h, w = 120, 160
    rng = np.random.default_rng(21)
    intr, rintr = ref_pair(KF, h, w)
    depth = scene_depth(h, w, intr.fx, intr.cx, intr.cy, rng)
    depth[5, 7] = np.nan
    n_ref = REF["KF"].normal_map(depth, rintr)
    n_got = KF.normal_map(depth, intr).cpu().numpy()
    assert np.array_equal(n_got, n_ref)
    normals = rng.normal(size=(h, w, 3))
    want = REF["KF"].depth_sample_weight(depth, rintr, normals)
    got = KF.depth_sample_weight(depth, intr, normals).cpu().numpy()
    assert np.array_equal(got, want)
    assert np.array_equal(KF.depth_sample_weight(depth, intr).cpu().numpy(),
                          REF["KF"].depth_sample_weight(depth, rintr))


@needs_ref
def test_fuse_color_more_than_64_members_bitexact(KF):
    """A keyframe that stays open for 70 frames (the reference has
    no member limit): the global-scratch median path."""
    from paper_1709_03763_b200 import geometry as MG

    h, w, n = 48, 64, 70
    rng = np.random.default_rng(70)
    intr, rintr = ref_pair(KF, h, w)
    RG, RK = REF["G"], REF["KF"]
    rposes = _poses(RG, n, step=0.002)
    mposes = [MG.Pose(p.rotation, p.translation) for p in rposes]
    rkf = mkf = None
    for i in range(n):
        d = scene_depth(h, w, intr.fx, intr.cx, intr.cy, rng)
        c = color_img(h, w, rng)
        if i % 9 == 4:
            c = np.full_like(c, 100.0)  # ties between members
        rf = RK.FrameObservation(i + 1, c, d, rposes[i])
        mf = KF.FrameObservation(i + 1, c, d, mposes[i])
        if rkf is None:
            rkf = RK.new_keyframe(rf, rintr)
            mkf = KF.new_keyframe(mf, intr)
        RK.fuse_depth(rkf, rf)
        KF.fuse_depth(mkf, mf)
    RK.fuse_color(rkf)
    KF.fuse_color(mkf)
    assert np.array_equal(mkf.color_valid.cpu().numpy(), rkf.color_valid)
    assert np.array_equal(mkf.color.cpu().numpy(), rkf.color)


def test_rf_fuse_depth_entry_point_matches_fuse_depth(KF):
    """The C ABI's standalone rf_fuse_depth (caller-supplied weight map; cub
    scan + ordered scatter + Eq. 1 merge) gives the keyframe planes the
    one-call-per-frame path (rf_fuse_frame, behind fuse_depth) gives."""
    import torch

    from paper_1709_03763_b200 import _lib as L
    from paper_1709_03763_b200 import geometry as MG
    from paper_1709_03763_b200.volume import pose_struct

    h, w = 120, 160
    rng = np.random.default_rng(77)
    intr = MG.Intrinsics(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=w, height=h)
    poses = [MG.Pose(MG.rotation_z(0.004 * i) @ MG.rotation_y(-0.003 * i),
                     np.array([0.01 * i, -0.005 * i, 0.003 * i])) for i in range(4)]
    frames = [scene_depth(h, w, intr.fx, intr.cx, intr.cy, rng) for _ in range(4)]
    kf = None
    for i, d in enumerate(frames):
        fo = KF.FrameObservation(i + 1, None, d, poses[i])
        if kf is None:
            kf = KF.new_keyframe(fo, intr)
        KF.fuse_depth(kf, fo)
    kd = torch.zeros((h, w), dtype=torch.float64, device="cuda:0")
    kw = torch.zeros_like(kd)
    for i, d in enumerate(frames):
        dt = torch.from_numpy(d).cuda()
        wm = KF.depth_weight_map(dt, intr)  # fuse_depth's map (:245-246)
        rel = pose_struct(MG.compose(MG.inverse(poses[0]), poses[i]))
        st = L.lib().rf_fuse_depth(kd.data_ptr(), kw.data_ptr(), dt.data_ptr(),
                                   wm.contiguous().data_ptr(), w, h, intr.fx, intr.fy, intr.cx,
                                   intr.cy, L.ctypes.byref(rel), KF.detect_blas_order(),
                                   torch.cuda.current_stream().cuda_stream)
        assert st == L.RF_OK
    torch.cuda.synchronize()
    assert np.array_equal(kd.cpu().numpy(), kf.depth.cpu().numpy())
    assert np.array_equal(kw.cpu().numpy(), kf.weight.cpu().numpy())
