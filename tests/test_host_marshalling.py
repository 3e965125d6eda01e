"""Host-side marshalling of the C ABI (no GPU needed): keyframe views built
from host planes carry host pointers for the library to stage, and poses
are packed row-major with the translation last."""

import numpy as np

from paper_1709_03763_b200 import volume as V
from paper_1709_03763_b200.geometry import Pose

import scenarios as S


def test_host_planes_are_passed_for_staging():
    rng = np.random.default_rng(3)
    f = S.random_frame(rng)
    view, keep = V.kf_view(f, device=0)
    assert view.planes_on_host == 1
    assert view.depth == keep[0].ctypes.data and view.weight == keep[1].ctypes.data
    assert view.color == keep[2].ctypes.data
    assert (view.width, view.height) == (f.intrinsics.width, f.intrinsics.height)
    assert not view.ready_event and view.memo_tag == 0  # the library derives the tag


def test_host_planes_are_converted_to_contiguous_f64():
    rng = np.random.default_rng(4)
    f = S.random_frame(rng)
    f.depth = np.asfortranarray(f.depth.astype(np.float32))
    view, keep = V.kf_view(f, device=0)
    assert keep[0].dtype == np.float64 and keep[0].flags.c_contiguous
    assert np.array_equal(keep[0], f.depth.astype(np.float64))


def test_pose_struct_layout():
    rng = np.random.default_rng(5)
    R = S.rot_z(rng.uniform(-3, 3)) @ S.rot_y(rng.uniform(-1, 1))
    t = rng.uniform(-5, 5, 3)
    p = V.pose_struct(Pose(R, t))
    assert list(p.R) == R.reshape(9).tolist() and list(p.t) == t.tolist()


def test_pose_copy_is_independent():
    p = Pose(S.rot_x(0.3), np.array([1.0, 2.0, 3.0]))
    q = p.copy()
    q.translation[0] = 9.0
    assert p.translation[0] == 1.0 and np.array_equal(q.rotation, p.rotation)


def test_views_are_memoised_per_keyframe_planes():
    """A correction re-marshals the same keyframes: the view of a keyframe is
    reused while its planes are the same objects (in-place edits keep the
    pointers), rebuilt when a plane is replaced, and never memoised when the
    planes had to be converted (a copy would go stale)."""
    rng = np.random.default_rng(5)
    f = S.random_frame(rng)
    v1, _ = V.kf_view(f, device=0)
    v2, _ = V.kf_view(f, device=0)
    assert v1 is v2
    f.depth = f.depth.copy()
    v3, _ = V.kf_view(f, device=0)
    assert v3 is not v1 and v3.depth == f.depth.ctypes.data
    g = S.random_frame(rng)
    g.depth = g.depth.astype(np.float32)
    w1, _ = V.kf_view(g, device=0)
    w2, _ = V.kf_view(g, device=0)
    assert w1 is not w2  # converted plane: a fresh copy every call


def test_memo_tag_travels_to_the_view():
    rng = np.random.default_rng(6)
    f = S.random_frame(rng)
    f.memo_tag = 12345
    view, _ = V.kf_view(f, device=0)
    assert view.memo_tag == 12345


def test_views_are_memoised_for_unhashable_keyframes():
    """keyframe_fusion.Keyframe is a plain (unhashable) dataclass: its views
    are memoised too, and dropped when the keyframe dies."""
    import gc

    from paper_1709_03763_b200.keyframe_fusion import Keyframe

    rng = np.random.default_rng(7)
    f = S.random_frame(rng)
    kf = Keyframe(intrinsics=f.intrinsics, pose=Pose.identity(), anchor_id=0,
                  rel_pose=Pose.identity(), depth=f.depth, weight=f.weight, color=f.color)
    v1, _ = V.kf_view(kf, device=0)
    v2, _ = V.kf_view(kf, device=0)
    assert v1 is v2
    key = id(kf)
    assert key in V._VIEWS
    del kf, v1, v2
    gc.collect()
    assert key not in V._VIEWS


def test_correction_batches_split_at_window_boundaries():
    """More entries than one native call holds are split into chunks of whole
    windows (finalize over > 4096 moved keyframes)."""
    calls = []

    class _Store:
        _router = None

    def fake(store, windows, cfg, next_center=None):
        calls.append(([len(w) for w in windows], next_center))
        return sum(len(w) for w in windows)

    orig = V._correct_windows
    V._correct_windows = fake
    try:
        windows = [[object()] * 10 for _ in range(1000)]
        n = V.correct_windows(_Store(), windows, None, next_center="c")
    finally:
        V._correct_windows = orig
    assert n == 10_000
    assert all(sum(sizes) <= V.MAX_CALL_ENTRIES for sizes, _ in calls)
    assert [c for _, c in calls] == [None] * (len(calls) - 1) + ["c"]
    assert sum(len(s) for s, _ in calls) == 1000
