"""Synthetic RGB-D workloads for measurement (not on the timed hot path).

Device counterpart of /root/reference/pkg/src/refusion/synth.py: analytic
scenes (:46-129), look-at trajectories (:136-213), sphere-traced depth +
Lambert colour + sigma0*z^2 noise (:220-283, rendered by rf_synth_render on
the GPU), plus the drift / anchor-correction events of make_sequence
(:310-390).  Used by bench.py and the large-scale tests to build configs
2-5 of BASELINE.json, which the 2.46 s/frame CPU renderer cannot produce.
"""

import ctypes
from dataclasses import dataclass

import itertools

import numpy as np

from . import _lib as L
from .geometry import Intrinsics, Pose, compose

SPHERE, BOX, ROOM = 0, 1, 2
DEFAULT_INTRINSICS = Intrinsics(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480)
LIGHT_DIR = np.array([0.35, -0.25, -0.9]) / np.linalg.norm([0.35, -0.25, -0.9])


@dataclass(frozen=True)
class Prim:
    kind: int
    center: tuple
    size: tuple
    albedo: tuple


def demo_scene():
    """synth.py:118-129 -- desk-scale room (config 1)."""
    return [
        Prim(ROOM, (0.0, 0.0, 1.5), (2.6, 2.2, 1.5), (205.0, 195.0, 180.0)),
        Prim(SPHERE, (1.1, 0.6, 0.5), (0.5, 0, 0), (60.0, 110.0, 200.0)),
        Prim(SPHERE, (-1.0, -0.8, 0.35), (0.35, 0, 0), (200.0, 80.0, 70.0)),
        Prim(BOX, (-0.2, 1.3, 0.4), (0.5, 0.35, 0.4), (90.0, 170.0, 90.0)),
    ]


def corridor_scene(seed=2, n_clutter=24):
    """Config 2: a 40 m x 2.4 m x 3 m corridor with seeded boxes / spheres
    along the walls."""
    rng = np.random.default_rng(seed)
    prims = [Prim(ROOM, (20.0, 0.0, 1.5), (20.0, 1.2, 1.5), (200.0, 190.0, 175.0))]
    for i in range(n_clutter):
        x = 1.5 + 37.0 * (i + rng.uniform(0.1, 0.9)) / n_clutter
        side = 1.0 if i % 2 == 0 else -1.0
        alb = tuple(float(a) for a in rng.uniform(40.0, 230.0, 3))
        if rng.random() < 0.5:
            hx, hy, hz = rng.uniform(0.15, 0.45), rng.uniform(0.1, 0.3), rng.uniform(0.2, 0.6)
            prims.append(Prim(BOX, (x, side * (1.2 - hy), hz), (hx, hy, hz), alb))
        else:
            r = rng.uniform(0.12, 0.3)
            prims.append(Prim(SPHERE, (x, side * (1.2 - r), rng.uniform(r, 2.4)), (r, 0, 0), alb))
    return prims


def look_at_pose(eye, target, up=(0.0, 0.0, 1.0)):
    """synth.py:136-151 -- optical axis toward target, image y down."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    z = fwd / np.linalg.norm(fwd)
    x = np.cross(z, np.asarray(up, dtype=np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return Pose(np.stack([x, y, z], axis=1), eye)


def corridor_trajectory(n_frames, length=38.0):
    """Straight dolly down the corridor with a small yaw / lateral oscillation."""
    poses = []
    for i in range(n_frames):
        s = i / max(n_frames - 1, 1)
        x = 1.0 + length * s
        y = 0.35 * np.sin(2.0 * np.pi * i / 400.0)
        yaw = 0.35 * np.sin(2.0 * np.pi * i / 250.0)
        eye = (x, y, 1.5)
        target = (x + np.cos(yaw), y + np.sin(yaw), 1.45)
        poses.append(look_at_pose(eye, target))
    return poses


def orbit_trajectory(n_waypoints=9, radius=1.2, height=1.3, frames_per_segment=11):
    """synth.py:154-171 + pose_at: orbit looking outward (config 1)."""
    way = []
    for i in range(n_waypoints + 1):
        ang = 2.0 * np.pi * (i % n_waypoints) / n_waypoints
        eye = np.array([radius * np.cos(ang), radius * np.sin(ang), height])
        tgt = np.array([2 * radius * np.cos(ang), 2 * radius * np.sin(ang), height])
        way.append(look_at_pose(eye, tgt))
    n = n_waypoints * frames_per_segment + 1
    out = []
    for idx in range(1, n + 1):
        g = (idx - 1) / frames_per_segment
        seg = min(int(np.floor(g)), n_waypoints - 1)
        out.append(pose_interpolate(way[seg], way[seg + 1], g - seg))
    return out


def axis_angle_rotation(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    n = np.linalg.norm(axis)
    if n == 0 or angle == 0:
        return np.eye(3)
    x, y, z = axis / n
    K = np.array([[0, -z, y], [z, 0, -x], [-y, x, 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


def pose_interpolate(T, U, t):
    """Geodesic interpolation T (t=0) -> U (t=1)."""
    rel = T.rotation.T @ U.rotation
    cos_a = min(1.0, max(-1.0, (np.trace(rel) - 1.0) / 2.0))
    angle = float(np.arccos(cos_a))
    if angle < 1e-12:
        R = T.rotation
    else:
        v = np.array([rel[2, 1] - rel[1, 2], rel[0, 2] - rel[2, 0], rel[1, 0] - rel[0, 1]])
        if np.linalg.norm(v) < 1e-12:
            R = T.rotation
        else:
            R = T.rotation @ axis_angle_rotation(v, angle * t)
    return Pose(R, (1.0 - t) * T.translation + t * U.translation)


def drift_poses(gt_poses, drift_t, drift_r, seed=1):
    """make_sequence's accumulating drift (synth.py:321-346): reported pose
    k = step^k composed onto ground truth."""
    rng = np.random.default_rng(seed)
    t_dir = rng.standard_normal(3)
    t_dir /= np.linalg.norm(t_dir)
    r_axis = rng.standard_normal(3)
    r_axis /= np.linalg.norm(r_axis)
    step = Pose(axis_angle_rotation(r_axis, drift_r), drift_t * t_dir)
    drift = Pose.identity()
    out = []
    for k, gt in enumerate(gt_poses):
        if k > 0:
            drift = compose(step, drift)
        out.append(compose(drift, gt))
    return out


# ---------------------------------------------------------------------------
# GPU rendering


class Renderer:
    """Renders frames of one analytic scene on a CUDA device."""

    def __init__(self, prims, intr=DEFAULT_INTRINSICS, device=0, z_max=5.0,
                 sigma0=0.0015, steps=256, tol=1e-5):
        import torch

        if len(prims) > 32:
            raise ValueError("at most 32 primitives per scene")
        self.torch = torch
        self.intr = intr
        self.device = device
        arr = (L.RfSynthPrim * len(prims))()
        for i, p in enumerate(prims):
            arr[i].kind = p.kind
            for j in range(3):
                arr[i].center[j] = float(p.center[j])
                arr[i].size[j] = float(p.size[j])
                arr[i].albedo[j] = float(p.albedo[j])
        raw = bytes(arr)
        self.n = len(prims)
        self.prims = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(f"cuda:{device}")
        self.params = L.RfSynthParams()
        self.params.z_max = z_max
        self.params.tol = tol
        self.params.sigma0 = sigma0
        self.params.ambient = 0.3
        self.params.diffuse = 0.7
        for j in range(3):
            self.params.light[j] = float(LIGHT_DIR[j])
        self.params.steps = steps

    def render(self, pose, seed=0, color=True):
        torch = self.torch
        from .volume import pose_struct

        h, w = self.intr.height, self.intr.width
        dev = f"cuda:{self.device}"
        depth = torch.empty((h, w), dtype=torch.float64, device=dev)
        col = torch.empty((h, w, 3), dtype=torch.float64, device=dev) if color else None
        self.params.seed = int(seed) & ((1 << 64) - 1)
        ps = pose_struct(pose)
        with torch.cuda.device(self.device):
            st = L.lib().rf_synth_render(
                self.prims.data_ptr(), self.n, ctypes.byref(ps), float(self.intr.fx),
                float(self.intr.fy), float(self.intr.cx), float(self.intr.cy), w, h,
                ctypes.byref(self.params), depth.data_ptr(),
                col.data_ptr() if col is not None else None,
                torch.cuda.current_stream().cuda_stream)
        if st != L.RF_OK:
            raise RuntimeError("rf_synth_render failed")
        return depth, col


_MEMO_TAGS = itertools.count(1)


class DeviceKeyframe:
    """A keyframe whose planes live in HBM (duck-typed like Keyframe).

    ``memo_tag`` identifies the keyframe to the volume's footprint memo
    (rf_kf_view.memo_tag): its host copy (to_host) keeps the tag, so a
    de-integration from host planes reuses the footprint its resident twin
    integrated (the memo still checks the planes' content hash)."""

    def __init__(self, intrinsics, pose, depth, weight, color, kf_id=-1, memo_tag=None):
        self.intrinsics = intrinsics
        self.pose = pose
        self.depth = depth
        self.weight = weight
        self.color = color
        self.kf_id = kf_id
        self.memo_tag = next(_MEMO_TAGS) if memo_tag is None else memo_tag

    def to_host(self, pinned=False):
        """Host copy with the same attributes (numpy, or pinned torch tensors)."""
        if pinned:
            planes = [None if t is None else t.cpu().pin_memory()
                      for t in (self.depth, self.weight, self.color)]
        else:
            planes = [None if t is None else t.cpu().numpy()
                      for t in (self.depth, self.weight, self.color)]
        return DeviceKeyframe(self.intrinsics, self.pose, *planes, kf_id=self.kf_id,
                              memo_tag=self.memo_tag)


def render_keyframe(renderer, pose, seed, kappa=5):
    """A keyframe standing in for kappa fused frames: rendered depth / colour,
    weight = kappa / z^2 (the frontal w_z of keyframe_fusion.py:191-208
    summed over the members)."""
    torch = renderer.torch
    depth, color = renderer.render(pose, seed=seed)
    valid = depth > 0
    weight = torch.where(valid, kappa / torch.clamp(depth * depth, min=1e-12),
                         torch.zeros_like(depth))
    return DeviceKeyframe(renderer.intr, pose, depth, weight, color)


def fused_keyframe(renderer, gt_frames, est_frames, seeds, first_index=1):
    """A keyframe fused from a burst of rendered frames, the way
    pipeline.run_pipeline builds one (/root/reference/pkg/src/refusion/
    pipeline.py:204-271): frame j is rendered at its ground-truth pose
    ``gt_frames[j]`` (noise seed ``seeds[j]``) and fused at its estimated
    pose ``est_frames[j]`` (keyframe_fusion.new_keyframe / fuse_depth), then
    the colour is finalised (fuse_color).  Returns a DeviceKeyframe at
    ``est_frames[0]`` holding the fused depth / weight / colour planes."""
    from . import keyframe_fusion as KF

    kf = None
    for j, (g, e, s) in enumerate(zip(gt_frames, est_frames, seeds)):
        depth, color = renderer.render(g, seed=s)
        obs = KF.FrameObservation(index=first_index + j, color=color, depth=depth, pose=e)
        if kf is None:
            kf = KF.new_keyframe(obs, renderer.intr)
        KF.fuse_depth(kf, obs)
    KF.fuse_color(kf)
    return DeviceKeyframe(renderer.intr, kf.pose, kf.depth, kf.weight, kf.color)


def burst_poses(gt_frames, kf_first, drifted_kf, kappa):
    """Estimated poses of the frames of keyframe k: the keyframe's drift
    (drifted_kf[k] vs gt_frames[k * kappa]) applied rigidly to its burst,
    so relative poses inside a burst are exact."""
    from .geometry import inverse

    k0 = kf_first * kappa
    corr = compose(drifted_kf, inverse(gt_frames[k0]))
    return [drifted_kf.copy()] + [compose(corr, gt_frames[k0 + j]) for j in range(1, kappa)]
