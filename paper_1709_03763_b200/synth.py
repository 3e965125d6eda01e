"""Synthetic RGB-D workloads (not on the timed hot path).

Device port of /root/reference/pkg/src/refusion/synth.py: analytic scenes
(:46-129), look-at trajectories (:136-213), sphere-traced depth + Lambert
colour (:220-267, rf_synth_depth / rf_synth_color on the GPU, bit-identical
to the reference), sigma0*z^2 noise (:270-283, numpy's generator on the
host) and make_sequence's drift / anchor-correction events (:310-390).
bench.py and the large-scale tests build configs 2-5 of BASELINE.json with
it; the reference's 2.46 s/frame CPU renderer cannot produce them.
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
    """Renders frames of one analytic scene on a CUDA device, bit-identical
    to the reference generator (render_depth -> add_noise -> render_color,
    synth.py:220-283 and :348-352): sphere tracing and shading run on the
    device (rf_synth_depth / rf_synth_color), the sigma0 * z^2 noise is
    numpy's default_rng(seed) stream drawn on the host."""

    def __init__(self, prims, intr=DEFAULT_INTRINSICS, device=0, z_max=5.0,
                 sigma0=0.0015, steps=256, tol=1e-5):
        self.scene = prims if isinstance(prims, AnalyticScene) else AnalyticScene(list(prims))
        self.intr = intr
        self.device = device
        self.z_max = z_max
        self.sigma0 = sigma0
        self.steps = steps
        self.tol = tol

    def render(self, pose, seed=0, color=True):
        """(depth, colour) CUDA tensors of the frame at ``pose``; ``seed`` is
        the numpy seed of its noise (the reference's make_sequence uses
        (seed, 7, index))."""
        import torch

        with torch.cuda.device(self.device):
            depth = render_depth(self.scene, pose, self.intr, z_max=self.z_max, steps=self.steps,
                                 tol=self.tol, as_tensor=True)
            if self.sigma0 > 0.0:
                noisy = add_noise(depth.cpu().numpy(), seed=seed, sigma0=self.sigma0)
                depth = torch.from_numpy(noisy).to(depth.device)
            col = render_color(self.scene, pose, self.intr, depth, as_tensor=True) if color \
                else None
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


# ---------------------------------------------------------------------------
# Faithful port of the reference generator: the same scenes,
# trajectories, events and pixels as /root/reference/pkg/src/refusion/
# synth.py, bit for bit.  Depth (sphere tracing) and colour (Lambert shading
# of the noisy depth) render on the device (rf_synth_depth / rf_synth_color,
# numpy's evaluation order, the host BLAS's multiply-add order calibrated
# below); the depth noise is numpy's PCG64 + ziggurat stream, drawn on the
# host by the same call the reference makes (add_noise); the optional
# colour blur is scipy's gaussian_filter(mode 'reflect') on the device.

Z_MAX_DEFAULT = 10.0
SPHERE_TRACE_STEPS = 256
SPHERE_TRACE_TOL = 1e-5
SIGMA0_DEFAULT = 0.0015
DEFAULT_ANCHOR_INTERVAL = 10
AMBIENT = 0.3
DIFFUSE = 0.7
_NORMAL_EPS = 1e-4


@dataclass(frozen=True)
class Sphere:
    """synth.py:46-53"""
    center: tuple
    radius: float
    albedo: tuple

    def prim(self):
        return Prim(SPHERE, tuple(self.center), (float(self.radius), 0.0, 0.0), tuple(self.albedo))


@dataclass(frozen=True)
class BoxSolid:
    """synth.py:56-66"""
    center: tuple
    half_extents: tuple
    albedo: tuple

    def prim(self):
        return Prim(BOX, tuple(self.center), tuple(self.half_extents), tuple(self.albedo))


@dataclass(frozen=True)
class RoomShell:
    """synth.py:69-81: a hollow box enclosing the scene."""
    center: tuple
    half_extents: tuple
    albedo: tuple

    def prim(self):
        return Prim(ROOM, tuple(self.center), tuple(self.half_extents), tuple(self.albedo))


class AnalyticScene:
    """Union of primitives (synth.py:84-112); the fields evaluate on the
    device.  ``sdf`` of a few host points (make_sequence's free-space check
    of the camera centre) uses numpy, in the reference's expressions."""

    def __init__(self, primitives):
        if not primitives:
            raise ValueError("scene needs at least one primitive")
        if len(primitives) > 32:
            raise ValueError("at most 32 primitives per scene")
        self.primitives = list(primitives)
        self._dev = {}

    def prims(self):
        return [p.prim() if hasattr(p, "prim") else p for p in self.primitives]

    def sdf(self, points):
        points = np.asarray(points, dtype=np.float64)
        out = []
        for p in self.prims():
            c = np.asarray(p.center)
            if p.kind == SPHERE:
                out.append(np.linalg.norm(points - c, axis=-1) - p.size[0])
                continue
            q = np.abs(points - c) - np.asarray(p.size)
            s = np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)
            out.append(-s if p.kind == ROOM else s)
        return np.stack(out).min(axis=0)

    def device_prims(self, device):
        import torch

        if device not in self._dev:
            prims = self.prims()
            arr = (L.RfSynthPrim * len(prims))()
            for i, p in enumerate(prims):
                arr[i].kind = p.kind
                for j in range(3):
                    arr[i].center[j] = float(p.center[j])
                    arr[i].size[j] = float(p.size[j])
                    arr[i].albedo[j] = float(p.albedo[j])
            self._dev[device] = (torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
                                 .to(f"cuda:{device}"), len(prims))
        return self._dev[device]


def reference_demo_scene():
    """synth.py:115-129 as an AnalyticScene."""
    return AnalyticScene([
        RoomShell(center=(0.0, 0.0, 1.5), half_extents=(2.6, 2.2, 1.5),
                  albedo=(205.0, 195.0, 180.0)),
        Sphere(center=(1.1, 0.6, 0.5), radius=0.5, albedo=(60.0, 110.0, 200.0)),
        Sphere(center=(-1.0, -0.8, 0.35), radius=0.35, albedo=(200.0, 80.0, 70.0)),
        BoxSolid(center=(-0.2, 1.3, 0.4), half_extents=(0.5, 0.35, 0.4),
                 albedo=(90.0, 170.0, 90.0)),
    ])


def _as_scene(scene):
    if isinstance(scene, AnalyticScene):
        return scene
    return AnalyticScene(list(scene))


_RENDER_ORDERS = None


def detect_render_orders(samples=96, seed=4242):
    """(gemm, gemv) multiply-add orders of the host BLAS for the renderer's
    two products, d_cam @ R.T ((h, w, 3) @ (3, 3)) and normal @ (-light)
    ((n, 3) @ (3,)) -- rf_blas_order codes, calibrated once per process like
    keyframe_fusion.detect_blas_order (BLAS kernels differ between hosts)."""
    global _RENDER_ORDERS
    if _RENDER_ORDERS is not None:
        return _RENDER_ORDERS
    from fractions import Fraction

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    cands = {
        1: lambda q, r: fma(q[2], r[2], fma(q[1], r[1], q[0] * r[0])),
        0: lambda q, r: (q[0] * r[0] + q[1] * r[1]) + q[2] * r[2],
        2: lambda q, r: fma(q[0], r[0], fma(q[1], r[1], q[2] * r[2])),
        3: lambda q, r: fma(q[2], r[2], fma(q[0], r[0], q[1] * r[1])),
    }
    rng = np.random.default_rng(seed)
    R = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    p = rng.normal(size=(48, 64, 3))
    got = (p @ R.T).reshape(-1, 3)
    pf = p.reshape(-1, 3)
    idx = rng.choice(len(pf), samples, replace=False)
    gemm = next((c for c, f in cands.items()
                 if all(f(pf[i], R[k]) == got[i, k] for i in idx for k in range(3))), 1)
    v = -(np.array([0.35, -0.25, -0.9]) / np.linalg.norm([0.35, -0.25, -0.9]))
    q = rng.normal(size=(4096, 3))
    gq = q @ v
    idx = rng.choice(len(q), samples, replace=False)
    gemv = next((c for c, f in cands.items() if all(f(q[i], v) == gq[i] for i in idx)), 3)
    _RENDER_ORDERS = (gemm, gemv)
    return _RENDER_ORDERS


def _ref_params(z_max, steps, tol, light_dir):
    gemm, gemv = detect_render_orders()
    sp = L.RfSynthRefParams()
    sp.z_max = float(z_max)
    sp.tol = float(tol)
    sp.ambient = AMBIENT
    sp.diffuse = DIFFUSE
    neg = -np.asarray(light_dir, dtype=np.float64)
    for j in range(3):
        sp.neg_light[j] = float(neg[j])
    sp.normal_eps = _NORMAL_EPS
    sp.steps = int(steps)
    sp.gemm_order = gemm
    sp.gemv_order = gemv
    return sp


def _device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the renderer needs a CUDA device (there is no CPU fallback)")
    return torch.cuda.current_device()


def render_depth(scene, pose, intr, z_max=Z_MAX_DEFAULT, steps=SPHERE_TRACE_STEPS,
                 tol=SPHERE_TRACE_TOL, as_tensor=False):
    """synth.py:220-250 on the device: sphere-traced z-depth, misses and
    beyond-range hits 0.  Returns a numpy (h, w) array (a CUDA tensor with
    ``as_tensor``), bit-identical to the reference's."""
    import torch

    from .volume import pose_struct

    scene = _as_scene(scene)
    dev = _device()
    prims, n = scene.device_prims(dev)
    depth = torch.empty((intr.height, intr.width), dtype=torch.float64, device=f"cuda:{dev}")
    sp = _ref_params(z_max, steps, tol, LIGHT_DIR)
    ps = pose_struct(pose)
    st = L.lib().rf_synth_depth(prims.data_ptr(), n, ctypes.byref(ps), float(intr.fx),
                                float(intr.fy), float(intr.cx), float(intr.cy), intr.width,
                                intr.height, ctypes.byref(sp), depth.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
    if st != L.RF_OK:
        raise RuntimeError("rf_synth_depth failed")
    return depth if as_tensor else depth.cpu().numpy()


def render_color(scene, pose, intr, depth, light_dir=LIGHT_DIR, as_tensor=False):
    """synth.py:253-267 on the device: flat-albedo Lambert shading of the
    hit points of ``depth`` (numpy or CUDA tensor); invalid pixels black."""
    import torch

    from .volume import pose_struct

    scene = _as_scene(scene)
    dev = _device()
    prims, n = scene.device_prims(dev)
    d = torch.as_tensor(np.ascontiguousarray(depth) if isinstance(depth, np.ndarray) else depth,
                        dtype=torch.float64).to(f"cuda:{dev}").contiguous()
    if tuple(d.shape) != (intr.height, intr.width):
        raise ValueError(f"depth shape {tuple(d.shape)} != {(intr.height, intr.width)}")
    color = torch.empty((intr.height, intr.width, 3), dtype=torch.float64, device=f"cuda:{dev}")
    sp = _ref_params(Z_MAX_DEFAULT, SPHERE_TRACE_STEPS, SPHERE_TRACE_TOL, light_dir)
    ps = pose_struct(pose)
    st = L.lib().rf_synth_color(prims.data_ptr(), n, ctypes.byref(ps), float(intr.fx),
                                float(intr.fy), float(intr.cx), float(intr.cy), intr.width,
                                intr.height, ctypes.byref(sp), d.data_ptr(), color.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
    if st != L.RF_OK:
        raise RuntimeError("rf_synth_color failed")
    return color if as_tensor else color.cpu().numpy()


def add_noise(depth, seed, sigma0=SIGMA0_DEFAULT):
    """synth.py:270-283: sigma(z) = sigma0 * z^2 Gaussian noise from numpy's
    default_rng(seed) -- the generator's stream is sequential (ziggurat
    rejections consume a variable number of draws), so it is drawn on the
    host by the same call; invalid pixels stay invalid, crossings clamp."""
    noisy = np.array(depth, dtype=np.float64, copy=True)
    if sigma0 == 0.0:
        return noisy
    rng = np.random.default_rng(seed)
    valid = noisy > 0.0
    z = noisy[valid]
    noisy[valid] = np.maximum(z + rng.standard_normal(z.shape) * sigma0 * z * z, 0.0)
    return noisy


def gaussian_blur(color, sigma, as_tensor=False):
    """scipy.ndimage.gaussian_filter(color, sigma=(sigma, sigma, 0.0)) on the
    device (mode 'reflect', truncate 4.0; scipy's symmetric correlate1d loop
    order), as make_sequence blurs colour (synth.py:353-355)."""
    import torch

    dev = _device()
    c = torch.as_tensor(np.ascontiguousarray(color) if isinstance(color, np.ndarray) else color,
                        dtype=torch.float64).to(f"cuda:{dev}").clone().contiguous()
    if sigma > 1e-15:
        radius = int(4.0 * float(sigma) + 0.5)
        if radius > 63:
            raise ValueError("blur sigma too large for the device filter (radius > 63)")
        x = np.arange(-radius, radius + 1)  # scipy _gaussian_kernel1d(sigma, 0, radius)
        phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
        phi = phi / phi.sum()
        g = L.RfSynthGauss()
        g.r = radius
        for j in range(radius + 1):
            g.w[j] = float(phi[radius + j])
        h, w = c.shape[0], c.shape[1]
        tmp = torch.empty_like(c)
        st = L.lib().rf_synth_blur(c.data_ptr(), tmp.data_ptr(), w, h, ctypes.byref(g),
                                   torch.cuda.current_stream().cuda_stream)
        if st != L.RF_OK:
            raise RuntimeError("rf_synth_blur failed")
    return c if as_tensor else c.cpu().numpy()


def orbit_waypoints(n, radius=1.2, height=1.3, center=(0.0, 0.0), outward=True):
    """synth.py:154-175"""
    if n < 2:
        raise ValueError(f"need at least 2 waypoints, got {n}")
    cx, cy = center
    points = []
    for i in range(n + 1):
        ang = 2.0 * np.pi * (i % n) / n
        eye = np.array([cx + radius * np.cos(ang), cy + radius * np.sin(ang), height])
        if outward:
            target = np.array([cx + 2.0 * radius * np.cos(ang),
                               cy + 2.0 * radius * np.sin(ang), height])
        else:
            target = np.array([cx, cy, height])
        points.append(look_at_pose(eye, target))
    return points


@dataclass
class TrajectorySpec:
    """synth.py:178-213: waypoint path plus drift and correction schedule."""
    waypoints: list
    frames_per_segment: int = 20
    drift_rate: tuple = (0.0, 0.0)
    correction_schedule: list = None

    def __post_init__(self):
        if self.correction_schedule is None:
            self.correction_schedule = []
        if len(self.waypoints) < 2:
            raise ValueError("need at least two waypoints")
        if self.frames_per_segment < 1:
            raise ValueError("frames_per_segment must be >= 1")
        if len(self.drift_rate) != 2 or min(self.drift_rate) < 0.0:
            raise ValueError("drift_rate must be (meters, radians), both >= 0")
        prev = 0
        for frame, fraction in self.correction_schedule:
            if frame <= prev:
                raise ValueError("correction frames must be increasing")
            if not 0.0 <= fraction <= 1.0:
                raise ValueError(f"correction fraction {fraction} outside [0, 1]")
            prev = frame

    @property
    def n_frames(self):
        return (len(self.waypoints) - 1) * self.frames_per_segment + 1

    def pose_at(self, index):
        from .geometry import pose_interpolate as interp

        g = (index - 1) / self.frames_per_segment
        seg = min(int(np.floor(g)), len(self.waypoints) - 2)
        return interp(self.waypoints[seg], self.waypoints[seg + 1], g - seg)


@dataclass(frozen=True)
class RenderedFrame:
    index: int
    depth: object
    color: object


@dataclass
class SyntheticSequence:
    frames: list
    gt_poses: dict
    drifted_poses: dict
    events: list
    intrinsics: Intrinsics

    @property
    def n_frames(self):
        return len(self.frames)


def make_sequence(scene, spec, intr, seed=0, noise_sigma0=0.0, blur_sigma_max=0.0,
                  anchor_interval=DEFAULT_ANCHOR_INTERVAL, z_max=Z_MAX_DEFAULT,
                  render_color_images=True, as_tensor=False):
    """synth.py:310-390 with the pixels rendered on the device: frames at
    ground truth, an accumulating drift on the reported trajectory, anchors
    every ``anchor_interval`` frames and scheduled corrections -- the same
    frames, poses and events as the reference.  ``as_tensor`` keeps the
    frames in HBM (CUDA tensors) instead of returning numpy arrays."""
    import torch

    from .geometry import pose_interpolate as interp
    from .geometry import rotation_from_axis_angle
    from .reintegration import PoseUpdateEvent

    scene = _as_scene(scene)
    rng = np.random.default_rng(seed)
    drift_t, drift_r = spec.drift_rate
    t_dir = rng.standard_normal(3)
    t_dir /= np.linalg.norm(t_dir)
    r_axis = rng.standard_normal(3)
    r_axis /= np.linalg.norm(r_axis)
    step = Pose(rotation_from_axis_angle(r_axis, drift_r), drift_t * t_dir)
    schedule = {frame: fraction for frame, fraction in spec.correction_schedule}
    frames, events = [], []
    gt_poses, drifted_poses, anchor_true, anchor_believed = {}, {}, {}, {}
    drift = Pose.identity()
    for index in range(1, spec.n_frames + 1):
        gt = spec.pose_at(index)
        if scene.sdf(gt.translation[None, :])[0] <= 0.0:
            raise ValueError(f"camera at frame {index} is not in free space")
        if index > 1:
            drift = compose(step, drift)
        drifted = compose(drift, gt)
        gt_poses[index] = gt
        drifted_poses[index] = drifted
        depth = render_depth(scene, gt, intr, z_max=z_max, as_tensor=True)
        if noise_sigma0 > 0.0:
            depth = torch.from_numpy(add_noise(depth.cpu().numpy(), seed=(seed, 7, index),
                                               sigma0=noise_sigma0)).to(depth.device)
        color = None
        if render_color_images:
            color = render_color(scene, gt, intr, depth, as_tensor=True)
            if blur_sigma_max > 0.0:
                sigma = rng.uniform(0.0, blur_sigma_max)
                color = gaussian_blur(color, sigma, as_tensor=True)
        if not as_tensor:
            depth = depth.cpu().numpy()
            color = color.cpu().numpy() if color is not None else None
        frames.append(RenderedFrame(index=index, depth=depth, color=color))
        if (index - 1) % anchor_interval == 0:
            anchor_true[index] = gt
            anchor_believed[index] = drifted
            events.append(PoseUpdateEvent(at_frame=index, anchor_poses={index: drifted.copy()},
                                          dvo_kf_flags={index}))
        if index in schedule:
            fraction = schedule[index]
            updated = {}
            for aid in anchor_believed:
                corrected = interp(anchor_believed[aid], anchor_true[aid], fraction)
                anchor_believed[aid] = corrected
                updated[aid] = corrected.copy()
            events.append(PoseUpdateEvent(at_frame=index, anchor_poses=updated,
                                          dvo_kf_flags=set()))
    return SyntheticSequence(frames=frames, gt_poses=gt_poses, drifted_poses=drifted_poses,
                             events=events, intrinsics=intr)
