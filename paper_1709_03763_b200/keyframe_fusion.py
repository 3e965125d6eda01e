"""Keyframe fusion on the device: collapse bursts of RGB-D frames into keyframes.

Drop-in for ``refusion.keyframe_fusion``
(/root/reference/pkg/src/refusion/keyframe_fusion.py): same classes,
functions, constants and errors.  Keyframe planes (depth, weight, colour,
colour_valid) and the retained member buffers live in HBM as torch CUDA
tensors; every per-pixel step runs in librefusion_b200.so (rf_depth_weight,
rf_fuse_depth, rf_color_prep, rf_fuse_color), bit-for-bit with the reference
on the same host (see DESIGN.md §2 for the one host-dependent step, the BLAS
order of geometry.transform, calibrated by ``detect_blas_order``).
"""

import ctypes
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib as L
from .errors import UndefinedOverlapError
from .geometry import Intrinsics, Pose, compose, inverse, ray_grid, rotation_angle, transform
from .volume import pose_struct

DELTA_DISC = 0.1       # keyframe_fusion.py:27
DELTA_OCCL = 0.05
UNSHARP_SIGMA = 1.5
UNSHARP_GAIN = 0.5

KF_CONST = "KF_CONST"
KF_DVO = "KF_DVO"
KF_DIST = "KF_DIST"
KF_OVRLP = "KF_OVRLP"
STRATEGY_KINDS = (KF_CONST, KF_DVO, KF_DIST, KF_OVRLP)

RF_DW_MASK = 1
RF_DW_MASK_ONLY = 2


def _torch():
    import torch

    return torch


def _dev():
    torch = _torch()
    L.lib()
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _plane(a, shape=None):
    """CUDA float64 contiguous tensor from numpy / torch input."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a.to(device=_dev(), dtype=torch.float64).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(_dev())
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"plane shape {tuple(t.shape)} != {tuple(shape)}")
    return t


def _check(status, what):
    if status != L.RF_OK:
        raise RuntimeError(f"{what}: {L.lib().rf_status_string(status).decode()}")


# ---------------------------------------------------------------------------
# host BLAS order of geometry.transform (p @ R.T + t)

_BLAS_ORDER = None


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def detect_blas_order(samples=64, seed=12345):
    """Which multiply-add order numpy's p @ R.T uses on this host (the
    reference's fused depth depends on it).  Returns an
    rf_blas_order code; the result is cached."""
    global _BLAS_ORDER
    if _BLAS_ORDER is not None:
        return _BLAS_ORDER
    rng = np.random.default_rng(seed)
    R = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    p = rng.normal(size=(4096, 3)) * 3.0   # a BLAS-sized call, as fuse_depth makes
    got = p @ R.T
    cands = {
        1: lambda q, r: _fma(q[2], r[2], _fma(q[1], r[1], q[0] * r[0])),
        0: lambda q, r: (q[0] * r[0] + q[1] * r[1]) + q[2] * r[2],
        2: lambda q, r: _fma(q[0], r[0], _fma(q[1], r[1], q[2] * r[2])),
        3: lambda q, r: _fma(q[2], r[2], _fma(q[0], r[0], q[1] * r[1])),
    }
    idx = rng.choice(len(p), samples, replace=False)
    for code, f in cands.items():
        if all(f(p[i], R[k]) == got[i, k] for i in idx for k in range(3)):
            _BLAS_ORDER = code
            return code
    _BLAS_ORDER = 1  # closest known order; results then agree to rounding only
    return _BLAS_ORDER


# ---------------------------------------------------------------------------
# data classes (keyframe_fusion.py:39-135)


@dataclass
class FrameObservation:
    """One registered RGB-D input frame with its current pose estimate."""

    index: int
    color: object
    depth: object
    pose: Pose

    def __post_init__(self):
        if self.index < 1:
            raise ValueError(f"frame index must be >= 1, got {self.index}")
        torch = _torch()
        if isinstance(self.depth, torch.Tensor):
            if self.depth.dim() != 2:
                raise ValueError("depth must be a 2-d map")
            dmin = float(torch.nan_to_num(self.depth, nan=0.0, posinf=0.0).min()) \
                if self.depth.numel() else 0.0
        else:
            self.depth = np.asarray(self.depth, dtype=np.float64)
            if self.depth.ndim != 2:
                raise ValueError("depth must be a 2-d map")
            bad = self.depth[np.isfinite(self.depth)]
            dmin = bad.min() if bad.size else 0.0
        if self.color is not None and tuple(self.color.shape[:2]) != tuple(self.depth.shape):
            raise ValueError(f"color {tuple(self.color.shape[:2])} and depth "
                             f"{tuple(self.depth.shape)} dimensions differ")
        if dmin < 0.0:
            raise ValueError("depth values must be >= 0 (0 = invalid)")


@dataclass(frozen=True)
class KeyframeStrategy:
    kind: str = KF_CONST
    kappa: int = 20
    delta_r: float = 0.35
    delta_t: float = 0.3
    overlap_min: float = 0.7

    def __post_init__(self):
        if self.kind not in STRATEGY_KINDS:
            raise ValueError(f"unknown strategy kind {self.kind!r}")
        if self.kappa < 1:
            raise ValueError(f"kappa must be >= 1, got {self.kappa}")
        if self.delta_r <= 0 or self.delta_t <= 0:
            raise ValueError("KF_DIST thresholds must be > 0")
        if not 0.0 < self.overlap_min < 1.0:
            raise ValueError(f"overlap_min must be in (0,1), got {self.overlap_min}")


@dataclass
class _MemberObservation:
    """Per-member buffers (device) kept until colour finalisation."""

    index: int
    color: object          # deblurred [h][w][3] f64 tensor, or None
    depth: object          # [h][w] f64 tensor
    pose: Pose
    blur_weight: object    # device scalar tensor (1.0 without colour)
    weight_map: object     # [h][w] f64 tensor


@dataclass
class Keyframe:
    intrinsics: Intrinsics
    pose: Pose
    anchor_id: int
    rel_pose: Pose
    depth: object
    weight: object
    color: object = None
    color_valid: object = None
    members: list = field(default_factory=list)
    observations: list = field(default_factory=list)
    kf_id: int = -1

    @property
    def finalized(self):
        return self.observations is None


def new_keyframe(frame, intrinsics, anchor_id=0, anchor_pose=None):
    """keyframe_fusion.py:118-135"""
    if anchor_pose is None:
        anchor_pose = Pose.identity()
    shape = (intrinsics.height, intrinsics.width)
    if tuple(frame.depth.shape) != shape:
        raise ValueError(f"frame depth {tuple(frame.depth.shape)} does not match intrinsics {shape}")
    torch = _torch()
    return Keyframe(
        intrinsics=intrinsics,
        pose=frame.pose.copy(),
        anchor_id=anchor_id,
        rel_pose=compose(inverse(anchor_pose), frame.pose),
        depth=torch.zeros(shape, dtype=torch.float64, device=_dev()),
        weight=torch.zeros(shape, dtype=torch.float64, device=_dev()),
    )


# ---------------------------------------------------------------------------
# per-frame depth weighting (keyframe_fusion.py:142-231)


def _depth_weight(depth, intr, delta_disc, flags):
    torch = _torch()
    d = _plane(depth, (intr.height, intr.width))
    out = torch.empty_like(d)
    _check(L.lib().rf_depth_weight(d.data_ptr(), intr.width, intr.height, float(intr.fx),
                                   float(intr.fy), float(intr.cx), float(intr.cy),
                                   float(delta_disc), flags, out.data_ptr(), _stream()),
           "rf_depth_weight")
    return out


def normal_map(depth, intr):
    """Unit surface normals [h][w][3] from central differences of unprojected
    points; zero at the border and next to invalid depth (device;
    keyframe_fusion.py:142-188)."""
    torch = _torch()
    d = _plane(depth, (intr.height, intr.width))
    out = torch.empty((intr.height, intr.width, 3), dtype=torch.float64, device=d.device)
    _check(L.lib().rf_normal_map(d.data_ptr(), intr.width, intr.height, float(intr.fx),
                                 float(intr.fy), float(intr.cx), float(intr.cy),
                                 out.data_ptr(), _stream()), "rf_normal_map")
    return out


def depth_sample_weight(depth, intr, normals=None):
    """w_z = cos(theta) / Z^2, zero where invalid (device;
    keyframe_fusion.py:191-208); ``normals`` default to normal_map(depth)."""
    if normals is None:
        return _depth_weight(depth, intr, 0.0, 0)
    torch = _torch()
    d = _plane(depth, (intr.height, intr.width))
    n = _plane(normals, (intr.height, intr.width, 3))
    out = torch.empty_like(d)
    _check(L.lib().rf_depth_sample_weight_normals(
        d.data_ptr(), n.data_ptr(), intr.width, intr.height, float(intr.fx), float(intr.fy),
        float(intr.cx), float(intr.cy), out.data_ptr(), _stream()),
        "rf_depth_sample_weight_normals")
    return out


def discontinuity_mask(depth, delta_disc=DELTA_DISC):
    """True where a pixel must be discarded (device; bool tensor)."""
    d = _plane(depth)
    h, w = d.shape
    intr = Intrinsics(1.0, 1.0, 0.0, 0.0, w, h)  # the mask ignores intrinsics
    return _depth_weight(d, intr, delta_disc, RF_DW_MASK_ONLY) > 0.5


def depth_weight_map(depth, intr, delta_disc=DELTA_DISC):
    """fuse_depth's per-frame map: w_z with discontinuities zeroed (:245-246)."""
    return _depth_weight(depth, intr, delta_disc, RF_DW_MASK)


# ---------------------------------------------------------------------------
# colour prep (keyframe_fusion.py:303-346)


_GAUSS = {}


def _gauss_weights(sigma, truncate=4.0):
    """scipy.ndimage._gaussian_kernel1d(sigma, 0, radius) -- host numpy, as scipy
    (cached per (sigma, truncate))."""
    key = (float(sigma), float(truncate))
    if key not in _GAUSS:
        _GAUSS[key] = _gauss_weights_uncached(sigma, truncate)
    return _GAUSS[key]


def _gauss_weights_uncached(sigma, truncate=4.0):
    radius = int(truncate * float(sigma) + 0.5)
    sigma2 = sigma * sigma
    x = np.arange(-radius, radius + 1)
    phi_x = np.exp(-0.5 / sigma2 * x ** 2)
    phi_x = phi_x / phi_x.sum()
    return np.ascontiguousarray(phi_x), radius


def grayscale(image):
    torch = _torch()
    img = _plane(image)
    if img.dim() == 2:
        return img
    h, w = img.shape[:2]
    out = torch.empty((h, w), dtype=torch.float64, device=img.device)
    _check(L.lib().rf_grayscale(img.data_ptr(), w, h, out.data_ptr(), _stream()), "rf_grayscale")
    return out


def blurriness(image):
    """Perceptual sharpness in [0, 1] (device; returns a Python float)."""
    torch = _torch()
    f = grayscale(image)
    h, w = f.shape
    out = torch.empty((), dtype=torch.float64, device=f.device)
    _check(L.lib().rf_blurriness(f.data_ptr(), w, h, out.data_ptr(), _stream()), "rf_blurriness")
    return float(out.item())


def unsharp_mask(image, sigma=UNSHARP_SIGMA, gain=UNSHARP_GAIN):
    torch = _torch()
    img = _plane(image)
    shape = img.shape
    h, w = shape[0], shape[1]
    c = 1 if img.dim() == 2 else shape[2]
    wts, radius = _gauss_weights(sigma)
    out = torch.empty_like(img)
    _check(L.lib().rf_unsharp_mask(img.data_ptr(), w, h, c, wts.ctypes.data_as(L.c_double_p),
                                   radius, float(gain), out.data_ptr(), _stream()),
           "rf_unsharp_mask")
    return out


def weighted_median(values, weights):
    """Host utility (keyframe_fusion.py:349-359): smallest value whose
    cumulative weight reaches half the total; lower value on an exact split."""
    values = np.asarray(values, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    if values.size == 0 or weights.sum() <= 0:
        raise ValueError("weighted median of no observations")
    order = np.argsort(values, kind="stable")
    cum = np.cumsum(weights[order])
    return float(values[order][np.searchsorted(cum, cum[-1] / 2.0)])


# ---------------------------------------------------------------------------
# fusion (keyframe_fusion.py:238-460)


def fuse_depth(kf, frame, delta_disc=DELTA_DISC):
    """Warp one frame into the keyframe and apply the running weighted
    average per target pixel; member buffers are retained on the device.
    One native call per frame (rf_fuse_frame): weight map, depth copy, warp +
    ordered scatter + Eq. 1 merge, colour prep."""
    if kf.finalized:
        raise ValueError("keyframe color already finalized; cannot add frames")
    torch = _torch()
    intr = kf.intrinsics
    h, w = intr.height, intr.width
    depth = _plane(frame.depth, (h, w))
    w_map = torch.empty_like(depth)
    depth_copy = torch.empty_like(depth)
    rel = pose_struct(compose(inverse(kf.pose), frame.pose))
    member_color = None
    color = None
    if frame.color is not None:
        color = _plane(frame.color, (h, w, 3))
        member_color = torch.empty_like(color)
        blur = torch.empty((), dtype=torch.float64, device=depth.device)
    else:
        blur = torch.ones((), dtype=torch.float64, device=depth.device)
    wts, radius = _gauss_weights(UNSHARP_SIGMA)
    _check(L.lib().rf_fuse_frame(
        kf.depth.data_ptr(), kf.weight.data_ptr(), depth.data_ptr(),
        color.data_ptr() if color is not None else None, w, h, float(intr.fx),
        float(intr.fy), float(intr.cx), float(intr.cy), ctypes.byref(rel), detect_blas_order(),
        float(delta_disc), wts.ctypes.data_as(L.c_double_p), radius, UNSHARP_GAIN,
        w_map.data_ptr(), depth_copy.data_ptr(),
        member_color.data_ptr() if member_color is not None else None,
        blur.data_ptr() if color is not None else None, _stream()), "rf_fuse_frame")
    kf.members.append(frame.index)
    kf.observations.append(_MemberObservation(
        index=frame.index, color=member_color, depth=depth_copy, pose=frame.pose.copy(),
        blur_weight=blur, weight_map=w_map))
    return kf


def fuse_color(kf, delta_occl=DELTA_OCCL):
    """Finalise the keyframe colour as the per-channel blur-weighted median of
    the member observations, then drop the member buffers."""
    if kf.finalized:
        raise ValueError("keyframe color already finalized")
    torch = _torch()
    intr = kf.intrinsics
    h, w = intr.height, intr.width
    kf.color = torch.zeros((h, w, 3), dtype=torch.float64, device=kf.depth.device)
    valid = torch.zeros((h, w), dtype=torch.uint8, device=kf.depth.device)
    members = [m for m in kf.observations if m.color is not None]
    views = (L.RfMemberView * max(len(members), 1))()
    for i, m in enumerate(members):
        views[i].depth = m.depth.data_ptr()
        views[i].w_map = m.weight_map.data_ptr()
        views[i].color = m.color.data_ptr()
        views[i].blur_weight = m.blur_weight.data_ptr()
        views[i].rel = pose_struct(compose(inverse(m.pose), kf.pose))
    _check(L.lib().rf_fuse_color(kf.depth.data_ptr(), kf.weight.data_ptr(), w, h,
                                 float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                                 len(members), views, float(delta_occl), detect_blas_order(),
                                 kf.color.data_ptr(), valid.data_ptr(), _stream()),
           "rf_fuse_color")
    kf.color_valid = valid.bool()
    kf.observations = None
    return kf


# ---------------------------------------------------------------------------
# keyframe boundary decisions (host, keyframe_fusion.py:467-511)


def _host(a):
    torch = _torch()
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def overlap_ratio(kf, frame, delta_occl=DELTA_OCCL):
    """Fraction of the keyframe's valid pixels visible in the frame (host)."""
    intr = kf.intrinsics
    weight, depth, fdepth = _host(kf.weight), _host(kf.depth), _host(frame.depth)
    valid = weight > 0.0
    total = int(valid.sum())
    if total == 0:
        raise UndefinedOverlapError("keyframe has no valid depth pixels")
    z = depth[valid]
    dir_x, dir_y = ray_grid(intr)
    p_star = np.stack([dir_x[valid] * z, dir_y[valid] * z, z], axis=1)
    q = transform(compose(inverse(frame.pose), kf.pose), p_star)
    qz = q[:, 2]
    front = qz > 0
    if not front.any():
        return 0.0
    u = np.floor(intr.fx * q[front, 0] / qz[front] + intr.cx + 0.5)
    v = np.floor(intr.fy * q[front, 1] / qz[front] + intr.cy + 0.5)
    inb = (u >= 0) & (u < intr.width) & (v >= 0) & (v < intr.height)
    if not inb.any():
        return 0.0
    zn = fdepth[v[inb].astype(np.int64), u[inb].astype(np.int64)]
    agree = (zn > 0) & (np.abs(zn - qz[front][inb]) <= delta_occl)
    return float(agree.sum()) / total


def keyframe_decision(strategy, kf, frame, dvo_kf_flags=None):
    """True when a new keyframe must start before fusing this frame."""
    if not kf.members:
        return False
    if strategy.kind == KF_CONST:
        return len(kf.members) >= strategy.kappa
    if strategy.kind == KF_DVO:
        return bool(dvo_kf_flags) and frame.index in dvo_kf_flags
    if strategy.kind == KF_DIST:
        rel = compose(inverse(kf.pose), frame.pose)
        return (rotation_angle(rel.rotation) > strategy.delta_r
                or float(np.linalg.norm(rel.translation)) > strategy.delta_t)
    if strategy.kind == KF_OVRLP:
        return overlap_ratio(kf, frame) < strategy.overlap_min
    raise ValueError(f"unknown strategy kind {strategy.kind!r}")
