"""Host-side pose algebra feeding the kernels' scalar arguments.

Mirrors /root/reference/pkg/src/refusion/geometry.py (Pose :41-62,
transform :101-104, compose :107-109, inverse :112-114, pose_distance
:160-170, ray_grid :266-275).  The expressions are evaluated with the same
numpy operations in the same order, so poses composed here are bit-identical
to the reference's on the same host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ORTHONORMAL_TOL = 1e-6
DEFAULT_DISTANCE_SCALE = np.array([2.0, 2.0, 2.0, 1.0, 1.0, 1.0])
_EYE3 = np.eye(3)
_EYE3.flags.writeable = False


@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point must lie inside the image")


@dataclass
class Pose:
    """p_world = rotation @ p_cam + translation."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        R = self.rotation
        err = np.abs(R.T @ R - _EYE3).max()
        if err > ORTHONORMAL_TOL:
            raise ValueError(f"rotation not orthonormal (err={err:.2e})")
        # the determinant test of geometry.py:52-53: a cofactor expansion
        # decides it, except within 1e-9 of the tolerance, where LAPACK's LU
        # determinant (the reference's np.linalg.det) does
        if R.shape == (3, 3):
            (a, b, c), (d, e, f), (g, h, i) = R.tolist()
            dev = abs(a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g) - 1.0)
            if abs(dev - ORTHONORMAL_TOL) < 1e-9:
                dev = abs(np.linalg.det(R) - 1.0)
        else:
            dev = abs(np.linalg.det(R) - 1.0)
        if dev > ORTHONORMAL_TOL:
            raise ValueError("rotation must have determinant +1")

    @classmethod
    def identity(cls):
        return cls(np.eye(3), np.zeros(3))

    def copy(self):
        # a copy of a validated pose is valid: skip __post_init__'s checks
        out = object.__new__(Pose)
        out.rotation = self.rotation.copy()
        out.translation = self.translation.copy()
        memo = self.__dict__.get("_rf_euler")
        if memo is not None:
            out._rf_euler = memo
        return out


def transform(T, p):
    p = np.asarray(p, dtype=np.float64)
    return p @ T.rotation.T + T.translation


def compose(T, U):
    """Apply U first, then T."""
    return Pose(T.rotation @ U.rotation, T.rotation @ U.translation + T.translation)


def inverse(T):
    r_inv = T.rotation.T
    return Pose(r_inv, -r_inv @ T.translation)


def rotation_x(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], dtype=np.float64)


def rotation_y(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], dtype=np.float64)


def rotation_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], dtype=np.float64)


def euler_zyx(R):
    """(yaw, pitch, roll); at the gimbal singularity roll is 0 and the
    remaining rotation is attributed to yaw (geometry.py:137-157)."""
    sp = min(1.0, max(-1.0, -R[2, 0]))
    pitch = np.arcsin(sp)
    if abs(sp) < 1.0 - 1e-12:
        yaw = np.arctan2(R[1, 0], R[0, 0])
        roll = np.arctan2(R[2, 1], R[2, 2])
    else:
        yaw = np.arctan2(-R[0, 1], R[1, 1])
        roll = 0.0
    return np.array([yaw, pitch, roll], dtype=np.float64)


def wrap_angle(a):
    return np.pi - np.mod(np.pi - np.asarray(a, dtype=np.float64), 2.0 * np.pi)


def _euler_of(pose):
    """euler_zyx(pose.rotation), memoised on the pose object while its
    rotation holds the same bits."""
    rb = pose.rotation.tobytes()
    memo = pose.__dict__.get("_rf_euler")
    if memo is not None and memo[0] == rb:
        return memo[1]
    e = euler_zyx(pose.rotation)
    e.flags.writeable = False
    try:
        pose._rf_euler = (rb, e)
    except AttributeError:
        pass
    return e


def pose_distance(T, U, s=DEFAULT_DISTANCE_SCALE):
    """Scaled norm of (wrapped Euler difference, translation difference)."""
    ea, eb = _euler_of(T), _euler_of(U)
    d = np.concatenate([wrap_angle(ea - eb), T.translation - U.translation])
    return float(np.linalg.norm(np.asarray(s, dtype=np.float64) * d))


def rotation_angle(R):
    cos_a = min(1.0, max(-1.0, (np.trace(R) - 1.0) / 2.0))
    angle = float(np.arccos(cos_a))
    return 0.0 if angle < 1e-12 else angle


def rotation_from_axis_angle(axis, angle):
    """Rodrigues rotation about a (not necessarily unit) axis
    (reference geometry.py:177-185, same expressions)."""
    axis = np.asarray(axis, dtype=np.float64)
    n = np.linalg.norm(axis)
    if n == 0 or angle == 0:
        return np.eye(3)
    x, y, z = axis / n
    K = np.array([[0, -z, y], [z, 0, -x], [-y, x, 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


def axis_angle_from_rotation(R):
    """Inverse of Rodrigues: (unit axis, angle in [0, pi])
    (reference geometry.py:188-204, same expressions)."""
    cos_a = min(1.0, max(-1.0, (np.trace(R) - 1.0) / 2.0))
    angle = float(np.arccos(cos_a))
    if angle < 1e-12:
        return np.array([1.0, 0.0, 0.0]), 0.0
    if np.pi - angle < 1e-6:
        M = (R + np.eye(3)) / 2.0
        axis = np.sqrt(np.maximum(np.diag(M), 0.0))
        k = int(np.argmax(axis))
        if axis[k] > 0:
            axis = M[:, k] / axis[k]
        return axis / np.linalg.norm(axis), angle
    v = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    return v / (2.0 * np.sin(angle)), angle


def pose_interpolate(T, U, t):
    """Geodesic interpolation T (t=0) -> U (t=1) (reference
    geometry.py:211-217): the synthetic trajectories' poses, bit for bit."""
    rel_R = T.rotation.T @ U.rotation
    axis, angle = axis_angle_from_rotation(rel_R)
    R = T.rotation @ rotation_from_axis_angle(axis, angle * t)
    trans = (1.0 - t) * T.translation + t * U.translation
    return Pose(R, trans)


def ray_grid(k):
    """Unit-depth ray directions ((u-cx)/fx, (v-cy)/fy), each (height, width)."""
    u = np.arange(k.width, dtype=np.float64)
    v = np.arange(k.height, dtype=np.float64)
    dir_x = np.broadcast_to((u - k.cx) / k.fx, (k.height, k.width))
    dir_y = np.broadcast_to(((v - k.cy) / k.fy)[:, None], (k.height, k.width))
    return np.ascontiguousarray(dir_x), np.ascontiguousarray(dir_y)


# ---------------------------------------------------------------------------
# batched host pose algebra for the correction scheduler: the same numpy
# operations as compose / euler_zyx / pose_distance above, over stacks.  A
# stacked np.matmul runs the scalar call's BLAS kernel per matrix, and the
# ufuncs run elementwise, so the results are the same bits; batch_exact()
# checks that once on this host (BLAS builds and SIMD ufunc loops differ
# between machines) and the callers fall back to the per-pose path if not.

_BATCH_OK = None


def compose_many(Ts, Us):
    """[compose(T, U) for T, U in zip(Ts, Us)] -- one batched matmul; poses
    whose validation lands within 1e-12 of the tolerance (or fails) are
    rebuilt with the checked constructor."""
    n = len(Us)
    if n == 0:
        return []
    RT = np.array([T.rotation for T in Ts])
    R = np.matmul(RT, np.array([U.rotation for U in Us]))
    t = np.matmul(RT, np.array([U.translation for U in Us])[..., None])[..., 0] + \
        np.array([T.translation for T in Ts])
    err = np.abs(np.matmul(R.transpose(0, 2, 1), R) - _EYE3).max(axis=(1, 2))
    a, b, c = R[:, 0, 0], R[:, 0, 1], R[:, 0, 2]
    d, e, f = R[:, 1, 0], R[:, 1, 1], R[:, 1, 2]
    g, h, i = R[:, 2, 0], R[:, 2, 1], R[:, 2, 2]
    dev = np.abs(a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g) - 1.0)
    safe = (err < ORTHONORMAL_TOL - 1e-12) & (np.abs(dev - ORTHONORMAL_TOL) >= 1e-9) & \
        (dev <= ORTHONORMAL_TOL)
    out = []
    for k in range(n):
        if safe[k]:
            p = object.__new__(Pose)
            p.rotation = R[k].copy()
            p.translation = t[k].copy()
        else:
            p = Pose(R[k], t[k])  # the exact checks (and their errors)
        out.append(p)
    return out


def euler_zyx_many(R):
    """euler_zyx over a stack [n][3][3] -> [n][3]."""
    sp = np.minimum(1.0, np.maximum(-1.0, -R[:, 2, 0]))
    pitch = np.arcsin(sp)
    reg = np.abs(sp) < 1.0 - 1e-12
    yaw = np.where(reg, np.arctan2(R[:, 1, 0], R[:, 0, 0]), np.arctan2(-R[:, 0, 1], R[:, 1, 1]))
    roll = np.where(reg, np.arctan2(R[:, 2, 1], R[:, 2, 2]), 0.0)
    return np.stack([yaw, pitch, roll], axis=1)


def pose_distance_many(As, Bs, s=DEFAULT_DISTANCE_SCALE):
    """[pose_distance(A, B, s)] over two lists of poses."""
    n = len(As)
    if n == 0:
        return np.empty(0)
    ea = euler_zyx_many(np.array([p.rotation for p in As]))
    eb = euler_zyx_many(np.array([p.rotation for p in Bs]))
    tA = np.array([p.translation for p in As])
    tB = np.array([p.translation for p in Bs])
    D = np.concatenate([wrap_angle(ea - eb), tA - tB], axis=1) * np.asarray(s, dtype=np.float64)
    return np.sqrt(np.array([np.dot(r, r) for r in D]))  # np.linalg.norm: sqrt(dot(x, x))


def batch_exact():
    """Do the batched forms give the per-pose bits on this host?  (cached)"""
    global _BATCH_OK
    if _BATCH_OK is None:
        rng = np.random.default_rng(20261017)
        ok = True
        for _ in range(4):
            def rp(scale):
                q = rng.normal(size=4)
                q /= np.linalg.norm(q)
                w, x, y, z = q
                R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                              [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                              [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
                return Pose(R, rng.normal(size=3) * scale)
            T = rp(3.0)
            rels = [rp(1.0) for _ in range(33)]
            many = compose_many([T] * len(rels), rels)
            one = [compose(T, U) for U in rels]
            ok &= all(np.array_equal(a.rotation, b.rotation) and
                      np.array_equal(a.translation, b.translation) for a, b in zip(many, one))
            others = [rp(2.0) for _ in range(33)]
            dm = pose_distance_many(one, others)
            ds = np.array([pose_distance(a, b) for a, b in zip(one, others)])
            ok &= bool(np.array_equal(dm, ds))
        _BATCH_OK = bool(ok)
    return _BATCH_OK
