"""The reference's kernel plugin point, served by the B200 library.

``refusion.kernels`` (/root/reference/pkg/src/refusion/kernels.py:19-41)
exports ``BACKEND``, ``fuse_block`` and ``nn_min_d2``.  This module exports
the same names; ``nn_min_d2`` (the evaluation metrics' nearest-point scan)
runs on the device too; ``fuse_block`` runs the sm_100a integrate / de-integrate
device code on one block (host arrays in, modified in place), with the same
argument meaning and the same return convention (voxel count, or -1 with
the block untouched on a removal-consistency failure,
_kernels_cy.pyx:14-108).

The per-block call exists for drop-in parity; the throughput path is the
batched volume API (``volume.integrate`` / ``reintegration``), which never
crosses the host per block.
"""

import numpy as np

from . import _lib as L

BACKEND = "b200"


def _f64(a, shape, name):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous float64 ndarray")
    if a.shape != shape:
        raise ValueError(f"{name} has shape {a.shape}, expected {shape}")
    return a.ctypes.data_as(L.c_double_p)


def fuse_block(d, w, c, ox, oy, oz, voxel_size, rot, tx, ty, tz, fx, fy, cx, cy,
               width, height, kf_depth, kf_weight, kf_color, mu, eps_w, remove):
    pd = _f64(d, (512,), "d")
    pw = _f64(w, (512,), "w")
    pc = _f64(c, (512, 3), "c")
    rot = np.ascontiguousarray(rot, dtype=np.float64)
    kd = np.ascontiguousarray(kf_depth, dtype=np.float64)
    kw = np.ascontiguousarray(kf_weight, dtype=np.float64)
    h, wd = int(height), int(width)
    if kd.shape != (h, wd) or kw.shape != (h, wd):
        raise ValueError("keyframe planes do not match width/height")
    kc = None
    if kf_color is not None:
        kc = np.ascontiguousarray(kf_color, dtype=np.float64)
        if kc.shape != (h, wd, 3):
            raise ValueError("keyframe color does not match width/height")
    count = L.ctypes.c_int32()
    st = L.lib().rf_fuse_block(
        pd, pw, pc, float(ox), float(oy), float(oz), float(voxel_size),
        rot.ctypes.data_as(L.c_double_p), float(tx), float(ty), float(tz),
        float(fx), float(fy), float(cx), float(cy), wd, h,
        kd.ctypes.data_as(L.c_double_p), kw.ctypes.data_as(L.c_double_p),
        None if kc is None else kc.ctypes.data_as(L.c_double_p),
        float(mu), float(eps_w), 1 if remove else 0, L.ctypes.byref(count))
    if st != L.RF_OK:
        raise RuntimeError(f"rf_fuse_block failed: {L.lib().rf_status_string(st).decode()}")
    return int(count.value)


def nn_min_d2(q, pts, out):
    """_kernels_cy.pyx:111-129 on the device (rf_nn_min_d2): out[i] = min over
    pts of (dx*dx + dy*dy) + dz*dz, bit for bit (the min is exact, so the
    device's point order cannot change it).  Same arguments: C-contiguous
    float64 q [n, 3], pts [m, 3], out [n], written in place."""
    n = q.shape[0] if isinstance(q, np.ndarray) else -1
    m = pts.shape[0] if isinstance(pts, np.ndarray) else -1
    pq = _f64(q, (n, 3), "q")
    pp = _f64(pts, (m, 3), "pts")
    po = _f64(out, (n,), "out")
    st = L.lib().rf_nn_min_d2(pq, n, pp, m, po, None)
    if st != L.RF_OK:
        raise RuntimeError(f"rf_nn_min_d2 failed: {L.lib().rf_status_string(st).decode()}")


__all__ = ["BACKEND", "fuse_block", "nn_min_d2"]
