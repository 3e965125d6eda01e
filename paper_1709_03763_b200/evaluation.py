"""Reconstruction quality metrics: the exact nearest-neighbour grid index on
the device.

Mirrors /root/reference/pkg/src/refusion/evaluation.py:108-251 -- GridIndex,
mad_correctness, mad_completeness -- with the same arguments, errors and
results bit for bit: the index (rf_grid_index_create / _query, csrc/
rf_eval.cu) buckets the points into cells on the device and each query scans
rings of cells outward, falling back to the exact linear scan where the
reference does; every distance is the IEEE square root of the exact minimum
squared distance, computed as the reference computes it.
"""

import ctypes

import numpy as np

from . import _lib as L
from .errors import EmptyInputError, EmptyModelError

DEFAULT_CELL_SIZE = 0.04  # evaluation.py:31


def _torch():
    import torch

    return torch


def _points_dev(points):
    torch = _torch()
    if isinstance(points, torch.Tensor):
        t = points.to(device=f"cuda:{torch.cuda.current_device()}", dtype=torch.float64)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    return torch.from_numpy(a).cuda()


class GridIndex:
    """Exact nearest-neighbour search over a uniform grid (device)."""

    def __init__(self, points, cell_size=DEFAULT_CELL_SIZE):
        host = points if not hasattr(points, "is_cuda") else None
        pts = np.asarray(points, dtype=np.float64) if host is not None else None
        if pts is not None:
            if pts.ndim != 2 or pts.shape[1] != 3 or pts.shape[0] == 0:
                raise EmptyInputError("index needs a non-empty (N, 3) point array")
            if not np.isfinite(pts).all():
                raise ValueError("index points must be finite")
        if cell_size <= 0.0:
            raise ValueError(f"cell_size must be > 0, got {cell_size}")
        torch = _torch()
        dev = _points_dev(pts if pts is not None else points)
        if dev.dim() != 2 or dev.shape[1] != 3 or dev.shape[0] == 0:
            raise EmptyInputError("index needs a non-empty (N, 3) point array")
        if pts is None and not bool(torch.isfinite(dev).all()):
            raise ValueError("index points must be finite")
        self.cell_size = float(cell_size)
        self.n_points = int(dev.shape[0])
        self.device = dev.device
        ptr = ctypes.c_void_p()
        st = L.lib().rf_grid_index_create(dev.data_ptr(), self.n_points, self.cell_size,
                                          ctypes.byref(ptr),
                                          torch.cuda.current_stream().cuda_stream)
        if st != L.RF_OK:
            raise RuntimeError(f"rf_grid_index_create: {L.lib().rf_status_string(st).decode()}")
        self._ptr = ptr

    def query(self, points):
        """Distances from each query point to its nearest indexed point
        (evaluation.py:216-227): a float for one point, else an array."""
        torch = _torch()
        if hasattr(points, "is_cuda"):
            q = points.to(self.device, torch.float64)
            single = q.dim() == 1
            q = q.reshape(-1, 3).contiguous()
        else:
            a = np.asarray(points, dtype=np.float64)
            single = a.ndim == 1
            q = _points_dev(np.atleast_2d(a))
        m = int(q.shape[0])
        out = torch.empty(m, dtype=torch.float64, device=self.device)
        st = L.lib().rf_grid_index_query(self._ptr, q.data_ptr(), m, out.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream)
        if st != L.RF_OK:
            raise RuntimeError(f"rf_grid_index_query: {L.lib().rf_status_string(st).decode()}")
        res = out.cpu().numpy()
        return float(res[0]) if single else res

    def close(self):
        if getattr(self, "_ptr", None) is not None and self._ptr.value:
            L.lib().rf_grid_index_destroy(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def _vertices(mesh):
    return getattr(mesh, "vertices", mesh)


def _points(cloud):
    return getattr(cloud, "points", cloud)


def mad_correctness(model, ref, cell_size=DEFAULT_CELL_SIZE):
    """Mean distance (mm) from model vertices to their nearest reference
    point (evaluation.py:230-239)."""
    verts, pts = np.asarray(_vertices(model)), np.asarray(_points(ref))
    if verts.shape[0] == 0:
        raise EmptyInputError("model mesh has no vertices")
    if pts.shape[0] == 0:
        raise EmptyInputError("reference cloud is empty")
    index = GridIndex(pts, cell_size)
    try:
        return 1000.0 * index.query(verts).mean()
    finally:
        index.close()


def mad_completeness(model, ref, cell_size=DEFAULT_CELL_SIZE):
    """Mean distance (mm) from reference points to the nearest model vertex
    (evaluation.py:242-251)."""
    verts, pts = np.asarray(_vertices(model)), np.asarray(_points(ref))
    if pts.shape[0] == 0:
        raise EmptyInputError("reference cloud is empty")
    if verts.shape[0] == 0:
        raise EmptyModelError("model mesh is empty: completeness is unbounded")
    index = GridIndex(verts, cell_size)
    try:
        return 1000.0 * index.query(pts).mean()
    finally:
        index.close()
