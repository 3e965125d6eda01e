"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the surface-correction hot path.

A slow, sequential restatement of the reference's volume semantics
(`/root/reference/pkg/src/refusion/volume.py`, `reintegration.py`) on top of
the plain-C kernels in ``rf_oracle.c`` (``liborc.so``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg may import
this module, and only as the checker; the product package never does.

The oracle is pinned against the reference by ``tests/test_oracle.py``,
which replays the golden vectors in ``tests/golden/`` (made by
``tests/golden/gen_golden.py`` from the reference itself).
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")

BLOCK_SIDE = 8
BLOCK_VOXELS = 512
EPS_W = 1e-9                 # volume.py:26
MIN_SAMPLE_Z_FACTOR = 0.25   # volume.py:30
PACK_BIAS = 1 << 20          # volume.py:35
PACK_SPAN = 1 << 21          # volume.py:36

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"oracle library {_LIB_PATH} not built (run `make -C oracle`)"
        )
    lib = ctypes.CDLL(_LIB_PATH)
    lib.orc_block_hash.restype = ctypes.c_int64
    lib.orc_block_hash.argtypes = [ctypes.c_int64] * 4
    lib.orc_fuse_block.restype = ctypes.c_int
    lib.orc_fuse_block.argtypes = (
        [_dp, _dp, _dp] + [ctypes.c_double] * 4 + [_dp]
        + [ctypes.c_double] * 7 + [ctypes.c_int, ctypes.c_int]
        + [_dp, _dp, _dp] + [ctypes.c_double, ctypes.c_double, ctypes.c_int]
    )
    lib.orc_footprint.restype = ctypes.c_int64
    lib.orc_footprint.argtypes = (
        [_dp, _dp, ctypes.c_int, ctypes.c_int] + [ctypes.c_double] * 4
        + [_dp, _dp, ctypes.c_double, ctypes.c_double, ctypes.c_int,
           ctypes.c_double, _lp, ctypes.c_int64]
    )
    return lib


_lib = _load()


def _ptr(a):
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------------------
# keys / hash  (volume.py:84-93, :137-148)


def block_hash(coord, buckets):
    if buckets <= 0:
        raise ValueError(f"buckets must be > 0, got {buckets}")
    return int(_lib.orc_block_hash(int(coord[0]), int(coord[1]), int(coord[2]),
                                   int(buckets)))


def pack_coords(bx, by, bz):
    bx, by, bz = (np.asarray(a, dtype=np.int64) for a in (bx, by, bz))
    return ((bx + PACK_BIAS) << 42) | ((by + PACK_BIAS) << 21) | (bz + PACK_BIAS)


def unpack_keys(keys):
    keys = np.asarray(keys, dtype=np.int64)
    kz = keys & (PACK_SPAN - 1)
    ky = (keys >> 21) & (PACK_SPAN - 1)
    kx = keys >> 42
    return kx - PACK_BIAS, ky - PACK_BIAS, kz - PACK_BIAS


def keys_to_coords(keys):
    bx, by, bz = unpack_keys(keys)
    return [(int(x), int(y), int(z)) for x, y, z in zip(bx, by, bz)]


# ---------------------------------------------------------------------------
# fuse_block  (_kernels_cy.pyx:14-108)


def fuse_block(d, w, c, ox, oy, oz, voxel_size, rot, tx, ty, tz,
               fx, fy, cx, cy, width, height, kf_depth, kf_weight, kf_color,
               mu, eps_w, remove):
    """Same signature and in-place semantics as ``refusion.kernels.fuse_block``."""
    for a in (d, w, c):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("block arrays must be C-contiguous float64")
    rot = np.ascontiguousarray(rot, dtype=np.float64)
    kd = np.ascontiguousarray(kf_depth, dtype=np.float64)
    kw = np.ascontiguousarray(kf_weight, dtype=np.float64)
    kc = None if kf_color is None else np.ascontiguousarray(kf_color, dtype=np.float64)
    return int(_lib.orc_fuse_block(
        _ptr(d), _ptr(w), _ptr(c), float(ox), float(oy), float(oz),
        float(voxel_size), _ptr(rot), float(tx), float(ty), float(tz),
        float(fx), float(fy), float(cx), float(cy), int(width), int(height),
        _ptr(kd), _ptr(kw), None if kc is None else _ptr(kc),
        float(mu), float(eps_w), 1 if remove else 0))


# ---------------------------------------------------------------------------
# footprint  (volume.py:151-197)


def n_steps_for(voxel_size, mu):
    return int(np.ceil(2.0 * mu / voxel_size)) + 1      # volume.py:172


def footprint_keys(depth, weight, intr, rotation, translation, voxel_size, mu):
    """Sorted unique packed keys of a keyframe's block footprint."""
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    weight = np.ascontiguousarray(weight, dtype=np.float64)
    rot = np.ascontiguousarray(rotation, dtype=np.float64)
    t = np.ascontiguousarray(translation, dtype=np.float64).reshape(3)
    span = BLOCK_SIDE * voxel_size
    inv_span = 1.0 / span                                  # volume.py:177
    cap = 1 << 16
    while True:
        out = np.empty(cap, dtype=np.int64)
        n = _lib.orc_footprint(
            _ptr(depth), _ptr(weight), int(intr.width), int(intr.height),
            float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
            _ptr(rot), _ptr(t), float(voxel_size), float(mu),
            n_steps_for(voxel_size, mu), inv_span,
            out.ctypes.data_as(_lp), cap)
        if n >= 0:
            return out[:n].copy()
        if n == -1:
            raise MemoryError("oracle footprint: out of memory")
        cap = -n


# ---------------------------------------------------------------------------
# store  (volume.py:69-123, :200-394)


class OracleError(Exception):
    pass


class StreamingContractError(OracleError):
    pass


class VolumeInconsistencyError(OracleError):
    pass


class Block:
    __slots__ = ("d", "w", "c")

    def __init__(self):
        self.d = np.zeros(BLOCK_VOXELS)
        self.w = np.zeros(BLOCK_VOXELS)
        self.c = np.zeros((BLOCK_VOXELS, 3))

    def copy(self):
        b = Block()
        b.d[:] = self.d
        b.w[:] = self.w
        b.c[:] = self.c
        return b


class OracleStore:
    """Restatement of TwoTierStore (volume.py:96-123) with explicit tiers."""

    def __init__(self, voxel_size, mu, stream_radius):
        self.voxel_size = float(voxel_size)
        self.mu = float(mu)
        self.stream_radius = float(stream_radius)
        self.span = BLOCK_SIDE * self.voxel_size
        self.active = {}
        self.host = {}
        self.blocks_streamed_in = 0
        self.blocks_streamed_out = 0
        self.sphere_relocations = 0
        self.last_center = None

    # -- helpers ------------------------------------------------------------
    def block_count(self):
        return len(self.active) + len(self.host)

    def find(self, coord):
        b = self.active.get(coord)
        return self.host.get(coord) if b is None else b

    def items(self):
        yield from self.active.items()
        yield from self.host.items()

    def _center_distance(self, coord):
        # volume.py:200-213 (Python float ** 2 -> libm pow, as the reference)
        span = self.span
        cx = (coord[0] + 0.5) * span
        cy = (coord[1] + 0.5) * span
        cz = (coord[2] + 0.5) * span
        c = self.last_center
        return float(np.sqrt((cx - c[0]) ** 2 + (cy - c[1]) ** 2 + (cz - c[2]) ** 2))

    # -- streaming (volume.py:341-379) --------------------------------------
    def _select(self, tier, center, outside):
        if not tier:
            return []
        keys = list(tier.keys())
        centers = (np.array(keys, dtype=np.float64) + 0.5) * self.span
        dist = np.linalg.norm(centers - center, axis=1)
        mask = dist > self.stream_radius if outside else dist <= self.stream_radius
        return [keys[i] for i in np.flatnonzero(mask)]

    def stream(self, center):
        center = np.asarray(center, dtype=np.float64).reshape(3)
        relocated = 0
        if self.last_center is not None:
            moved = float(np.linalg.norm(center - self.last_center))
            if moved > BLOCK_SIDE * self.voxel_size:
                relocated = 1
        self.last_center = center.copy()
        self.sphere_relocations += relocated
        out = self._select(self.active, center, True)
        for coord in out:
            self.host[coord] = self.active.pop(coord)
        into = self._select(self.host, center, False)
        for coord in into:
            self.active[coord] = self.host.pop(coord)
        self.blocks_streamed_out += len(out)
        self.blocks_streamed_in += len(into)
        return {"streamed_in": len(into), "streamed_out": len(out),
                "relocated": relocated}

    # -- allocation (volume.py:223-249) -------------------------------------
    def _allocate(self, coords):
        if not coords:
            return set()
        if self.last_center is None:
            raise StreamingContractError("stream() must position the sphere first")
        new = set()
        for coord in coords:
            if coord in self.active:
                continue
            dist = self._center_distance(coord)
            if coord in self.host:
                raise StreamingContractError(f"block {coord} sits in the host tier")
            if dist > self.stream_radius:
                raise StreamingContractError(f"block {coord} outside the sphere")
            self.active[coord] = Block()
            new.add(coord)
        return new

    def footprint(self, kf, pose):
        keys = footprint_keys(kf.depth, kf.weight, kf.intrinsics, pose.rotation,
                              pose.translation, self.voxel_size, self.mu)
        return keys_to_coords(keys)

    def _fuse(self, blk, coord, kf, pose, remove):
        # volume.py:252-293
        intr = kf.intrinsics
        span = self.span
        rot_wc = np.ascontiguousarray(np.asarray(pose.rotation).T, dtype=np.float64)
        t = np.asarray(pose.translation, dtype=np.float64)
        color = getattr(kf, "color", None)
        return fuse_block(
            blk.d, blk.w, blk.c, coord[0] * span, coord[1] * span,
            coord[2] * span, self.voxel_size, rot_wc, float(t[0]), float(t[1]),
            float(t[2]), intr.fx, intr.fy, intr.cx, intr.cy, intr.width,
            intr.height, kf.depth, kf.weight, color, self.mu, EPS_W, remove)

    def allocate_blocks(self, kf, pose):
        return self._allocate(self.footprint(kf, pose))

    def integrate(self, kf, pose):
        """volume.py:296-312; returns (new_coords, blocks_touched, voxels_updated)."""
        coords = self.footprint(kf, pose)
        new = self._allocate(coords)
        total = 0
        for coord in coords:
            total += self._fuse(self.active[coord], coord, kf, pose, False)
        return new, len(coords), total

    def deintegrate(self, kf, pose):
        """volume.py:315-338"""
        coords = self.footprint(kf, pose)
        self._allocate(coords)
        done = []
        for coord in coords:
            n = self._fuse(self.active[coord], coord, kf, pose, True)
            if n < 0:
                for prev in done:
                    self._fuse(self.active[prev], prev, kf, pose, False)
                raise VolumeInconsistencyError(f"negative weight in block {coord}")
            done.append(coord)

    def garbage_collect(self):
        """volume.py:382-390"""
        freed = 0
        for tier in (self.active, self.host):
            dead = [c for c, b in tier.items() if not b.w.any()]
            for c in dead:
                del tier[c]
            freed += len(dead)
        return freed

    def total_weight(self):
        """volume.py:393-394"""
        return float(sum(b.w.sum() for _, b in self.items()))

    # -- correction (reintegration.py:156-181) ------------------------------
    def correct_entries(self, entries):
        """entries: list of objects with .kf, .integrated_pose, .target_pose"""
        if not entries:
            return 0
        self.stream(entries[0].integrated_pose.translation)
        removed = []
        try:
            for e in entries:
                self.stream(e.integrated_pose.translation)
                self.deintegrate(e.kf, e.integrated_pose)
                removed.append(e)
        except VolumeInconsistencyError:
            for e in removed:
                self.stream(e.integrated_pose.translation)
                self.integrate(e.kf, e.integrated_pose)
            raise
        self.stream(entries[0].target_pose.translation)
        for e in entries:
            self.stream(e.target_pose.translation)
            self.integrate(e.kf, e.target_pose)
            e.integrated_pose = e.target_pose.copy()
        self.garbage_collect()
        return len(entries)

    # -- export in the shape the product's export uses ----------------------
    def export(self):
        """(sorted packed keys int64[n], d[n,512], w[n,512], c[n,512,3])"""
        coords = sorted(c for c, _ in self.items())
        n = len(coords)
        keys = pack_coords([c[0] for c in coords], [c[1] for c in coords],
                           [c[2] for c in coords]) if n else np.zeros(0, np.int64)
        d = np.zeros((n, BLOCK_VOXELS))
        w = np.zeros((n, BLOCK_VOXELS))
        c = np.zeros((n, BLOCK_VOXELS, 3))
        for i, coord in enumerate(coords):
            b = self.find(coord)
            d[i], w[i], c[i] = b.d, b.w, b.c
        return np.asarray(keys, dtype=np.int64), d, w, c
