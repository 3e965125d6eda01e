"""Deterministic, seeded inputs shared by the golden-vector generator
(tests/golden/gen_golden.py, which runs the reference) and the tests (which
run the oracle and the CUDA path).  Nothing here imports the reference or
the product: it only builds numpy inputs and describes operation scripts.

The generators restate the reference tests' own fixtures:
 * ``fuse_block_case``   -- tests/test_kernels_parity.py:18-51
 * ``random_frame``      -- tests/test_volume.py:27-33
 * ``single_ray_frame``  -- tests/test_volume.py:93-100
(paths under /root/reference/pkg/).
"""

import hashlib
from collections import namedtuple

import numpy as np

Intr = namedtuple("Intr", "fx fy cx cy width height")

SMALL_INTR = Intr(15.0, 15.0, 7.5, 5.5, 16, 12)
TINY_INTR = Intr(100.0, 100.0, 2.0, 2.0, 5, 5)
MID_INTR = Intr(50.0, 50.0, 31.5, 23.5, 64, 48)
QVGA_INTR = Intr(262.5, 262.5, 159.5, 119.5, 320, 240)
VGA_INTR = Intr(525.0, 525.0, 319.5, 239.5, 640, 480)


class SPose:
    """Minimal pose: p_world = rotation @ p_cam + translation."""

    def __init__(self, rotation, translation):
        self.rotation = np.asarray(rotation, dtype=np.float64)
        self.translation = np.asarray(translation, dtype=np.float64).reshape(3)

    def copy(self):
        return SPose(self.rotation.copy(), self.translation.copy())


class Frame:
    """Duck-typed keyframe: exactly the attributes the volume API reads
    (reference tests/test_volume.py:12-20)."""

    def __init__(self, depth, weight, color, intrinsics):
        self.depth = depth
        self.weight = weight
        self.color = color
        self.intrinsics = intrinsics


class Entry:
    """Duck-typed ledger entry (reintegration.py:28-35) for _correct_entries."""

    def __init__(self, kf, integrated_pose, target_pose):
        self.kf = kf
        self.integrated_pose = integrated_pose
        self.target_pose = target_pose


def rot_x(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], dtype=np.float64)


def rot_y(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], dtype=np.float64)


def rot_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], dtype=np.float64)


def identity():
    return SPose(np.eye(3), np.zeros(3))


def random_frame(rng, intr=SMALL_INTR, z_lo=1.0, z_hi=2.0, holes=0.2,
                 with_color=True):
    shape = (intr.height, intr.width)
    depth = rng.uniform(z_lo, z_hi, shape)
    weight = rng.uniform(0.5, 2.0, shape)
    weight[rng.random(shape) < holes] = 0.0
    color = rng.uniform(0.0, 1.0, shape + (3,)) if with_color else None
    return Frame(depth, weight, color, intr)


def single_ray_frame(depth_m):
    depth = np.zeros((5, 5))
    weight = np.zeros((5, 5))
    depth[2, 2] = depth_m
    weight[2, 2] = 1.0
    return Frame(depth, weight, None, TINY_INTR)


def wall_frame(intr, z, rng=None, tilt=0.0, noise=0.0, holes=0.0):
    """A (possibly tilted, noisy) plane in front of the camera."""
    h, w = intr.height, intr.width
    u = np.arange(w, dtype=np.float64)
    v = np.arange(h, dtype=np.float64)
    xn = (u - intr.cx) / intr.fx
    depth = np.empty((h, w))
    for r in range(h):
        # plane z = z0 + tilt * x  ->  depth along ray: z0 / (1 - tilt * xn)
        depth[r] = z / (1.0 - tilt * xn)
    weight = np.full((h, w), 1.0)
    if rng is not None and noise > 0:
        depth += rng.normal(0.0, noise, depth.shape) * depth * depth
    if rng is not None and holes > 0:
        weight[rng.random((h, w)) < holes] = 0.0
    color = np.empty((h, w, 3))
    color[..., 0] = (u[None, :] * 3.0) % 255.0
    color[..., 1] = (v[:, None] * 5.0) % 255.0
    color[..., 2] = 128.0
    return Frame(depth, weight, color, intr)


def fuse_block_case(rng, mode):
    """tests/test_kernels_parity.py:18-51"""
    d = np.zeros(512)
    w = np.zeros(512)
    c = np.zeros((512, 3))
    if mode == "sparse":
        seen = rng.random(512) < 0.6
        w[seen] = rng.uniform(0.25, 4.0, seen.sum())
        d[seen] = rng.uniform(-0.06, 0.06, seen.sum())
        c[seen] = rng.uniform(0.0, 1.0, (seen.sum(), 3))
    elif mode == "full":
        w[:] = rng.uniform(2.5, 4.0, 512)
        d[:] = rng.uniform(-0.06, 0.06, 512)
        c[:] = rng.uniform(0.0, 1.0, (512, 3))
    h, wd = 12, 16
    depth = rng.uniform(0.2, 1.2, (h, wd))
    weight = rng.uniform(0.0, 2.0, (h, wd))
    weight[rng.random((h, wd)) < 0.3] = 0.0
    color = rng.uniform(0.0, 1.0, (h, wd, 3))
    theta = rng.uniform(-0.4, 0.4)
    rot = np.ascontiguousarray(rot_y(theta))
    cam = rng.uniform(-0.3, 0.3, 3)
    intr = (12.0, 12.0, 7.5, 5.5, wd, h)
    origin = rng.uniform(-0.2, 0.2, 3) + np.array([0.0, 0.0, 0.4])
    return (d, w, c), (origin, 0.01, rot, cam, intr, depth, weight, color)


def fuse_block_cases():
    """[(state, scene, remove)] -- integrate, removal (incl. failures) and
    integrate-then-remove round trips (second element remove=='roundtrip')."""
    out = []
    rng = np.random.default_rng(101)
    for trial in range(24):
        st, sc = fuse_block_case(rng, "sparse" if trial % 2 == 0 else "empty")
        out.append((st, sc, False))
    rng = np.random.default_rng(202)
    for trial in range(24):
        st, sc = fuse_block_case(rng, "full" if trial % 2 == 0 else "sparse")
        out.append((st, sc, True))
    rng = np.random.default_rng(303)
    for _ in range(8):
        st, sc = fuse_block_case(rng, "empty")
        out.append((st, sc, "roundtrip"))
    return out


# ---------------------------------------------------------------------------
# footprint cases


def footprint_cases():
    """[(name, frame, pose, voxel_size, mu)]"""
    cases = []
    rng = np.random.default_rng(7)
    cases.append(("single_ray_2m", single_ray_frame(2.0), identity(), 0.01, 0.08))
    cases.append(("single_ray_near", single_ray_frame(0.03), identity(), 0.01, 0.06))
    f = random_frame(rng)
    cases.append(("small_identity", f, identity(), 0.01, 0.06))
    cases.append(("small_rot", random_frame(rng),
                  SPose(rot_y(0.2), [0.1, -0.05, 0.02]), 0.01, 0.06))
    cases.append(("small_rot5mm", random_frame(rng),
                  SPose(rot_z(0.7) @ rot_x(-0.3), [-1.3, 2.05, 0.4]), 0.005, 0.06))
    g = random_frame(rng, intr=MID_INTR, z_lo=0.3, z_hi=4.0, holes=0.3)
    g.depth[rng.random(g.depth.shape) < 0.05] = np.nan
    g.depth[rng.random(g.depth.shape) < 0.05] = np.inf
    g.depth[rng.random(g.depth.shape) < 0.05] = 0.0
    g.depth[rng.random(g.depth.shape) < 0.05] = 0.02   # below mu: zlo clamps
    cases.append(("mid_invalids", g, SPose(rot_y(-0.5) @ rot_x(0.1),
                                           [0.3, 0.2, -0.7]), 0.004, 0.05))
    q = wall_frame(QVGA_INTR, 1.4, rng=rng, tilt=0.3, noise=0.0015, holes=0.02)
    cases.append(("qvga_wall", q, SPose(rot_z(2.1) @ rot_y(0.3), [5.0, -3.0, 1.2]),
                  0.005, 0.06))
    e = random_frame(rng)
    e.weight[:] = 0.0
    cases.append(("empty", e, identity(), 0.01, 0.06))
    return cases


def hash_cases():
    coords = [(0, 0, 0), (3, -7, 11), (-1, -2, -3), (100, -200, 300),
              (-12345, 0, 999), (1, 1, 1), (1048575, -1048576, 77),
              (-1048576, 1048575, -1048576), (524287, 524287, -524288)]
    buckets = [1, 7, 4096, 65536, 1 << 22, 1000003, (1 << 31) - 1]
    rng = np.random.default_rng(5)
    for _ in range(40):
        coords.append(tuple(int(x) for x in rng.integers(-(1 << 20), 1 << 20, 3)))
    return [(c, b) for c in coords for b in buckets]


# ---------------------------------------------------------------------------
# volume operation scripts
#
# ops: ("stream", center) | ("integrate", kf, pose) | ("deintegrate", kf, pose)
#      | ("gc",) | ("total_weight",) | ("correct", [(kf, old, new)...], next)
# kf / pose / old / new index into the scenario's frame / pose lists.


def volume_scripts():
    """[(name, cfg dict, frames, poses, ops)]"""
    out = []
    rng = np.random.default_rng(17)
    frames = [random_frame(rng) for _ in range(3)]
    poses = [SPose(rot_y(0.2), [0.1, -0.05, 0.02]), identity(),
             SPose(np.eye(3), [1.0, 0.0, 0.0])]
    cfg = dict(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    out.append(("int_int_deint_gc", cfg, frames, poses, [
        ("stream", [0.1, -0.05, 0.02]), ("integrate", 0, 0), ("integrate", 1, 0),
        ("total_weight",), ("deintegrate", 0, 0), ("total_weight",), ("gc",),
        ("integrate", 2, 1), ("deintegrate", 2, 1), ("gc",), ("total_weight",)]))
    out.append(("wrong_pose_restores", cfg, frames, poses, [
        ("stream", [0, 0, 0]), ("integrate", 0, 1), ("integrate", 1, 1),
        ("deintegrate", 0, 2), ("total_weight",), ("gc",)]))
    out.append(("inverse_pair_frees_all", cfg, frames, poses, [
        ("stream", [0, 0, 0]), ("integrate", 1, 1), ("deintegrate", 1, 1),
        ("total_weight",), ("gc",)]))
    out.append(("host_tier_rejected", cfg, frames, poses, [
        ("stream", [0, 0, 0]), ("integrate", 0, 1), ("stream", [100.0, 0, 0]),
        ("deintegrate", 0, 1), ("stream", [0, 0, 0]), ("gc",)]))
    small = dict(voxel_size=0.01, mu=0.08, stream_radius=1.2)
    out.append(("contract_partial_alloc", small, frames, poses, [
        ("stream", [-1.0, 0.0, 1.5]), ("integrate", 0, 1), ("stream", [-0.6, 0.0, 1.0]),
        ("integrate", 1, 1), ("stream", [-0.8, -0.3, 1.2]), ("integrate", 2, 1),
        ("gc",), ("total_weight",)]))
    out.append(("no_stream_rejected", cfg, frames, poses, [
        ("integrate", 0, 1)]))
    # streaming bookkeeping with relocations and re-entry
    out.append(("stream_walk", dict(voxel_size=0.01, mu=0.06, stream_radius=2.6),
                frames, poses, [
        ("stream", [0, 0, 0]), ("integrate", 0, 1), ("integrate", 1, 0),
        ("stream", [0.05, 0, 0]), ("stream", [0.5, 0, 0]), ("stream", [1.2, 0.3, 0]),
        ("stream", [2.5, 0, 0]), ("stream", [4.0, 0.0, 1.0]), ("stream", [0, 0, 0]),
        ("integrate", 2, 1), ("stream", [0.0, 0.0, 1.5]), ("deintegrate", 1, 0),
        ("gc",), ("total_weight",)]))
    # window corrections (reintegration.py:156-181)
    wf = [random_frame(rng) for _ in range(4)]
    xp = [SPose(np.eye(3), [0.05 * i, 0.0, 0.0]) for i in range(4)]
    newp = [SPose(rot_z(0.01 * i), [0.05 * i + 0.03, 0.01, 0.0]) for i in range(4)]
    bad = [SPose(np.eye(3), [2.5, 0, 0]), SPose(np.eye(3), [2.6, 0, 0])]
    wposes = xp + newp + bad
    ops = [("stream", [0, 0, 0])]
    for i in range(4):
        ops += [("stream", xp[i].translation.tolist()), ("integrate", i, i)]
    ops += [("correct", [(0, 0, 4), (1, 1, 5), (2, 2, 6)], [0.5, 0.0, 0.0]),
            ("total_weight",),
            ("correct", [(3, 3, 7)], None), ("total_weight",),
            # abort: entry with a pose it was never integrated at
            ("correct", [(0, 4, 0), (1, 8, 9)], None), ("total_weight",)]
    out.append(("window_corrections", cfg, wf, wposes, ops))
    return out


def digest_export(keys, d, w, c):
    """sha256 over sorted keys and the matching D/W/C bytes."""
    keys = np.asarray(keys, dtype=np.int64)
    order = np.argsort(keys, kind="stable")
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(keys[order]).tobytes())
    h.update(np.ascontiguousarray(np.asarray(d)[order], dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(np.asarray(w)[order], dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(np.asarray(c)[order], dtype=np.float64).tobytes())
    return h.hexdigest()


def digest_block(d, w, c):
    h = hashlib.sha256()
    for a in (d, w, c):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def run_script(adapter, cfg, frames, poses, ops):
    """Replay an op script through an adapter; returns a JSON-able log with,
    per op, its result (or the error class name), the streaming counters and
    a digest of the full volume state after the op."""
    store = adapter.make_store(cfg)
    log = []
    for op in ops:
        kind = op[0]
        rec = {"op": kind}
        try:
            if kind == "stream":
                rec["result"] = adapter.stream(store, np.asarray(op[1], dtype=np.float64))
            elif kind == "integrate":
                new, touched, updated = adapter.integrate(store, frames[op[1]], poses[op[2]])
                rec["result"] = {"new": sorted(int(k) for k in new),
                                 "blocks_touched": int(touched),
                                 "voxels_updated": int(updated)}
            elif kind == "deintegrate":
                adapter.deintegrate(store, frames[op[1]], poses[op[2]])
                rec["result"] = None
            elif kind == "gc":
                rec["result"] = int(adapter.gc(store))
            elif kind == "total_weight":
                rec["result"] = float(adapter.total_weight(store))
            elif kind == "correct":
                entries = [Entry(frames[k], poses[o].copy(), poses[n].copy())
                           for k, o, n in op[1]]
                nxt = None if op[2] is None else np.asarray(op[2], dtype=np.float64)
                rec["result"] = int(adapter.correct(store, entries, nxt))
            else:
                raise ValueError(kind)
        except Exception as exc:  # noqa: BLE001 -- error class is the result
            name = type(exc).__name__
            if name not in ("StreamingContractError", "VolumeInconsistencyError"):
                raise
            rec["error"] = name
        keys, d, w, c = adapter.export(store)
        rec["n_blocks"] = int(len(keys))
        rec["digest"] = digest_export(keys, d, w, c)
        rec["counters"] = [int(x) for x in adapter.counters(store)]
        log.append(rec)
    return log


# ---------------------------------------------------------------------------
# marching cubes (meshing.py:112-245)


def mesh_volume(seed=5, voxel=0.01):
    """A deterministic block set around two spheres: D = signed distance,
    W > 0 except a few seeded holes (unobserved corners), C a smooth colour
    ramp; some blocks of the shell are left out (absent +axis neighbours),
    coordinates straddle zero, and exact zeros / equal corner pairs occur
    (t = 0 and the midpoint rule).  Returns (keys, data[n][5][512], host_mask)
    with host_mask marking blocks the reference keeps in its host tier."""
    rng = np.random.default_rng(seed)
    span = 8 * voxel
    centres = [np.array([0.013, -0.021, 0.047]), np.array([-0.09, 0.05, 0.0])]
    radii = [0.075, 0.045]
    coords = set()
    for c, r in zip(centres, radii):
        lo = np.floor((c - r - 2 * voxel) / span).astype(int)
        hi = np.floor((c + r + 2 * voxel) / span).astype(int)
        for bx in range(lo[0], hi[0] + 1):
            for by in range(lo[1], hi[1] + 1):
                for bz in range(lo[2], hi[2] + 1):
                    coords.add((bx, by, bz))
    coords = sorted(coords)
    drop = rng.random(len(coords)) < 0.08
    coords = [c for c, d in zip(coords, drop) if not d]
    l = np.arange(512)
    lx, ly, lz = l & 7, (l >> 3) & 7, l >> 6
    keys, data = [], []
    for (bx, by, bz) in coords:
        p = np.stack([(bx * 8 + lx + 0.5) * voxel, (by * 8 + ly + 0.5) * voxel,
                      (bz * 8 + lz + 0.5) * voxel], axis=1)
        d = np.min([np.linalg.norm(p - c, axis=1) - r for c, r in zip(centres, radii)], axis=0)
        d = np.round(d / voxel * 64) / 64 * voxel   # quantised: exact zeros, equal pairs
        w = 1.0 + (l % 5) * 0.25
        w[rng.random(512) < 0.02] = 0.0
        col = np.stack([200 * p[:, 0] + 100, 150 + 0 * p[:, 1] - 300 * p[:, 1], 90 + 400 * p[:, 2]],
                       axis=0)
        blk = np.concatenate([d[None], w[None], col], axis=0)
        keys.append(((bx + (1 << 20)) << 42) | ((by + (1 << 20)) << 21) | (bz + (1 << 20)))
        data.append(blk)
    keys = np.array(keys, dtype=np.int64)
    host = rng.random(len(keys)) < 0.3
    return keys, np.array(data), host
