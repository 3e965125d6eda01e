"""Parity of the CUDA volume path (through the C ABI) with the reference.

* golden vectors produced by the reference itself (tests/golden/), bit-exact;
* the CPU oracle (pinned to those vectors) at larger sizes, bit-exact;
* size-independent properties at full 640x480 keyframes.
"""

import json
import os

import numpy as np
import pytest

import oracle as O
import scenarios as S
from adapters import ProductAdapter, logs_match

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "volume_golden.json")))


@pytest.fixture(scope="module")
def V():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import volume

    return volume


def assert_same_state(store, ref):
    got, want = store.export(), ref.export()
    assert np.array_equal(got[0], want[0]), (
        f"block sets differ: {len(got[0])} vs {len(want[0])}, "
        f"{len(set(got[0].tolist()) ^ set(want[0].tolist()))} in symmetric difference")
    for name, a, b in zip("dwc", got[1:], want[1:]):
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{name} differs at {len(bad)} entries, first {bad[:3]}")


# ---------------------------------------------------------------------------
# the plugin point: kernels.fuse_block (_kernels_cy.pyx:14-108)


def test_fuse_block_golden_bitexact():
    from paper_1709_03763_b200 import kernels as K

    assert K.BACKEND == "b200"
    cases = S.fuse_block_cases()
    fails = 0
    for (state, scene, remove), want in zip(cases, GOLDEN["fuse_block"]):
        d, w, c = (a.copy() for a in state)
        origin, vs, rot, cam, intr, depth, weight, color = scene
        fx, fy, cx, cy, width, height = intr
        args = (origin[0], origin[1], origin[2], vs, rot, cam[0], cam[1], cam[2],
                fx, fy, cx, cy, width, height, depth, weight, color, 0.06, 1e-9)
        if remove == "roundtrip":
            assert K.fuse_block(d, w, c, *args, False) == want["n_add"]
            n = K.fuse_block(d, w, c, *args, True)
            assert not w.any()
        else:
            n = K.fuse_block(d, w, c, *args, bool(remove))
            if n == -1:
                fails += 1
                assert S.digest_block(d, w, c) == S.digest_block(*state)
        assert n == want["n"]
        assert S.digest_block(d, w, c) == want["digest"]
    assert fails > 0


def test_fuse_block_random_vs_oracle():
    from paper_1709_03763_b200 import kernels as K

    rng = np.random.default_rng(909)
    for trial in range(60):
        mode = ("sparse", "full", "empty")[trial % 3]
        state, scene = S.fuse_block_case(rng, mode)
        origin, vs, rot, cam, intr, depth, weight, color = scene
        fx, fy, cx, cy, width, height = intr
        col = None if trial % 5 == 0 else color
        args = (origin[0], origin[1], origin[2], vs, rot, cam[0], cam[1], cam[2],
                fx, fy, cx, cy, width, height, depth, weight, col, 0.06, 1e-9)
        for remove in (False, True):
            a = [x.copy() for x in state]
            b = [x.copy() for x in state]
            assert K.fuse_block(*a, *args, remove) == O.fuse_block(*b, *args, remove)
            for x, y in zip(a, b):
                assert np.array_equal(x, y)


# ---------------------------------------------------------------------------
# footprint + allocation


def test_footprint_golden(V):
    for (name, f, p, vs, mu), want in zip(S.footprint_cases(), GOLDEN["footprint"]):
        cfg = V.VolumeConfig(voxel_size=vs, mu=mu, stream_radius=1e6)
        coords = V.keyframe_block_footprint(f, p, cfg)
        keys = V.pack_keys(coords).tolist() if coords else []
        assert keys == want["keys"], name
        assert [V.block_hash(c, 65536) for c in coords] == want["hash_65536"]


@pytest.mark.parametrize("idx", range(len(S.volume_scripts())))
def test_volume_script_golden(V, idx):
    name, cfg, frames, poses, ops = S.volume_scripts()[idx]
    want = GOLDEN["scripts"][idx]
    got = S.run_script(ProductAdapter(), cfg, frames, poses, ops)
    ok, why = logs_match(got, want["log"])
    assert ok, f"{name}: {why}"


def test_allocate_single_ray_band(V):
    # reference tests/test_volume.py:103-116
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.08, stream_radius=4.0)
    store = V.TwoTierStore(block_capacity=64)
    V.stream(store, np.zeros(3), cfg)
    new = V.allocate_blocks(store, S.single_ray_frame(2.0), S.identity(), cfg)
    assert {(0, 0, 24), (0, 0, 25)} <= new <= {(0, 0, k) for k in (23, 24, 25, 26)}
    assert V.allocate_blocks(store, S.single_ray_frame(2.0), S.identity(), cfg) == set()
    assert store.block_count() == len(new)


def test_allocate_requires_stream(V):
    from paper_1709_03763_b200.errors import StreamingContractError

    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.08, stream_radius=4.0)
    store = V.TwoTierStore(block_capacity=64)
    with pytest.raises(StreamingContractError):
        V.allocate_blocks(store, S.single_ray_frame(2.0), S.identity(), cfg)
    assert store.block_count() == 0
    # an empty footprint never needs the sphere
    empty = S.Frame(np.zeros((5, 5)), np.zeros((5, 5)), None, S.TINY_INTR)
    assert V.allocate_blocks(store, empty, S.identity(), cfg) == set()


def test_first_sample_running_average(V):
    # reference tests/test_volume.py:169-196 (hand-computed golden values)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.08, stream_radius=4.0)

    def gray(depth_m, g):
        f = S.single_ray_frame(depth_m)
        f.color = np.full((5, 5, 3), g)
        return f

    store = V.TwoTierStore(block_capacity=64)
    V.stream(store, np.zeros(3), cfg)
    V.integrate(store, gray(2.005, 0.5), S.identity(), cfg)
    lin = 64 * 7
    blk = store.find((0, 0, 24))
    assert blk.w[lin] == 1.0
    assert abs(blk.d[lin] - 0.01) < 1e-12
    assert np.all(np.abs(blk.c[lin] - 0.5) < 1e-12)
    V.integrate(store, gray(2.025, 0.9), S.identity(), cfg)
    blk = store.find((0, 0, 24))
    assert blk.w[lin] == 2.0
    assert abs(blk.d[lin] - 0.02) < 1e-12
    assert np.all(np.abs(blk.c[lin] - 0.7) < 1e-12)


def test_capacity_exhaustion_raises(V):
    from paper_1709_03763_b200.errors import CapacityError

    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    store = V.TwoTierStore(block_capacity=16)
    V.stream(store, np.zeros(3), cfg)
    with pytest.raises(CapacityError):
        V.integrate(store, S.random_frame(np.random.default_rng(3)), S.identity(), cfg)


# ---------------------------------------------------------------------------
# larger parity vs the oracle


def _vga_frame(rng, z=1.4, tilt=0.25, holes=0.05, color=True):
    f = S.wall_frame(S.VGA_INTR, z, rng=rng, tilt=tilt, noise=0.0015, holes=holes)
    if not color:
        f.color = None
    return f


@pytest.mark.parametrize("vs", [0.01, 0.005])
def test_vga_integrate_deintegrate_bitexact(V, vs):
    rng = np.random.default_rng(int(vs * 1e4))
    cfg = V.VolumeConfig(voxel_size=vs, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    poses = [S.SPose(S.rot_z(0.3) @ S.rot_y(0.1), [0.2, 0.1, 0.3]),
             S.SPose(S.rot_z(0.31) @ S.rot_y(0.12), [0.21, 0.08, 0.31])]
    frames = [_vga_frame(rng), _vga_frame(rng, z=1.6, tilt=-0.2, color=False)]
    store = V.TwoTierStore(block_capacity=1 << 15)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    for s in (store,):
        V.stream(s, poses[0].translation, cfg)
    ref.stream(poses[0].translation)
    for f, p in zip(frames, poses):
        rec = V.integrate(store, f, p, cfg)
        new, touched, updated = ref.integrate(f, p)
        assert rec.new_blocks == new
        assert (rec.blocks_touched, rec.voxels_updated) == (touched, updated)
    assert_same_state(store, ref)
    V.deintegrate(store, frames[0], poses[0], cfg)
    ref.deintegrate(frames[0], poses[0])
    assert_same_state(store, ref)
    assert V.garbage_collect(store) == ref.garbage_collect()
    assert_same_state(store, ref)


def test_vga_window_correction_bitexact(V):
    rng = np.random.default_rng(77)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=6.0)
    frames = [_vga_frame(rng, z=1.2 + 0.1 * i, tilt=0.1 * i) for i in range(4)]
    old = [S.SPose(S.rot_z(0.05 * i), [0.03 * i, 0.0, 0.1]) for i in range(4)]
    new = [S.SPose(S.rot_z(0.05 * i + 0.01), [0.03 * i + 0.02, 0.01, 0.1]) for i in range(4)]
    store = V.TwoTierStore(block_capacity=1 << 15)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    for f, p in zip(frames, old):
        V.stream(store, p.translation, cfg)
        V.integrate(store, f, p, cfg)
        ref.stream(p.translation)
        ref.integrate(f, p)
    ents = [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)]
    rents = [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)]
    assert V.correct_entries(store, ents, cfg, np.array([0.5, 0.0, 0.0])) == 4
    ref.correct_entries(rents)
    ref.stream(np.array([0.5, 0.0, 0.0]))
    assert_same_state(store, ref)
    c = store.counters()
    assert (c.blocks_streamed_in, c.blocks_streamed_out, c.sphere_relocations) == (
        ref.blocks_streamed_in, ref.blocks_streamed_out, ref.sphere_relocations)
    for e in ents:
        assert np.array_equal(e.integrated_pose.translation, e.target_pose.translation)


def test_determinism_same_window_twice(V):
    rng = np.random.default_rng(5)
    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0)
    frames = [_vga_frame(rng, z=1.3 + 0.05 * i) for i in range(3)]
    poses = [S.SPose(S.rot_y(0.02 * i), [0.02 * i, 0.0, 0.0]) for i in range(3)]
    outs = []
    for _ in range(2):
        store = V.TwoTierStore(block_capacity=1 << 16)
        V.stream(store, np.zeros(3), cfg)
        for f, p in zip(frames, poses):
            V.integrate(store, f, p, cfg)
        outs.append(store.export())
        store.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_save_load_roundtrip(V, tmp_path):
    rng = np.random.default_rng(67)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    pose = S.SPose(S.rot_y(0.15), [0.05, 0.0, 0.1])
    store = V.TwoTierStore(block_capacity=1 << 12)
    V.stream(store, pose.translation, cfg)
    V.integrate(store, S.random_frame(rng), pose, cfg)
    V.integrate(store, S.random_frame(rng), pose, cfg)
    V.stream(store, pose.translation + np.array([1.5, 0.0, 0.0]), cfg)
    path = os.fspath(tmp_path / "snap.sdf")
    V.save_volume(store, path, cfg)
    loaded, vs, mu = V.load_volume(path)
    assert (vs, mu) == (cfg.voxel_size, cfg.mu)
    assert loaded.block_count() == store.block_count()
    assert V.compare_volumes(store, loaded) == (0.0, 0.0, 0.0)
    V.stream(loaded, np.zeros(3), cfg)  # binds and uploads
    assert V.compare_volumes(store, loaded) == (0.0, 0.0, 0.0)


def test_snapshot_bytes_match_reference(V, tmp_path):
    """save_volume streams SDFV1 records formatted on the device: the file is
    byte-identical to the reference's save_volume of the same blocks, and the
    reference's file loads back bit for bit (volume.py:397-442)."""
    from refimport import reference

    ref = reference()
    if ref is None:
        pytest.skip("reference build (oracle/_ref) absent")
    RV = ref["V"]
    rng = np.random.default_rng(71)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=4.0)
    pose = S.SPose(S.rot_y(0.15), [0.05, 0.0, 0.1])
    store = V.TwoTierStore(block_capacity=1 << 12)
    V.stream(store, pose.translation, cfg)
    for _ in range(2):
        V.integrate(store, S.random_frame(rng), pose, cfg)
    old_chunk = V._SNAP_CHUNK
    V._SNAP_CHUNK = 7  # several chunks
    try:
        ours = tmp_path / "ours.sdf"
        V.save_volume(store, os.fspath(ours), cfg)
    finally:
        V._SNAP_CHUNK = old_chunk
    keys, d, w, c = store.export()
    rs = RV.TwoTierStore()
    for k, dd, ww, cc in zip(keys, d, w, c):
        coord = tuple(int(x) for x in V.unpack_keys(np.array([k]))[0])
        rs.active[coord] = RV.VoxelBlock(coord, dd.copy(), ww.copy(), cc.copy())
    theirs = tmp_path / "ref.sdf"
    RV.save_volume(rs, os.fspath(theirs), RV.VolumeConfig(voxel_size=cfg.voxel_size, mu=cfg.mu))
    assert ours.read_bytes() == theirs.read_bytes()
    loaded, vs, mu = V.load_volume(os.fspath(theirs))
    V.stream(loaded, np.zeros(3), cfg)
    for a, b in zip(loaded.export(), store.export()):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("exp_span", [8, 60, 600])
def test_shared_denominator_division_is_ieee(exp_span):
    """The kernels divide by Markstein correction with a shared reciprocal;
    it must reproduce IEEE division bit for bit (reference: plain C '/')."""
    import ctypes

    from paper_1709_03763_b200 import _lib as L

    bad = ctypes.c_uint64()
    assert L.lib().rf_selftest_division(1 << 27, 1234 + exp_span, exp_span,
                                        ctypes.byref(bad)) == 0
    assert bad.value == 0


@pytest.mark.parametrize("shape", [(640, 480, 319.5, 239.5), (1920, 1080, 959.25, 540.75),
                                   (64, 48, 31.5, 23.5)])
def test_screened_projection_is_exact(shape):
    """The integrate kernels pick each voxel's pixel with an approximate
    reciprocal and fall back to IEEE division within 2^-24 of a pixel
    boundary; the pixel / in-image decision must equal the exact one."""
    import ctypes

    from paper_1709_03763_b200 import _lib as L

    w, h, cx, cy = shape
    bad = ctypes.c_uint64()
    assert L.lib().rf_selftest_projection(w, h, cx, cy, 1 << 26, 77, ctypes.byref(bad)) == 0
    assert bad.value == 0


def test_extreme_values_take_the_exact_tail(V):
    """Voxels whose update operands leave the fast paths' exponent range
    (here colours ~1e305 / 1e-310 written into blocks) are re-fused by the
    kernels' exact IEEE tail: results stay bit-identical to the oracle for
    integration, the removal check and the removal."""
    rng = np.random.default_rng(5)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    pose = S.SPose(S.rot_z(0.2) @ S.rot_y(0.05), [0.1, 0.05, 0.2])
    f0, f1 = _vga_frame(rng), _vga_frame(rng, z=1.55, tilt=0.05)
    store = V.TwoTierStore(block_capacity=1 << 15)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    V.stream(store, pose.translation, cfg)
    ref.stream(pose.translation)
    V.integrate(store, f0, pose, cfg)
    ref.integrate(f0, pose)
    keys, d, w, c = ref.export()
    coords = O.keys_to_coords(keys)
    pick = rng.choice(len(coords), size=min(40, len(coords)), replace=False)
    for j in pick:
        b = ref.find(coords[j])
        vox = rng.choice(512, size=64, replace=False)
        b.c[vox[:32], 0] = 1e305
        b.c[vox[32:], 2] = 1e-310
        store.put_block(coords[j], b.d.copy(), b.w.copy(), b.c.copy())
    assert_same_state(store, ref)
    rec = V.integrate(store, f1, pose, cfg)
    _, touched, updated = ref.integrate(f1, pose)
    assert (rec.blocks_touched, rec.voxels_updated) == (touched, updated)
    assert_same_state(store, ref)
    V.deintegrate(store, f0, pose, cfg)
    ref.deintegrate(f0, pose)
    assert_same_state(store, ref)


def _contract_window_case(cfg, rng):
    """Search (with the oracle) a keyframe + (old, new) pose pair whose
    re-integration fails the streaming contract on the INTEGRATION while the
    removal succeeds: footprint blocks near the sphere's rim quantise in or
    out with the pose."""
    for _ in range(400):
        f = S.random_frame(rng, z_lo=0.92, z_hi=1.02)
        old = S.SPose(S.rot_y(rng.uniform(-0.3, 0.3)) @ S.rot_x(rng.uniform(-0.3, 0.3)),
                      rng.uniform(-0.02, 0.02, 3))
        new = S.SPose(old.rotation @ S.rot_z(rng.uniform(-0.3, 0.3)),
                      old.translation + rng.uniform(-0.03, 0.03, 3))
        ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
        try:
            ref.stream(old.translation)
            ref.integrate(f, old)
            ref.stream(old.translation)
            ref.deintegrate(f, old)
        except O.OracleError:
            continue
        try:
            ref.stream(new.translation)
            ref.integrate(f, new)
        except O.StreamingContractError:
            return f, old, new
    pytest.skip("no rim case found")


def test_window_integration_contract_error_matches_oracle(V):
    """A window whose integration violates the streaming contract after its
    removal succeeded (the pair runs as one merged removal + integration
    kernel): the removal completes, the integration keeps its sorted-prefix
    partial allocation, the error is StreamingContractError -- the state of
    the reference's sequential _correct_entries."""
    from paper_1709_03763_b200.errors import StreamingContractError

    rng = np.random.default_rng(91)
    cfg = V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=1.25, hash_buckets=1 << 14)
    f, old, new = _contract_window_case(cfg, rng)
    other = S.random_frame(rng, z_lo=0.5, z_hi=0.7)
    store = V.TwoTierStore(block_capacity=1 << 14)
    ref = O.OracleStore(cfg.voxel_size, cfg.mu, cfg.stream_radius)
    for kf, p in ((other, old), (f, old)):
        V.stream(store, p.translation, cfg)
        V.integrate(store, kf, p, cfg)
        ref.stream(p.translation)
        ref.integrate(kf, p)
    ents = [S.Entry(f, old.copy(), new.copy())]
    rents = [S.Entry(f, old.copy(), new.copy())]
    with pytest.raises(StreamingContractError):
        V.correct_entries(store, ents, cfg)
    with pytest.raises(O.StreamingContractError):
        ref.correct_entries(rents)
    assert_same_state(store, ref)


@pytest.mark.parametrize("vs", [0.01, 0.005, 0.004])
def test_footprint_far_from_origin_matches_oracle(V, vs):
    """The footprint kernel skips samples whose affine block estimate is
    provably inside the previous sample's block; far from the origin the
    block coordinates are large (~1e5 spans) and the estimate's rounding
    largest -- the key set must still be the oracle's, bit for bit."""
    rng = np.random.default_rng(int(vs * 1e4))
    cfg = V.VolumeConfig(voxel_size=vs, mu=0.06, stream_radius=1e7)
    for t in ([0.0, 0.0, 0.0], [3000.0, -1200.0, 41.0], [-2.5e3, 7.0e2, -9.0e2]):
        f = _vga_frame(rng, z=1.3, tilt=0.2)
        pose = S.SPose(S.rot_z(rng.uniform(-3, 3)) @ S.rot_y(rng.uniform(-1, 1)), t)
        got = V.pack_keys(V.keyframe_block_footprint(f, pose, cfg)).tolist()
        want = O.footprint_keys(f.depth, f.weight, f.intrinsics, pose.rotation,
                                pose.translation, vs, cfg.mu)
        assert sorted(got) == sorted(np.asarray(want).tolist())
