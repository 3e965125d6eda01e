"""Multi-process (world_size 2, gloo, CPU) check of the hash-sharding
protocol the B200 kernels implement:

* ownership owner(key) = splitmix64(key) mod G -- the Python restatement
  here must equal the C ABI's rf_key_owner;
* the streaming contract is evaluated over the WHOLE footprint on every
  shard (the first violating key in sorted order is global);
* a de-integration's failing key is the MIN over shards (one all_reduce
  per de-integration), and blocks below it are removed + re-added -- what
  k_shard_sync does on the device (every shard's check publishes its first
  failing key into every shard's verdict slot with a system-scope atomicMin
  over NVLink, each shard applies the global minimum; k_fuse<kRemoveReadd>
  removes + re-adds the blocks below it);
* a correction window whose removal fails re-integrates the entries it
  already removed (reintegration.py:156-181) on every shard -- the device's
  rf_correct_windows recovery.

* routed footprints (k_route / rf_route): each rank samples only the pixel
  tiles t with t mod G == rank, keys go to their owners (all-to-all) and
  the minimum violating key to every rank -- the same volume, including
  the partial allocation a contract error leaves behind.

Each rank runs the CPU oracle restricted to its own blocks; the union of
the ranks' volumes must equal the unsharded oracle bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

MASK64 = (1 << 64) - 1


def owner(key, shards):
    z = (int(key) + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z % shards


def test_owner_matches_c_abi():
    from paper_1709_03763_b200 import _lib

    lib = _lib.load_library()
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 62, 2000)
    for g in (2, 3, 8):
        for k in keys[:500]:
            assert lib.rf_key_owner(int(k), g) == owner(k, g)
        counts = np.bincount([owner(k, g) for k in keys], minlength=g)
        assert counts.min() > 0.6 * len(keys) / g  # balanced


class ShardModel:
    """The oracle volume restricted to one shard's blocks.  routed: the
    footprint is built as k_route builds it -- this rank samples only the
    16x16 pixel tiles t with t mod G == rank, sends every key to its owner
    (all-to-all) and the minimum violating key to everyone (all_reduce)."""

    def __init__(self, O, vs, mu, radius, rank, shards, routed=False):
        self.O = O
        self.st = O.OracleStore(vs, mu, radius)
        self.rank, self.G = rank, shards
        self.routed = routed

    def mine(self, coord):
        return owner(int(self.O.pack_coords(*coord)), self.G) == self.rank

    def _routed_footprint(self, kf, pose):
        import torch

        O, st = self.O, self.st
        intr = kf.intrinsics
        tiles_x = -(-intr.width // 16)
        v, u = np.mgrid[0:intr.height, 0:intr.width]
        tile = (v // 16) * tiles_x + (u // 16)
        w = np.where(tile % self.G == self.rank, kf.weight, 0.0)  # my pixels only
        keys = O.footprint_keys(kf.depth, w, intr, pose.rotation, pose.translation,
                                st.voxel_size, st.mu)
        big = (1 << 63) - 1
        bad = [int(k) for k in keys
               if st.last_center is None or st._center_distance(O.keys_to_coords([k])[0])
               > st.stream_radius]
        out = [[int(k) for k in keys if owner(k, self.G) == o] for o in range(self.G)]
        inbox = [None] * self.G
        gathered = [None] * self.G  # the all-to-all, as an all-gather on gloo
        dist.all_gather_object(gathered, out)
        for src in range(self.G):
            inbox[src] = gathered[src][self.rank]
        t = torch.tensor([min(bad) if bad else big], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        mine = sorted(set(k for seg in inbox for k in seg))
        return O.keys_to_coords(np.array(mine, dtype=np.int64)), int(t.item())

    def _footprint(self, kf, pose):
        """(this shard's coords in sorted order, first violating key or None)"""
        if self.routed:
            coords, bad = self._routed_footprint(kf, pose)
            return coords, (None if bad == (1 << 63) - 1 else bad)
        coords = self.st.footprint(kf, pose)
        st = self.st
        if coords and st.last_center is None:
            raise self.O.StreamingContractError("no sphere")
        first_bad = next((c for c in coords if st._center_distance(c) > st.stream_radius), None)
        bad = None if first_bad is None else int(self.O.pack_coords(*first_bad))
        return [c for c in coords if self.mine(c)], bad

    def _allocate_mine(self, mine, bad):
        for c in mine:
            if bad is not None and int(self.O.pack_coords(*c)) >= bad:
                break
            if c not in self.st.active:
                self.st.active[c] = self.O.Block()
        if bad is not None:
            raise self.O.StreamingContractError(str(bad))

    def integrate(self, kf, pose):
        mine, bad = self._footprint(kf, pose)
        self._allocate_mine(mine, bad)
        for c in mine:
            self.st._fuse(self.st.active[c], c, kf, pose, False)

    def deintegrate(self, kf, pose):
        mine, bad = self._footprint(kf, pose)
        self._allocate_mine(mine, bad)
        local_fail = None
        for c in mine:  # check phase, sorted order
            trial = self.st.active[c].copy()
            if self.st._fuse(trial, c, kf, pose, True) < 0:
                local_fail = c
                break
        big = (1 << 63) - 1
        key = np.array([big if local_fail is None else int(self.O.pack_coords(*local_fail))])
        import torch

        t = torch.from_numpy(key)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        fail = int(t.item())
        for c in mine:
            if int(self.O.pack_coords(*c)) >= fail:
                break
            self.st._fuse(self.st.active[c], c, kf, pose, True)
            if fail != big:
                self.st._fuse(self.st.active[c], c, kf, pose, False)
        if fail != big:
            raise self.O.VolumeInconsistencyError("negative weight")

    def correct_entries(self, entries):
        """reintegration._correct_entries' removal half with its rollback
        (reintegration.py:156-174), every removal's verdict global."""
        removed = []
        try:
            for kf, old in entries:
                self.deintegrate(kf, old)
                removed.append((kf, old))
        except self.O.VolumeInconsistencyError:
            for kf, old in removed:
                self.integrate(kf, old)
            raise


def _ref_correct_entries(O, ref, entries):
    removed = []
    try:
        for kf, old in entries:
            ref.deintegrate(kf, old)
            removed.append((kf, old))
    except O.VolumeInconsistencyError:
        for kf, old in removed:
            ref.integrate(kf, old)
        raise


def _worker(rank, world, port, result_path, routed=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import scenarios as S

    rng = np.random.default_rng(17)
    frames = [S.random_frame(rng) for _ in range(3)]
    pose = S.SPose(S.rot_y(0.2), [0.1, -0.05, 0.02])
    wrong = S.SPose(np.eye(3), [1.0, 0.0, 0.0])
    events = []
    m = ShardModel(O, 0.01, 0.06, 4.0, rank, world, routed)
    m.st.stream(pose.translation)
    for f in frames:
        m.integrate(f, pose)
    m.deintegrate(frames[0], pose)
    try:
        m.deintegrate(frames[1], wrong)
    except O.VolumeInconsistencyError:
        events.append("inconsistent")
    m.integrate(frames[0], pose)
    try:  # entry 1 fails: entry 0's removal is rolled back on every rank
        m.correct_entries([(frames[0], pose), (frames[1], wrong), (frames[2], pose)])
    except O.VolumeInconsistencyError:
        events.append("window")
    far = np.asarray(pose.translation) + np.array([-2.4, 0.0, 0.0])
    moved = S.SPose(S.rot_y(0.5), np.asarray(pose.translation) + np.array([0.3, 0.0, 0.0]))
    m.st.stream(far)
    try:  # part of the footprint lies outside the sphere: partial allocation
        m.integrate(frames[2], moved)
    except O.StreamingContractError:
        events.append("contract")
    partial = m.st.export()
    m.st.garbage_collect()
    parts = [None] * world
    dist.all_gather_object(parts, (m.st.export(), events, partial))
    if rank == 0:
        ref = O.OracleStore(0.01, 0.06, 4.0)
        ref.stream(pose.translation)
        for f in frames:
            ref.integrate(f, pose)
        ref.deintegrate(frames[0], pose)
        ref_events = []
        try:
            ref.deintegrate(frames[1], wrong)
        except O.VolumeInconsistencyError:
            ref_events.append("inconsistent")
        ref.integrate(frames[0], pose)
        try:
            _ref_correct_entries(O, ref, [(frames[0], pose), (frames[1], wrong), (frames[2], pose)])
        except O.VolumeInconsistencyError:
            ref_events.append("window")
        ref.stream(far)
        n_alloc = len(ref.active)
        try:
            ref.integrate(frames[2], moved)
        except O.StreamingContractError:
            ref_events.append("contract")
        ok_partial = len(ref.active) > n_alloc  # the case allocates before it raises
        want_partial = ref.export()
        ref.garbage_collect()
        want = ref.export()
        keys = np.concatenate([p[0][0] for p in parts])
        order = np.argsort(keys)
        ok = np.array_equal(keys[order], want[0])
        for i in (1, 2, 3):
            got = np.concatenate([p[0][i] for p in parts])[order]
            ok = ok and np.array_equal(got, want[i])
        ok = ok and all(p[1] == ref_events for p in parts)
        ok = ok and ref_events == ["inconsistent", "window", "contract"] and ok_partial
        pk = np.concatenate([p[2][0] for p in parts])
        po = np.argsort(pk)
        ok = ok and np.array_equal(pk[po], want_partial[0])
        for i in (1, 2, 3):
            ok = ok and np.array_equal(np.concatenate([p[2][i] for p in parts])[po],
                                       want_partial[i])
        with open(result_path, "w") as fh:
            fh.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_sharded_oracle_equals_unsharded(tmp_path):
    out = tmp_path / "result.txt"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"


def test_two_rank_gloo_routed_footprints_equal_unsharded(tmp_path):
    """k_route's protocol: each rank samples half of the pixel tiles, keys go
    to their owners, the violating key is reduced -- same volume."""
    out = tmp_path / "result.txt"
    mp.spawn(_worker, args=(2, _free_port(), str(out), True), nprocs=2, join=True)
    assert out.read_text() == "ok"
