"""Multi-process (world_size 2, gloo, CPU) check of the hash-sharding
protocol the B200 kernels implement:

* ownership owner(key) = splitmix64(key) mod G -- the Python restatement
  here must equal the C ABI's rf_key_owner;
* the streaming contract is evaluated over the WHOLE footprint on every
  shard (the first violating key in sorted order is global);
* a de-integration's failing key is the MIN over shards (one all_reduce
  per de-integration), and blocks below it are removed + re-added.

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
    """The oracle volume restricted to one shard's blocks."""

    def __init__(self, O, vs, mu, radius, rank, shards):
        self.O = O
        self.st = O.OracleStore(vs, mu, radius)
        self.rank, self.G = rank, shards

    def mine(self, coord):
        return owner(int(self.O.pack_coords(*coord)), self.G) == self.rank

    def _allocate(self, coords):
        st = self.st
        if coords and st.last_center is None:
            raise self.O.StreamingContractError("no sphere")
        first_bad = next((c for c in coords if st._center_distance(c) > st.stream_radius), None)
        for c in coords:
            if c == first_bad:
                raise self.O.StreamingContractError(str(c))
            if self.mine(c) and c not in st.active:
                st.active[c] = self.O.Block()

    def integrate(self, kf, pose):
        coords = self.st.footprint(kf, pose)
        self._allocate(coords)
        for c in coords:
            if self.mine(c):
                self.st._fuse(self.st.active[c], c, kf, pose, False)

    def deintegrate(self, kf, pose):
        coords = self.st.footprint(kf, pose)
        self._allocate(coords)
        mine = [c for c in coords if self.mine(c)]
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


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import scenarios as S

    rng = np.random.default_rng(17)
    frames = [S.random_frame(rng) for _ in range(3)]
    pose = S.SPose(S.rot_y(0.2), [0.1, -0.05, 0.02])
    wrong = S.SPose(np.eye(3), [1.0, 0.0, 0.0])
    events = []
    m = ShardModel(O, 0.01, 0.06, 4.0, rank, world)
    m.st.stream(pose.translation)
    for f in frames:
        m.integrate(f, pose)
    m.deintegrate(frames[0], pose)
    try:
        m.deintegrate(frames[1], wrong)
    except O.VolumeInconsistencyError:
        events.append("inconsistent")
    m.st.garbage_collect()
    parts = [None] * world
    dist.all_gather_object(parts, (m.st.export(), events))
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
        ref.garbage_collect()
        want = ref.export()
        keys = np.concatenate([p[0][0] for p in parts])
        order = np.argsort(keys)
        ok = np.array_equal(keys[order], want[0])
        for i in (1, 2, 3):
            got = np.concatenate([p[0][i] for p in parts])[order]
            ok = ok and np.array_equal(got, want[i])
        ok = ok and all(p[1] == ref_events for p in parts)
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
