"""Pin the CPU oracle (oracle/) to the reference's golden vectors.

The vectors in tests/golden/volume_golden.json were produced by running the
reference package itself (tests/golden/gen_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

import oracle as O
import scenarios as S
from adapters import OracleAdapter

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "volume_golden.json")))


def test_block_hash_golden():
    for coord, buckets, want in GOLDEN["hash"]:
        assert O.block_hash(coord, buckets) == want, (coord, buckets)


def test_block_hash_reference_fixed_points():
    # reference tests/test_volume.py:57-81 and SURVEY §8c extra vectors
    assert O.block_hash((0, 0, 0), 65536) == 0
    assert O.block_hash((3, -7, 11), 4096) == 2743
    assert O.block_hash((-1, -2, -3), 65536) == 30158
    assert O.block_hash((100, -200, 300), 65536) == 41272
    assert O.block_hash((-12345, 0, 999), 65536) == 50282
    assert O.block_hash((1, 1, 1), 1 << 22) == 3689295


def test_fuse_block_golden():
    cases = S.fuse_block_cases()
    assert len(cases) == len(GOLDEN["fuse_block"])
    fails = 0
    for (state, scene, remove), want in zip(cases, GOLDEN["fuse_block"]):
        d, w, c = (a.copy() for a in state)
        origin, vs, rot, cam, intr, depth, weight, color = scene
        fx, fy, cx, cy, width, height = intr
        args = (origin[0], origin[1], origin[2], vs, rot, cam[0], cam[1], cam[2],
                fx, fy, cx, cy, width, height, depth, weight, color, 0.06, 1e-9)
        if remove == "roundtrip":
            assert O.fuse_block(d, w, c, *args, False) == want["n_add"]
            n = O.fuse_block(d, w, c, *args, True)
            assert not w.any()
        else:
            n = O.fuse_block(d, w, c, *args, bool(remove))
            if n == -1:
                fails += 1
                assert S.digest_block(d, w, c) == S.digest_block(*state)
        assert n == want["n"]
        assert S.digest_block(d, w, c) == want["digest"]
    assert fails > 0


def test_footprint_golden():
    for (name, f, p, vs, mu), want in zip(S.footprint_cases(), GOLDEN["footprint"]):
        assert want["name"] == name
        keys = O.footprint_keys(f.depth, f.weight, f.intrinsics, p.rotation,
                                p.translation, vs, mu)
        assert keys.tolist() == want["keys"], name
        coords = O.keys_to_coords(keys)
        assert [O.block_hash(c, 65536) for c in coords] == want["hash_65536"]


@pytest.mark.parametrize("idx", range(len(S.volume_scripts())))
def test_volume_script_golden(idx):
    name, cfg, frames, poses, ops = S.volume_scripts()[idx]
    want = GOLDEN["scripts"][idx]
    assert want["name"] == name
    got = S.run_script(OracleAdapter(), cfg, frames, poses, ops)
    assert len(got) == len(want["log"])
    for g, w in zip(got, want["log"]):
        assert g == w, (name, g["op"])
