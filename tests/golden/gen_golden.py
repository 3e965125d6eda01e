"""Generate the golden vectors in tests/golden/ by running the REFERENCE.

Run in the build container (the reference tree exists only there):

    make -C oracle ref            # builds oracle/_ref (reference + Cython kernel)
    python tests/golden/gen_golden.py

It imports the unmodified reference package ``refusion`` from oracle/_ref
(compiled backend) -- or from /root/reference/pkg/src with the numpy
backend when the build is absent -- feeds it the seeded inputs of
tests/scenarios.py and writes what it returns.  The outputs pin the oracle
(tests/test_oracle.py) and, through it, the CUDA path.  Nothing at test time
reads /root/reference.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "tests"))

_REF_BUILD = os.path.join(REPO, "oracle", "_ref")
if os.path.isdir(os.path.join(_REF_BUILD, "refusion")):
    sys.path.insert(0, _REF_BUILD)
    os.environ.setdefault("REFUSION_BACKEND", "compiled")
else:
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ.setdefault("REFUSION_BACKEND", "python")

import scenarios as S  # noqa: E402
from refusion import kernels as RK  # noqa: E402
from refusion import reintegration as RR  # noqa: E402
from refusion import volume as RV  # noqa: E402
from refusion.geometry import Intrinsics, Pose  # noqa: E402


def ref_intr(i):
    return Intrinsics(fx=i.fx, fy=i.fy, cx=i.cx, cy=i.cy, width=i.width,
                      height=i.height)


def ref_frame(f):
    return S.Frame(f.depth, f.weight, f.color, ref_intr(f.intrinsics))


def ref_pose(p):
    return Pose(p.rotation, p.translation)


class RefAdapter:
    """Drives the reference's own volume / reintegration API."""

    def __init__(self):
        self._frames = {}

    def make_store(self, cfg):
        self.cfg = RV.VolumeConfig(**cfg)
        return RV.TwoTierStore()

    def _f(self, f):
        key = id(f)
        if key not in self._frames:
            self._frames[key] = ref_frame(f)
        return self._frames[key]

    def stream(self, store, c):
        return RV.stream(store, c, self.cfg)

    def integrate(self, store, f, p):
        rec = RV.integrate(store, self._f(f), ref_pose(p), self.cfg)
        keys = [int(RV._pack_coords(*c)) for c in rec.new_blocks]
        return keys, rec.blocks_touched, rec.voxels_updated

    def deintegrate(self, store, f, p):
        RV.deintegrate(store, self._f(f), ref_pose(p), self.cfg)

    def gc(self, store):
        return RV.garbage_collect(store)

    def total_weight(self, store):
        return RV.total_weight(store)

    def correct(self, store, entries, nxt):
        ents = [S.Entry(self._f(e.kf), ref_pose(e.integrated_pose),
                        ref_pose(e.target_pose)) for e in entries]
        n = RR._correct_entries(store, ents, self.cfg)
        if nxt is not None:
            RV.stream(store, nxt, self.cfg)
        return n

    def export(self, store):
        coords = sorted(c for c, _ in store.iter_blocks())
        keys = np.array([RV._pack_coords(*c) for c in coords], dtype=np.int64)
        n = len(coords)
        d = np.zeros((n, 512))
        w = np.zeros((n, 512))
        c = np.zeros((n, 512, 3))
        for i, coord in enumerate(coords):
            b = store.find(coord)
            d[i], w[i], c[i] = b.d, b.w, b.c
        return keys, d, w, c

    def counters(self, store):
        return (store.blocks_streamed_in, store.blocks_streamed_out,
                store.sphere_relocations)


def gen_hash():
    return [[list(c), b, RV.block_hash(c, b)] for c, b in S.hash_cases()]


def gen_fuse_block():
    out = []
    for state, scene, remove in S.fuse_block_cases():
        d, w, c = (a.copy() for a in state)
        origin, vs, rot, cam, intr, depth, weight, color = scene
        fx, fy, cx, cy, width, height = intr
        args = (origin[0], origin[1], origin[2], vs, rot, cam[0], cam[1], cam[2],
                fx, fy, cx, cy, width, height, depth, weight, color, 0.06, 1e-9)
        if remove == "roundtrip":
            n1 = RK.fuse_block(d, w, c, *args, False)
            n = RK.fuse_block(d, w, c, *args, True)
            out.append({"mode": "roundtrip", "n_add": int(n1), "n": int(n),
                        "digest": S.digest_block(d, w, c)})
        else:
            n = RK.fuse_block(d, w, c, *args, bool(remove))
            out.append({"mode": "remove" if remove else "integrate", "n": int(n),
                        "digest": S.digest_block(d, w, c)})
    return out


def gen_footprint():
    out = []
    for name, f, p, vs, mu in S.footprint_cases():
        cfg = RV.VolumeConfig(voxel_size=vs, mu=mu, stream_radius=1e6)
        coords = RV.keyframe_block_footprint(ref_frame(f), ref_pose(p), cfg)
        keys = [int(RV._pack_coords(*c)) for c in coords]
        out.append({"name": name, "keys": keys,
                    "hash_65536": [RV.block_hash(c, 65536) for c in coords]})
    return out


def gen_scripts():
    out = []
    for name, cfg, frames, poses, ops in S.volume_scripts():
        log = S.run_script(RefAdapter(), cfg, frames, poses, ops)
        out.append({"name": name, "log": log})
    return out


def main():
    golden = {
        "generator": "tests/golden/gen_golden.py",
        "reference_backend": RK.BACKEND,
        "hash": gen_hash(),
        "fuse_block": gen_fuse_block(),
        "footprint": gen_footprint(),
        "scripts": gen_scripts(),
    }
    path = os.path.join(HERE, "volume_golden.json")
    with open(path, "w") as fh:
        json.dump(golden, fh, indent=0, sort_keys=True)
    print(f"wrote {path} (backend {RK.BACKEND})")


if __name__ == "__main__":
    main()
