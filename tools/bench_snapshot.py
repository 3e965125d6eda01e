"""SDFV1 snapshots: save_volume streamed from the device and
load_volume, on a corridor volume (the bench's first --keyframes keyframes),
beside the reference's save_volume timed on a bounded sample of the same
blocks (oracle/_ref).  One JSON line; the files go to a temporary directory.

    python tools/bench_snapshot.py [--keyframes 40]"""

import argparse
import json
import os
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keyframes", type=int, default=6)
    ap.add_argument("--ref-blocks", type=int, default=5000)
    args = ap.parse_args()

    import numpy as np
    import torch

    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    gt, gt_kf, drifted = B.kf_poses(args.keyframes)
    kfs = B.build_keyframes(args.keyframes, gt, drifted)
    cfg = V.VolumeConfig(voxel_size=B.VOXEL, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << 21)
    store = V.TwoTierStore(block_capacity=1_500_000)
    for k in range(args.keyframes):
        kf = kfs[k]
        V.stream(store, drifted[k].translation, cfg)
        V.integrate(store, kf, drifted[k], cfg)
    torch.cuda.synchronize()
    n = store.block_count()
    out = {"workload": f"C2 corridor, first {args.keyframes} keyframes at 5 mm: {n} blocks"}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "v.sdf")
        t0 = time.perf_counter()
        V.save_volume(store, path, cfg)
        out["save_s"] = round(time.perf_counter() - t0, 3)
        size = os.path.getsize(path)
        out["file_bytes"] = size
        out["save_GBps"] = round(size / out["save_s"] / 1e9, 2)
        t0 = time.perf_counter()
        loaded, _, _ = V.load_volume(path)
        V.stream(loaded, drifted[-1].translation, cfg)  # binds and uploads
        torch.cuda.synchronize()
        out["load_s"] = round(time.perf_counter() - t0, 3)
        out["roundtrip_equal"] = V.compare_volumes(store, loaded) == (0.0, 0.0, 0.0)
        loaded.close()
        ref_dir = os.path.join(REPO, "oracle", "_ref")
        if os.path.isdir(os.path.join(ref_dir, "refusion")):
            sys.path.insert(0, ref_dir)
            from refusion import volume as RV

            keys, d, w, c = store.export()
            m = min(args.ref_blocks, n)
            rs = RV.TwoTierStore()
            for i in range(m):
                coord = tuple(int(x) for x in V.unpack_keys(keys[i:i + 1])[0])
                rs.active[coord] = RV.VoxelBlock(coord, d[i], w[i], c[i])
            t0 = time.perf_counter()
            RV.save_volume(rs, os.path.join(tmp, "ref.sdf"),
                           RV.VolumeConfig(voxel_size=cfg.voxel_size, mu=cfg.mu))
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"kind": "reference", "cores": 1,
                                   "sample": f"save_volume of {m} blocks",
                                   "save_s_per_block": dt / m,
                                   "save_s_extrapolated": round(dt / m * n, 2)}
            out["save_speedup"] = round(dt / m * n / out["save_s"], 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
