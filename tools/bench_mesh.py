"""Marching cubes on the bench's volume: the 400-keyframe C2
corridor at 5 mm built as bench.py builds it, meshed on the device
(rf_marching_cubes), and the reference's CPU marching_cubes timed on a
bounded sample of the same blocks (oracle/_ref when present, else the numpy
oracle restatement), extrapolated per block.  One JSON line.

    python tools/bench_mesh.py [--keyframes 400] [--cpu-blocks 300]"""

import argparse
import ctypes
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keyframes", type=int, default=400)
    ap.add_argument("--cpu-blocks", type=int, default=300)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()

    import numpy as np
    import torch

    from paper_1709_03763_b200 import meshing as M
    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    gt, gt_kf, drifted = B.kf_poses(args.keyframes)
    kfs = B.build_keyframes(args.keyframes, gt, drifted)
    cfg = V.VolumeConfig(voxel_size=B.VOXEL, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << 21)
    store = V.TwoTierStore(block_capacity=2_800_000)
    for k in range(args.keyframes):
        kf = kfs[k]
        V.stream(store, drifted[k].translation, cfg)
        V.integrate(store, kf, drifted[k], cfg)
    torch.cuda.synchronize()
    n_blocks = store.block_count()

    nv, nt = ctypes.c_int64(), ctypes.c_int64()

    def count_only():
        store._call("rf_marching_cubes", None, None, None, 0, 0, ctypes.byref(nv), ctypes.byref(nt))

    count_only()
    mesh = M.marching_cubes(store, cfg)  # warm
    t_count, t_full = [], []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        count_only()
        t_count.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        mesh = M.marching_cubes(store, cfg)
        t_full.append(time.perf_counter() - t0)

    t_weld = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        welded = M.welded_mesh(store, cfg, 1e-7)
        t_weld.append(time.perf_counter() - t0)

    # reference on a bounded sample of blocks (their +axis neighbours included)
    keys, d, w, c = store.export()
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(len(keys), size=min(args.cpu_blocks, len(keys)), replace=False))
    kind = "port"
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    cpu_s = None
    if os.path.isdir(os.path.join(ref_dir, "refusion")):
        sys.path.insert(0, ref_dir)
        from refusion import meshing as RM
        from refusion import volume as RV

        rs = RV.TwoTierStore()
        for i in range(len(keys)):
            k = int(keys[i])
            coord = ((k >> 42) - (1 << 20), ((k >> 21) & ((1 << 21) - 1)) - (1 << 20),
                     (k & ((1 << 21) - 1)) - (1 << 20))
            rs.active[coord] = RV.VoxelBlock(coord, d[i], w[i], c[i])
        coords = sorted(rs.active)
        sample = [coords[i] for i in pick]
        t0 = time.perf_counter()
        for coord in sample:
            RM._block_cells(rs, rs.find(coord), RV.VolumeConfig(voxel_size=B.VOXEL))
        cpu_s = time.perf_counter() - t0
        kind = "reference"
    else:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import mesh_oracle as MO

        data = np.concatenate([d[:, None], w[:, None], np.transpose(c, (0, 2, 1))], axis=1)
        index = {int(k): i for i, k in enumerate(keys)}
        t0 = time.perf_counter()
        for i in pick:
            MO._cells(index, data, MO._coords(keys[i]), B.VOXEL)
        cpu_s = time.perf_counter() - t0
    cpu_per_block = cpu_s / len(pick)
    dev = min(t_count) + 0.0
    full = min(t_full)
    out_bytes = mesh.n_vertices * 48 + mesh.n_triangles * 24
    print(json.dumps({
        "workload": f"C2 corridor {args.keyframes} KF at 5 mm: {n_blocks} blocks",
        "vertices": mesh.n_vertices, "triangles": mesh.n_triangles,
        "device_count_pass_ms": round(1e3 * dev, 2),
        "mesh_to_host_ms": round(1e3 * full, 2),
        "mesh_bytes": out_bytes,
        "blocks_per_s_to_host": round(n_blocks / full, 1),
        "cpu_baseline": {"kind": kind, "cores": 1, "sample": f"{len(pick)} random blocks",
                         "s_per_block": cpu_per_block,
                         "blocks_per_s": round(1.0 / cpu_per_block, 1),
                         "extrapolated_s_whole_volume": round(cpu_per_block * n_blocks, 1)},
        "speedup_to_host": round(cpu_per_block * n_blocks / full, 1),
        "welded_on_device_to_host_ms": round(1e3 * min(t_weld), 2),
        "welded_vertices": welded.n_vertices, "welded_triangles": welded.n_triangles,
    }))


if __name__ == "__main__":
    main()
