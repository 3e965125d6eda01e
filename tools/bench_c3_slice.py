"""C3's single-GPU slice (BASELINE configs[2]): a building --
outer RoomShell 40 x 40 x 3 m with interior BoxSolid walls and door gaps (a
union of RoomShells would intersect the rooms, synth.py:70-97) -- walked
through its 3 x 3 rooms and back to the start, 20,000 frames fused
kappa = 10 into 2,000 keyframes at 5 mm, integrated at drifted poses; then a
loop closure moves every anchor to its true pose and `finalize` re-integrates
every moved keyframe.  C3 runs hash-sharded over 8 GPUs; this is ONE shard
(rank 0 of 8: replicated ray sampling, the blocks it owns), i.e. one GPU's
share of the job, with all 2,000 keyframes resident in its HBM.

One JSON line: frames / keyframes / blocks, the fusion and build times, and
the finalize: keyframes re-integrated per second on this shard.  Device timed
with CUDA events; the building frames come from the device port of the
reference renderer (bit-identical to synth.py).

    python tools/bench_c3_slice.py [--keyframes 2000] [--kappa 10] [--shards 8]

C5's single-GPU slice (BASELINE configs[4]: 4,000 keyframes at 4 mm, the
scaling sweep's volume) is the same run at --keyframes 4000 --kappa 5
--voxel 0.004 --tag C5 (the building stands in for C5's scene; shard 0 of 8)."""

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def building(SY):
    """Outer shell + a 3 x 3 grid of rooms (walls 0.15 m thick, a 1.2 m door
    gap in every wall segment between two rooms) + a few furniture pieces."""
    P = []
    P.append(SY.Prim(SY.ROOM, (20.0, 20.0, 1.5), (20.0, 20.0, 1.5), (200.0, 195.0, 185.0)))
    cell, half_t, door = 40.0 / 3.0, 0.075, 0.6
    for k in (1, 2):  # interior wall lines x = k * cell and y = k * cell
        c = k * cell
        for seg in range(3):  # three segments per line, a door at each segment's middle
            a, b = seg * cell, (seg + 1) * cell
            mid = 0.5 * (a + b)
            for lo, hi in ((a, mid - door), (mid + door, b)):
                hc, hl = 0.5 * (lo + hi), 0.5 * (hi - lo)
                alb = (150.0 + 20 * k, 160.0 + 10 * seg, 170.0)
                P.append(SY.Prim(SY.BOX, (c, hc, 1.5), (half_t, hl, 1.5), alb))   # x wall
                P.append(SY.Prim(SY.BOX, (hc, c, 1.5), (hl, half_t, 1.5), alb))   # y wall
    assert len(P) == 25
    for i, (x, y) in enumerate([(5, 8), (26, 5), (34, 28), (8, 33), (20, 20)]):
        P.append(SY.Prim(SY.BOX, (x, y, 0.4), (0.6, 0.4, 0.4), (80.0 + 30 * i, 140.0, 90.0)))
    return P


def tour(SY, n_frames):
    """A loop through the 3 x 3 rooms: room centres in serpentine order,
    crossing every shared wall through its door, back to the first room."""
    cell = 40.0 / 3.0
    c = [cell * (i + 0.5) for i in range(3)]
    order = [(0, 0), (1, 0), (2, 0), (2, 1), (1, 1), (0, 1), (0, 2), (1, 2), (2, 2), (2, 1),
             (1, 1), (1, 0), (0, 0)]
    pts = [(c[i], c[j]) for i, j in order]
    seg = [(pts[k], pts[k + 1]) for k in range(len(pts) - 1)]
    per = n_frames // len(seg)
    poses = []
    import numpy as np

    for k, ((x0, y0), (x1, y1)) in enumerate(seg):
        for f in range(per):
            s = f / per
            x, y = x0 + s * (x1 - x0), y0 + s * (y1 - y0)
            yaw = np.arctan2(y1 - y0, x1 - x0) + 0.6 * np.sin(2 * np.pi * (k * per + f) / 300.0)
            poses.append(SY.look_at_pose((x, y, 1.5), (x + np.cos(yaw), y + np.sin(yaw), 1.4)))
    while len(poses) < n_frames:
        poses.append(poses[-1].copy())
    return poses


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keyframes", type=int, default=2000)
    ap.add_argument("--kappa", type=int, default=10)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--blocks", type=int, default=2_400_000)
    ap.add_argument("--voxel", type=float, default=None, help="voxel size (default: the bench's 5 mm)")
    ap.add_argument("--hash-bits", type=int, default=21)
    ap.add_argument("--tag", default="C3")
    args = ap.parse_args()

    import numpy as np
    import torch

    import bench as B
    from paper_1709_03763_b200 import geometry as G
    from paper_1709_03763_b200 import reintegration as R
    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    n_kf, kappa = args.keyframes, args.kappa
    gt = tour(SY, n_kf * kappa)
    gt_kf = [gt[k * kappa] for k in range(n_kf)]
    drifted = SY.drift_poses(gt_kf, B.DRIFT_T, B.DRIFT_R, seed=1)
    rend = SY.Renderer(building(SY), SY.DEFAULT_INTRINSICS, device=0)
    t0 = time.time()
    kfs = []
    for k in range(n_kf):
        k0 = k * kappa
        kf = SY.fused_keyframe(rend, gt[k0:k0 + kappa], SY.burst_poses(gt, k, drifted[k], kappa),
                               [B.frame_seed(k0 + j) for j in range(kappa)], first_index=k0 + 1)
        kf.pose = drifted[k]
        kfs.append(kf)
    torch.cuda.synchronize()
    fuse_s = time.time() - t0

    voxel = args.voxel or B.VOXEL
    cfg = V.VolumeConfig(voxel_size=voxel, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << args.hash_bits)
    store = V.TwoTierStore(block_capacity=args.blocks, shard_rank=args.rank,
                           shard_count=args.shards)
    store._bind(cfg)
    store._call("rf_reserve", B.W, B.H, 4 * 1024)
    ledger = R.IntegrationLedger()
    true_a, bel = {}, {}
    t0 = time.time()
    for k, (kf, pose) in enumerate(zip(kfs, drifted)):
        a = k // B.EVENT_EVERY_KF
        if a not in bel:
            true_a[a], bel[a] = gt_kf[k], drifted[k]
            ledger.declare_anchor(a, drifted[k])
        ledger.add(kf, k + 1, a, G.compose(G.inverse(bel[a]), drifted[k]), drifted[k])
        V.stream(store, pose.translation, cfg)
        V.integrate(store, kf, pose, cfg)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    blocks = store.block_count()
    # the loop closure: every anchor back to its true pose (fraction 1.0)
    R.apply_pose_update(ledger, R.PoseUpdateEvent(at_frame=n_kf * kappa,
                                                  anchor_poses={a: p.copy() for a, p in
                                                                true_a.items()}))
    stream = torch.cuda.current_stream()
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    a_ev.record(stream)
    n = R.finalize(store, ledger, cfg)
    b_ev.record(stream)
    b_ev.synchronize()
    fin_ms = a_ev.elapsed_time(b_ev)
    out = {
        "config": f"{args.tag} single-GPU slice: building 40x40x3 m (outer RoomShell + interior "
                  f"BoxSolid walls with door gaps, 3x3 rooms), {n_kf * kappa} frames -> "
                  f"{n_kf} keyframes (kappa {kappa}), {voxel * 1e3:g} mm, drifted poses, loop closure "
                  f"(every anchor to its true pose) -> finalize; shard {args.rank} of "
                  f"{args.shards} (replicated sampling, owned blocks), all keyframes in HBM",
        "frames": n_kf * kappa, "keyframes": n_kf, "fusion_s": round(fuse_s, 1),
        "device_mem_used_gb": round((lambda f: (f[1] - f[0]) / 1e9)(torch.cuda.mem_get_info()), 1),
        "build_integrate_s": round(build_s, 2), "shard_blocks": blocks,
        "finalize": {"keyframes_corrected": n, "ms": fin_ms,
                     "keyframes_per_s": n / (fin_ms / 1e3), "wall_s": round(time.time() - t0, 2),
                     "timing": "CUDA events around reintegration.finalize"},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
