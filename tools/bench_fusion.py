"""Keyframe fusion on the device (SURVEY §8 rows a1 fuse_depth, a2 fuse_color):
kappa = 5 corridor frames (640x480, rendered on the GPU with noise) fused into
each keyframe, device time per operation with CUDA events, and the
reference's CPU keyframe_fusion (oracle/_ref, compiled backend) timed on one
keyframe of the same frames beside it, its result compared bit for bit.
One JSON line.

    python tools/bench_fusion.py [--keyframes 12] [--kappa 5]"""

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keyframes", type=int, default=12)
    ap.add_argument("--kappa", type=int, default=5)
    args = ap.parse_args()

    import numpy as np
    import torch

    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import synth as SY

    torch.cuda.set_device(0)
    n_frames = args.keyframes * args.kappa
    traj = SY.corridor_trajectory(B.N_FRAMES)[:n_frames]  # the bench trajectory
    rend = SY.Renderer(SY.corridor_scene(), SY.DEFAULT_INTRINSICS, device=0)
    frames = []
    for i in range(n_frames):
        d, c = rend.render(traj[i], seed=7000 + i)
        frames.append((d, c))
    torch.cuda.synchronize()
    intr = SY.DEFAULT_INTRINSICS
    stream = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    KF.detect_blas_order()
    t_depth, t_color = [], []
    for k in range(args.keyframes):
        kf = None
        for j in range(args.kappa):
            i = k * args.kappa + j
            fo = KF.FrameObservation(i + 1, frames[i][1], frames[i][0], traj[i])
            if kf is None:
                kf = KF.new_keyframe(fo, intr)
            a = ev()
            KF.fuse_depth(kf, fo)
            b = ev()
            t_depth.append((a, b))
        a = ev()
        KF.fuse_color(kf)
        b = ev()
        t_color.append((a, b))
    torch.cuda.synchronize()
    skip = args.kappa  # first keyframe: warm-up
    dms = [a.elapsed_time(b) for a, b in t_depth[skip:]]
    cms = [a.elapsed_time(b) for a, b in t_color[1:]]

    # reference: one keyframe of the same frames on the host CPU
    ref = None
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "refusion")):
        sys.path.insert(0, ref_dir)
        os.environ.setdefault("REFUSION_BACKEND", "compiled")
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        from refusion import geometry as RG
        from refusion import keyframe_fusion as RK

        rintr = RG.Intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
        host = [(d.cpu().numpy(), c.cpu().numpy()) for d, c in frames[: args.kappa]]
        rposes = [RG.Pose(np.asarray(p.rotation), np.asarray(p.translation))
                  for p in traj[: args.kappa]]
        rkf = None
        t0 = time.perf_counter()
        for j in range(args.kappa):
            rf = RK.FrameObservation(j + 1, host[j][1], host[j][0], rposes[j])
            if rkf is None:
                rkf = RK.new_keyframe(rf, rintr)
            RK.fuse_depth(rkf, rf)
        t1 = time.perf_counter()
        RK.fuse_color(rkf)
        t2 = time.perf_counter()
        # the device's first keyframe, recomputed for the comparison
        kf = None
        for j in range(args.kappa):
            fo = KF.FrameObservation(j + 1, frames[j][1], frames[j][0], traj[j])
            if kf is None:
                kf = KF.new_keyframe(fo, intr)
            KF.fuse_depth(kf, fo)
        KF.fuse_color(kf)
        same = (np.array_equal(kf.depth.cpu().numpy(), rkf.depth)
                and np.array_equal(kf.weight.cpu().numpy(), rkf.weight)
                and np.array_equal(kf.color.cpu().numpy(), rkf.color))
        ref = {"kind": "reference", "cores": 1, "sample": f"1 keyframe of {args.kappa} frames",
               "fuse_depth_ms_per_frame": round(1e3 * (t1 - t0) / args.kappa, 1),
               "fuse_color_ms_per_keyframe": round(1e3 * (t2 - t1), 1),
               "bit_identical": bool(same)}
    npix = intr.width * intr.height
    # algorithmic bytes: fuse_depth reads the frame depth + colour, reads and
    # writes the keyframe depth / weight, writes the member copies (depth,
    # weight map, prepared colour); fuse_color reads kappa members' depth,
    # weight map and colour plus the keyframe planes, writes colour + valid
    depth_bytes = npix * (8 + 24 + 32 + 8 + 8 + 24)
    color_bytes = npix * (args.kappa * (8 + 8 + 24) + 16 + 24 + 1)
    dmean, cmean = float(np.mean(dms)), float(np.mean(cms))
    out = {
        "workload": f"C2 corridor frames 640x480, kappa {args.kappa}, "
                    f"{args.keyframes - 1} timed keyframes",
        "fuse_depth_ms_per_frame": round(dmean, 4),
        "fuse_color_ms_per_keyframe": round(cmean, 4),
        "keyframe_ms": round(args.kappa * dmean + cmean, 4),
        "fuse_depth_GBps_alg": round(depth_bytes / dmean / 1e6, 1),
        "fuse_color_GBps_alg": round(color_bytes / cmean / 1e6, 1),
        "cpu_baseline": ref,
    }
    if ref:
        out["speedup_keyframe"] = round(
            (args.kappa * ref["fuse_depth_ms_per_frame"] + ref["fuse_color_ms_per_keyframe"])
            / (args.kappa * dmean + cmean), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
