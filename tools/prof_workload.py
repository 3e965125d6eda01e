"""Small fixed workload for ncu captures (one GPU): build a corridor volume
from --build keyframes, then run --corrections single-keyframe corrections.
Kernel launch order: build = (reset, stream, footprint, commit, fuse<0>) x N,
then per correction (reset, stream x2, footprint, commit, fuse<1>, fuse<2>,
stream x2, footprint, commit, fuse<0>, gc, stream)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1709_03763_b200 import reintegration as R  # noqa: E402
from paper_1709_03763_b200 import synth as SY  # noqa: E402
from paper_1709_03763_b200 import volume as V  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--build", type=int, default=20)
ap.add_argument("--corrections", type=int, default=2)
ap.add_argument("--voxel", type=float, default=bench.VOXEL)
a = ap.parse_args()

torch.cuda.set_device(0)
gt_kf, drifted = bench.kf_poses(400)
rend = SY.Renderer(SY.corridor_scene(), SY.DEFAULT_INTRINSICS)
kfs = [SY.render_keyframe(rend, gt_kf[k], seed=1000 + k) for k in range(a.build)]
cfg = V.VolumeConfig(voxel_size=a.voxel, mu=bench.MU, stream_radius=bench.RADIUS,
                     hash_buckets=1 << 21)
store = V.TwoTierStore(block_capacity=600_000)
for kf, p in zip(kfs, drifted):
    V.stream(store, p.translation, cfg)
    V.integrate(store, kf, p, cfg)
torch.cuda.synchronize()
for i in range(a.corrections):
    e = R.LedgerEntry(kfs[i], -1, drifted[i], gt_kf[i], 0, gt_kf[i])
    V.correct_entries(store, [e], cfg, next_center=gt_kf[i].translation)
    drifted[i] = gt_kf[i]
torch.cuda.synchronize()
print("blocks", store.block_count())
