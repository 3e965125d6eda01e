"""Where the end-to-end (host keyframes) correction time goes: pinned H2D
bandwidth of the keyframe planes alone, then the same corrections with the
keyframes resident vs uploaded per call (one GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1709_03763_b200 import reintegration as R  # noqa: E402
from paper_1709_03763_b200 import synth as SY  # noqa: E402
from paper_1709_03763_b200 import volume as V  # noqa: E402

torch.cuda.set_device(0)
n = 40
gt_f, gt, dr = bench.kf_poses(n)
kfs = bench.build_keyframes(n, gt_f, dr)
host = [k.to_host(pinned=True) for k in kfs]
torch.cuda.synchronize()
# 1. H2D bandwidth, 10 keyframes' planes
dst = [torch.empty_like(k.depth) for k in kfs[:10]] + [torch.empty_like(k.color) for k in kfs[:10]]
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(10):
        dst[i].copy_(host[i].depth, non_blocking=True)
        dst[10 + i].copy_(host[i].color, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
nbytes = 10 * 640 * 480 * 32
print(f"H2D depth+colour of 10 KF: {nbytes / dt / 1e9:.1f} GB/s ({1e3 * dt:.2f} ms)")
cfg = V.VolumeConfig(voxel_size=bench.VOXEL, mu=bench.MU, stream_radius=bench.RADIUS,
                     hash_buckets=1 << 21)
store = V.TwoTierStore(block_capacity=2_000_000)
for kf, p in zip(kfs, dr):
    V.stream(store, p.translation, cfg)
    V.integrate(store, kf, p, cfg)
torch.cuda.synchronize()


def run(planes, label):
    ts = []
    for rep in range(4):
        ledger = R.IntegrationLedger()
        ledger.declare_anchor(0, SY.pose_interpolate(dr[0], dr[0], 0.0))
        for i in range(10):
            e = ledger.add(planes[i], i + 1, 0, dr[i], dr[i])
            e.integrated_pose = dr[i].copy() if rep % 2 == 0 else gt[i].copy()
            e.target_pose = gt[i].copy() if rep % 2 == 0 else dr[i].copy()
        torch.cuda.synchronize()
        t = time.perf_counter()
        R.correct_topk(store, ledger, list(range(1, 11)), cfg)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    print(label, " ".join(f"{x:.2f}" for x in ts), "ms per 10-KF correction")


run(kfs, "resident")
run(host, "host   ")
run(kfs, "resident")
run(host, "host   ")
