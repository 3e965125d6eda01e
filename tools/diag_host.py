"""Host-side cost of one correct_topk call (Python marshalling before the
native call, the native enqueue, the wait) on device-resident keyframes."""
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
n = 20
gt_f, gt, dr = bench.kf_poses(n)
kfs = bench.build_keyframes(n, gt_f, dr)
cfg = V.VolumeConfig(voxel_size=bench.VOXEL, mu=bench.MU, stream_radius=bench.RADIUS,
                     hash_buckets=1 << 21)
store = V.TwoTierStore(block_capacity=1_000_000)
for kf, p in zip(kfs, dr):
    V.stream(store, p.translation, cfg)
    V.integrate(store, kf, p, cfg)
torch.cuda.synchronize()
marks = {}
orig = store._call


def timed_call(name, *args):
    marks["enter"] = time.perf_counter()
    orig(name, *args)
    marks["exit"] = time.perf_counter()


store._call = timed_call
for rep in range(6):
    ledger = R.IntegrationLedger()
    ledger.declare_anchor(0, dr[0])
    for i in range(10):
        e = ledger.add(kfs[i], i + 1, 0, dr[i], dr[i])
        e.integrated_pose = (dr[i] if rep % 2 == 0 else gt[i]).copy()
        e.target_pose = (gt[i] if rep % 2 == 0 else dr[i]).copy()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R.correct_topk(store, ledger, list(range(1, 11)), cfg)
    t1 = time.perf_counter()
    print(f"total {1e3 * (t1 - t0):.3f} ms  python-before {1e3 * (marks['enter'] - t0):.3f} ms  "
          f"native {1e3 * (marks['exit'] - marks['enter']):.3f} ms  python-after "
          f"{1e3 * (t1 - marks['exit']):.3f} ms")
