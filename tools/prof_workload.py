"""Small fixed workload for ncu captures (one GPU): build a corridor volume
from --build keyframes, then run --corrections single-keyframe corrections.
Kernel launch order per correction: reset, stream, (kf_hash, cached) or
footprint, spill, commit, k_fuse<1> (removal check), k_fuse<2> (removal),
stream, kf_hash, footprint, spill, commit, k_fuse<0> (integrate), gc,
stream.  --json writes the corrections' algorithmic bytes per fuse launch
(80 B x voxels_updated + 40 B x H*W, the bench's roofline model) so an ncu
capture of the same launches can be set beside them (tools/ncu_traffic.py)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1709_03763_b200 import _lib as L  # noqa: E402
from paper_1709_03763_b200 import reintegration as R  # noqa: E402
from paper_1709_03763_b200 import synth as SY  # noqa: E402
from paper_1709_03763_b200 import volume as V  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--build", type=int, default=20)
ap.add_argument("--corrections", type=int, default=2)
ap.add_argument("--voxel", type=float, default=bench.VOXEL)
ap.add_argument("--json", default=None)
a = ap.parse_args()

torch.cuda.set_device(0)
gt, gt_kf, drifted = bench.kf_poses(400)
kfs = bench.build_keyframes(a.build, gt, drifted)  # the bench's fused keyframes
cfg = V.VolumeConfig(voxel_size=a.voxel, mu=bench.MU, stream_radius=bench.RADIUS,
                     hash_buckets=1 << 21)
store = V.TwoTierStore(block_capacity=600_000)
for kf, p in zip(kfs, drifted):
    V.stream(store, p.translation, cfg)
    V.integrate(store, kf, p, cfg)
torch.cuda.synchronize()
lib = L.lib()
lib.rf_profile_begin(store._ptr)
# NVTX range "corrections": ncu --nvtx --nvtx-include "corrections/" captures
# exactly these launches, whose algorithmic bytes --json reports
torch.cuda.nvtx.range_push("corrections")
for i in range(a.corrections):
    e = R.LedgerEntry(kfs[i], -1, drifted[i], gt_kf[i], 0, gt_kf[i])
    V.correct_entries(store, [e], cfg, next_center=gt_kf[i].translation)
    drifted[i] = gt_kf[i]
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
prof = L.RfProfile()
lib.rf_profile_end(store._ptr, L.ctypes.byref(prof))
out = {"blocks": store.block_count(), "corrections": a.corrections,
       "fuse_launches": int(prof.fuse_launches), "voxels_updated": int(prof.voxels_updated),
       "blocks_touched": int(prof.blocks_touched),
       "alg_bytes_per_fuse_launch": (80.0 * prof.voxels_updated + 40.0 * prof.pixels)
       / max(prof.fuse_launches, 1),
       "fuse_us_per_launch_events": 1e3 * prof.fuse_ms / max(prof.fuse_launches, 1),
       # the roofline kernel (k_fuse<kIntegrate>): the corrections' integrations
       "integrate_launches": int(prof.integrate_launches),
       "alg_bytes_per_integrate_launch": (80.0 * prof.integrate_voxels +
                                          40.0 * prof.integrate_pixels)
       / max(prof.integrate_launches, 1),
       "integrate_us_per_launch_events": 1e3 * prof.integrate_ms / max(prof.integrate_launches, 1),
       "removal_ops": int(prof.removal_ops),
       "removal_us_per_op_events": 1e3 * prof.removal_ms / max(prof.removal_ops, 1)}
print(json.dumps(out))
if a.json:
    json.dump(out, open(a.json, "w"), indent=1)
