#!/usr/bin/env python
"""C1 (BASELINE configs[0]) end to end: the demo room, 100 frames 640x480
fused into 20 keyframes, 1 cm voxels, the frame-100 pose update corrected
with correct_window(m=20), finalize, marching cubes -- the device pipeline
(paper_1709_03763_b200.pipeline.run_pipeline) against the unmodified
reference pipeline (oracle/_ref, refusion.pipeline.run_pipeline) on the SAME
frames (rendered by the reference's synth), timed on this box, results
compared bit for bit.  Writes one JSON object (stdout, or --out).

Correction throughput = keyframes re-integrated / wall time inside the
correction calls (the frame-100 window + finalize; one KF
re-integration = de-integration at the old pose + integration at the new
one, including footprints, allocation, streaming and GC).

  python tools/bench_c1.py [--out profiles/r2_c1.json] [--repeat 2]
"""

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--repeat", type=int, default=2, help="device runs (first one warms up)")
    ap.add_argument("--no-reference", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch

    import pipeline_cases as PC
    from refimport import reference

    reference()
    import refusion.keyframe_fusion as RKF
    import refusion.pipeline as RP
    import refusion.volume as RV

    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import pipeline as P
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    seq = PC.c1_sequence()
    render_s = time.perf_counter() - t0
    vol = dict(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    dcfg = P.RunConfig(strategy=KF.KeyframeStrategy(kind="KF_CONST", kappa=5), m=20,
                       volume=V.VolumeConfig(**vol), reintegration_mode="consecutive_window",
                       block_capacity=1 << 17)
    dev = []
    for _ in range(max(1, args.repeat)):
        dds = PC.device_dataset(seq)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run = P.run_pipeline(dds, dcfg)
        torch.cuda.synchronize()
        dev.append((time.perf_counter() - t0, run))
    dev_s, drun = dev[-1]
    dstats = drun[1]
    out = {
        "config": "C1: demo room, 100 frames 640x480 -> 20 KF (KF_CONST kappa 5), 1 cm voxels, "
                  "mu 0.06, stream radius 6 m, correct_window(m=20) at the frame-100 pose "
                  "update + finalize; frames rendered by the reference synth "
                  "(sigma0 0.0015, drift 2 mm / 1 mrad per frame, seed 1)",
        "render_s": render_s,
        "device": {"run_s": dev_s, "fuse_ms": dstats.fuse_ms,
                   "integrate_ms": dstats.integrate_ms, "correct_ms": dstats.correct_ms,
                   "corrected_entries": dstats.corrected_entries,
                   "keyframes": dstats.keyframe_count,
                   "correction_kf_per_s": dstats.corrected_entries / (dstats.correct_ms / 1e3),
                   "blocks": int(len(drun[2].export()[0])),
                   "mesh_vertices": int(drun[0].n_vertices),
                   "timing": "host wall clock, device synchronised at every phase boundary"},
    }
    if not args.no_reference:
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        rcfg = RP.RunConfig(strategy=RKF.KeyframeStrategy(kind="KF_CONST", kappa=5), m=20,
                            volume=RV.VolumeConfig(**vol),
                            reintegration_mode="consecutive_window")
        t0 = time.perf_counter()
        rrun = RP.run_pipeline(PC.reference_dataset(seq), rcfg)
        ref_s = time.perf_counter() - t0
        rstats = rrun[1]
        got, want = drun[2].export(), PC.reference_store_export(rrun[2])
        same = (np.array_equal(got[0], want[0])
                and all(np.array_equal(a, b) for a, b in zip(got[1:], want[1:]))
                and np.array_equal(drun[0].vertices, rrun[0].vertices)
                and np.array_equal(drun[0].triangles, rrun[0].triangles)
                and np.array_equal(drun[0].colors, rrun[0].colors))
        out["reference"] = {"run_s": ref_s, "fuse_ms": rstats.fuse_ms,
                            "integrate_ms": rstats.integrate_ms,
                            "correct_ms": rstats.correct_ms,
                            "corrected_entries": rstats.corrected_entries,
                            "correction_kf_per_s": rstats.corrected_entries
                            / (rstats.correct_ms / 1e3),
                            "cores": 1, "threads_available": os.cpu_count(),
                            "kind": "reference (oracle/_ref, compiled backend)"}
        out["bitexact_volume_and_mesh"] = bool(same)
        out["speedup"] = {
            "correction": out["device"]["correction_kf_per_s"]
            / out["reference"]["correction_kf_per_s"],
            "whole_run": ref_s / dev_s,
            "fusion": rstats.fuse_ms / dstats.fuse_ms,
            "integration": rstats.integrate_ms / dstats.integrate_ms,
        }
    text = json.dumps(out, indent=1)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
