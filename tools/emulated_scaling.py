"""Per-shard device work of the hash-sharded correction at G shards, measured
on ONE B200 by emulation (the scaling model of DESIGN.md §7).

G shard stores live on the one device.  Each is driven by its own thread
through the bench's correction workload (bench.py: C2 corridor, top-10
corrections), in lockstep where the routed footprints need it.  A global
lock serialises the native calls, so every kernel runs alone on the GPU and
each shard's rf_profile (CUDA events around every kernel of the volume)
is its exclusive device time by kernel class; the primary number is the
wall time a shard spends inside its native calls per step (enqueue plus
execution -- every call synchronises -- with no other shard on the GPU).  A real G-GPU run takes about the slowest
shard's time per step, so the predicted parallel efficiency is

    E(G) = T_1 / (G * max_r T_r(G))

(without NVLink transfer and barrier latency, which one GPU cannot show).
Modes: "routed" (rf_route: every shard samples 1/G of the pixel tiles and
stores keys into the owners' inboxes) and "replicated" (every shard samples
every ray and keeps its own keys).

Usage: python tools/emulated_scaling.py [--shards 1,2,4,8] [--keyframes 400]
Writes one JSON line per (mode, G) and a summary line to stdout."""

import argparse
import ctypes
import json
import os
import sys
import threading
import time

# one hardware work queue per stream: the shards' streams must not share
# queues (see tests/conftest.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", default="1,2,4,8")
    ap.add_argument("--modes", default="routed,replicated")
    ap.add_argument("--keyframes", type=int, default=400)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--voxel", type=float, default=None, help="voxel size (default: bench's)")
    args = ap.parse_args()

    import torch

    from paper_1709_03763_b200 import _lib as L
    from paper_1709_03763_b200 import geometry as Gm
    from paper_1709_03763_b200 import reintegration as R
    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    lib = L.lib()
    gt, gt_kf, drifted = B.kf_poses(args.keyframes)
    kfs = B.build_keyframes(args.keyframes, gt, drifted)
    torch.cuda.synchronize()
    voxel = args.voxel or B.VOXEL
    cfg = V.VolumeConfig(voxel_size=voxel, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << 22 if voxel < B.VOXEL else 1 << 21)
    n_anchors = (args.keyframes + B.EVENT_EVERY_KF - 1) // B.EVENT_EVERY_KF
    events = B.make_events(n_anchors, args.warmup + 2 * args.steps + 2)

    def run(G, mode):
        cap = int(2_600_000 * (B.VOXEL / voxel) ** 3) // G + 200_000
        stores = [V.TwoTierStore(block_capacity=cap, shard_rank=r, shard_count=G)
                  for r in range(G)]
        if G > 1 and mode == "routed":
            # native calls are serialised below, so a shard's call cannot wait
            # for another's: no device-side removal verdicts (one NVLink round
            # trip per removal on real GPUs, not in this model)
            V.connect_shards(stores, cfg, verdicts=False)
        lock = threading.Lock()
        native = [0.0] * G  # per shard: wall time inside its native calls
        for r, s in enumerate(stores):
            s._bind(cfg)
            inner = s._call_status

            def locked(*a, _inner=inner, _r=r):
                with lock:
                    t = time.perf_counter()
                    try:
                        return _inner(*a)
                    finally:
                        native[_r] += time.perf_counter() - t

            s._call_status = locked
        out = [None] * G

        def body(r):
            torch.cuda.set_device(0)
            s = stores[r]
            try:
                scen = B.Scenario(R, Gm, SY, gt_kf, drifted, kfs, events)
                for kf, pose in zip(kfs, drifted):
                    V.stream(s, pose.translation, cfg)
                    V.integrate(s, kf, pose, cfg)

                def one(i):
                    R.apply_pose_update(scen.ledger, scen.event(i))
                    picks = R.select_topk(scen.ledger, B.M_TOPK)
                    nxt = scen.ledger.entries[picks[0] - 1].target_pose.translation
                    return R.correct_topk(s, scen.ledger, picks, cfg, next_center=nxt)

                for i in range(args.warmup):
                    one(i)
                # timed steps: native-call wall time (the calls synchronise,
                # so this is enqueue + device execution, one shard at a time)
                with lock:
                    native[r] = 0.0
                n = 0
                for i in range(args.warmup, args.warmup + args.steps):
                    n += one(i)
                nat = native[r]
                # profiled steps: per-kernel-class device time (events)
                with lock:
                    lib.rf_profile_begin(s._ptr)
                for i in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
                    one(i)
                prof = L.RfProfile()
                with lock:
                    lib.rf_profile_end(s._ptr, ctypes.byref(prof))
                out[r] = (n, prof, s.block_count(), nat)
            except Exception as e:  # noqa: BLE001 -- reported below
                out[r] = e

        t0 = time.time()
        th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.time() - t0
        for s in stores:
            s.close()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        for o in out:
            if isinstance(o, Exception):
                raise o
        per = []
        for n, p, nb, nat in out:
            ms = p.fuse_ms + p.check_ms + p.footprint_ms + p.other_ms
            per.append({"ms_per_step": 1e3 * nat / args.steps,
                        "events_ms_per_step": ms / args.steps, "fuse": p.fuse_ms / args.steps,
                        "check": p.check_ms / args.steps,
                        "footprint": p.footprint_ms / args.steps,
                        "other": p.other_ms / args.steps, "launches": p.kernel_launches // args.steps,
                        "blocks": nb, "corrected": n})
        return per, wall

    res = {}
    for mode in args.modes.split(","):
        for G in [int(g) for g in args.shards.split(",")]:
            if G == 1 and mode != args.modes.split(",")[0]:
                continue
            per, wall = run(G, mode if G > 1 else "single")
            worst = max(p["ms_per_step"] for p in per)
            res[(mode, G)] = worst
            line = {"mode": mode if G > 1 else "single", "shards": G,
                    "max_shard_ms_per_step": round(worst, 4),
                    "mean_shard_ms_per_step": round(sum(p["ms_per_step"] for p in per) / G, 4),
                    "shards_detail": [{k: (round(v, 4) if isinstance(v, float) else v)
                                       for k, v in p.items()} for p in per],
                    "wall_s": round(wall, 1)}
            print(json.dumps(line), flush=True)
    t1 = res.get((args.modes.split(",")[0], 1))
    if t1:
        summ = {"T1_ms_per_step": round(t1, 4)}
        for (mode, G), t in sorted(res.items()):
            if G > 1:
                summ[f"E_{mode}_{G}"] = round(t1 / (G * t), 3)
        print(json.dumps({"summary": summ}), flush=True)


if __name__ == "__main__":
    main()
