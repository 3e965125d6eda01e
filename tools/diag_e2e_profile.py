"""Where the end-to-end correction time goes: the bench's corrections with
keyframes resident vs uploaded from pinned host memory -- each run on a fresh
volume with the same event sequence, so both apply exactly the same
corrections -- with the wall time, the device-event time around the call, and
(profiled runs) rf_profile's per-kernel-class device time.  Diagnostic only."""

import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench as B  # noqa: E402


def main():
    import torch

    from paper_1709_03763_b200 import _lib as L
    from paper_1709_03763_b200 import geometry as G
    from paper_1709_03763_b200 import reintegration as R
    from paper_1709_03763_b200 import synth as SY
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    n_kf = int(os.environ.get("KF", "200"))
    steps = 8
    gt_f, gt, dr = B.kf_poses(n_kf)
    kfs = B.build_keyframes(n_kf, gt_f, dr)
    cfg = V.VolumeConfig(voxel_size=B.VOXEL, mu=B.MU, stream_radius=B.RADIUS,
                         hash_buckets=1 << 21)
    n_anchors = (n_kf + B.EVENT_EVERY_KF - 1) // B.EVENT_EVERY_KF
    events = B.make_events(n_anchors, 4 * steps + 8)
    lib = L.lib()
    stream = torch.cuda.current_stream()
    host = {id(kf): kf.to_host(pinned=True) for kf in kfs}

    def run(label, on_host, profile):
        """A fresh volume and ledger, the same event sequence: every run applies
        exactly the same corrections, so runs differ only in the keyframes'
        location (HBM or pinned host memory) and in profiling."""
        store = V.TwoTierStore(block_capacity=2_000_000)
        for kf, p in zip(kfs, dr):
            V.stream(store, p.translation, cfg)
            V.integrate(store, kf, p, cfg)
        scen = B.Scenario(R, G, SY, gt, dr, kfs, events)
        if on_host:
            for e in scen.ledger.entries:
                e.kf = host[id(e.kf)]
        torch.cuda.synchronize()
        idx = [0]

        def one():
            ev = scen.event(idx[0])
            idx[0] += 1
            R.apply_pose_update(scen.ledger, ev)
            picks = R.select_topk(scen.ledger, B.M_TOPK)
            nxt = scen.ledger.entries[picks[0] - 1].target_pose.translation
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            t = time.perf_counter()
            a.record(stream)
            R.correct_topk(store, scen.ledger, picks, cfg, next_center=nxt)
            b.record(stream)
            b.synchronize()
            return 1e3 * (time.perf_counter() - t), a.elapsed_time(b)

        for _ in range(3):
            one()
        if profile:
            lib.rf_profile_begin(store._ptr)
        walls, devs = [], []
        for _ in range(steps):
            w, d = one()
            walls.append(w)
            devs.append(d)
        out = {"mode": label, "profiled": profile, "wall_ms": round(sum(walls) / steps, 3),
               "event_ms": round(sum(devs) / steps, 3)}
        if profile:
            prof = L.RfProfile()
            lib.rf_profile_end(store._ptr, ctypes.byref(prof))
            out.update({"integrate_ms": round(prof.integrate_ms / steps, 3),
                        "removal_ms": round(prof.removal_ms / steps, 3),
                        "fuse_ms": round(prof.fuse_ms / steps, 3),
                        "check_ms": round(prof.check_ms / steps, 3),
                        "footprint_ms": round(prof.footprint_ms / steps, 3),
                        "other_ms": round(prof.other_ms / steps, 3)})
        print(json.dumps(out), flush=True)
        store.close()
        torch.cuda.synchronize()

    for profile in (False, True):
        run("resident", False, profile)
        run("host", True, profile)
    run("resident", False, False)


if __name__ == "__main__":
    main()
