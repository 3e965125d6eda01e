"""TEST INFRASTRUCTURE -- datasets for the end-to-end pipeline parity runs.

Frames are rendered by the reference's own synthetic generator
(/root/reference/pkg/src/refusion/synth.py:220-376, imported from the
reference build in oracle/_ref), so the device pipeline and the reference
pipeline consume bit-identical inputs.  ``sequence`` reproduces
``synth.make_sequence`` (drifted poses, anchor and correction events) but
renders the frames in a process pool: each frame is a pure function of the
scene, its ground-truth pose and the per-frame noise seed (seed, 7, index).
"""

import os

import numpy as np

from refimport import reference

C1 = dict(waypoints=9, radius=1.2, height=1.3, frames_per_segment=11, drift=(0.002, 0.001),
          schedule=[(100, 1.0)], seed=1, sigma0=0.0015, z_max=5.0, anchor_interval=10)


def _ref_synth():
    reference()
    import refusion.synth as RS

    return RS


def _render_one(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    RS = _ref_synth()
    scene, gt, intr, seed, index, sigma0, z_max = args
    depth = RS.render_depth(scene, gt, intr, z_max=z_max)
    if sigma0 > 0.0:
        depth = RS.add_noise(depth, seed=(seed, 7, index), sigma0=sigma0)
    color = RS.render_color(scene, gt, intr, depth)
    return index, depth, color


def sequence(scene, spec, intr, seed=0, noise_sigma0=0.0, anchor_interval=10, z_max=10.0,
             workers=None):
    """synth.make_sequence(scene, spec, intr, seed, noise_sigma0,
    anchor_interval=..., z_max=...) with the frames rendered in parallel."""
    RS = _ref_synth()
    real = (RS.render_depth, RS.render_color, RS.add_noise)
    h, w = intr.height, intr.width
    try:  # poses and events only: the frame loop's other steps do not look at pixels
        RS.render_depth = lambda *a, **k: np.zeros((h, w))
        RS.render_color = lambda *a, **k: np.zeros((h, w, 3))
        RS.add_noise = lambda d, **k: d
        seq = RS.make_sequence(scene, spec, intr, seed=seed, noise_sigma0=noise_sigma0,
                               anchor_interval=anchor_interval, z_max=z_max)
    finally:
        RS.render_depth, RS.render_color, RS.add_noise = real
    jobs = [(scene, seq.gt_poses[f.index], intr, seed, f.index, noise_sigma0, z_max)
            for f in seq.frames]
    n = workers or min(len(jobs), os.cpu_count() or 1)
    if n > 1 and len(jobs) > 2:
        import concurrent.futures as cf
        import multiprocessing as mp

        with cf.ProcessPoolExecutor(n, mp_context=mp.get_context("spawn")) as ex:
            out = list(ex.map(_render_one, jobs, chunksize=1))
    else:
        out = [_render_one(j) for j in jobs]
    frames = [RS.RenderedFrame(index=i, depth=d, color=c) for i, d, c in out]
    return RS.SyntheticSequence(frames=frames, gt_poses=seq.gt_poses,
                                drifted_poses=seq.drifted_poses, events=seq.events,
                                intrinsics=intr)


def c1_sequence(workers=None):
    """BASELINE configs[0] / SURVEY §8(d) C1: demo room, 9-waypoint orbit x 11
    frames = 100 frames at 640x480, drift (2 mm, 1 mrad) per frame, noise
    sigma0 0.0015, one full correction at frame 100."""
    RS = _ref_synth()
    c = C1
    spec = RS.TrajectorySpec(
        waypoints=RS.orbit_waypoints(c["waypoints"], radius=c["radius"], height=c["height"]),
        frames_per_segment=c["frames_per_segment"], drift_rate=c["drift"],
        correction_schedule=c["schedule"])
    return sequence(RS.demo_scene(), spec, RS.DEFAULT_INTRINSICS, seed=c["seed"],
                    noise_sigma0=c["sigma0"], anchor_interval=c["anchor_interval"],
                    z_max=c["z_max"], workers=workers)


def small_sequence():
    """The reference's own pipeline fixture (tests/test_pipeline.py:61-70):
    41 frames at 64x48 around the demo room, drifting, with a mid-run and a
    final correction."""
    RS = _ref_synth()
    import refusion.geometry as RG

    intr = RG.Intrinsics(60.0, 60.0, 31.5, 23.5, 64, 48)
    spec = RS.TrajectorySpec(waypoints=RS.orbit_waypoints(4, radius=1.2, height=1.3),
                             frames_per_segment=10, drift_rate=(0.004, 0.003),
                             correction_schedule=[(15, 0.5), (41, 1.0)])
    return RS.make_sequence(RS.demo_scene(), spec, intr, seed=3, anchor_interval=5)


def reference_dataset(seq):
    reference()
    from refusion.dataset_io import Dataset
    from refusion.keyframe_fusion import FrameObservation

    frames = [FrameObservation(index=f.index, color=f.color, depth=f.depth,
                               pose=seq.drifted_poses[f.index]) for f in seq.frames]
    return Dataset(frames=frames, intrinsics=seq.intrinsics, gt_poses=seq.gt_poses,
                   events=seq.events)


class DeviceDataset:
    def __init__(self, frames, intrinsics, events, gt_poses=None):
        self.frames, self.intrinsics, self.events, self.gt_poses = \
            frames, intrinsics, events, gt_poses

    @property
    def n_frames(self):
        return len(self.frames)


def device_dataset(seq):
    """The same sequence in the device package's own types."""
    from paper_1709_03763_b200 import geometry as G
    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import reintegration as R

    def pose(p):
        return G.Pose(p.rotation, p.translation)

    i = seq.intrinsics
    intr = G.Intrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height)
    frames = [KF.FrameObservation(index=f.index, color=f.color, depth=f.depth,
                                  pose=pose(seq.drifted_poses[f.index])) for f in seq.frames]
    events = [R.PoseUpdateEvent(at_frame=e.at_frame,
                                anchor_poses={a: pose(p) for a, p in e.anchor_poses.items()},
                                dvo_kf_flags=set(e.dvo_kf_flags)) for e in seq.events]
    return DeviceDataset(frames, intr, events, {k: pose(v) for k, v in seq.gt_poses.items()})


def reference_store_export(store):
    """(keys sorted, d[n,512], w[n,512], c[n,512,3]) of a reference store,
    both tiers (the device export's layout)."""
    from oracle import pack_coords

    blocks = dict(store.active)
    blocks.update(store.host)
    coords = sorted(blocks)
    if not coords:
        return (np.zeros(0, np.int64), np.zeros((0, 512)), np.zeros((0, 512)),
                np.zeros((0, 512, 3)))
    a = np.asarray(coords, dtype=np.int64)
    keys = pack_coords(a[:, 0], a[:, 1], a[:, 2])
    order = np.argsort(keys, kind="stable")
    d = np.stack([blocks[coords[j]].d for j in order])
    w = np.stack([blocks[coords[j]].w for j in order])
    c = np.stack([blocks[coords[j]].c for j in order])
    return keys[order], d, w, c
