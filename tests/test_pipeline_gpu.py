"""End-to-end pipeline on the device vs the reference pipeline
(/root/reference/pkg/src/refusion/pipeline.py:179-292 run from oracle/_ref
on the same host and the same frames): keyframe fusion, integration,
window / top-k corrections and finalize, checked bit for bit on the final
volume, the ledger, the streaming counters and the mesh.  Also the
reference's own pipeline tests (tests/test_pipeline.py) on the device."""

import math
import os
import time

import numpy as np
import pytest

import pipeline_cases as PC
from refimport import reference

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(reference() is None, reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def P():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import pipeline

    return pipeline


@pytest.fixture(scope="module")
def small():
    seq = PC.small_sequence()
    return seq, PC.reference_dataset(seq), PC.device_dataset(seq)


def _run_pair(P, seq_pair, kind, kappa, m, mode, vs=0.02, radius=5.0):
    import refusion.keyframe_fusion as RKF
    import refusion.pipeline as RP
    import refusion.volume as RV

    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import volume as V

    _, rds, dds = seq_pair
    rcfg = RP.RunConfig(strategy=RKF.KeyframeStrategy(kind=kind, kappa=kappa), m=m,
                        volume=RV.VolumeConfig(voxel_size=vs, mu=0.06, stream_radius=radius),
                        reintegration_mode=mode)
    dcfg = P.RunConfig(strategy=KF.KeyframeStrategy(kind=kind, kappa=kappa), m=m,
                       volume=V.VolumeConfig(voxel_size=vs, mu=0.06, stream_radius=radius),
                       reintegration_mode=mode, block_capacity=1 << 16)
    return RP.run_pipeline(rds, rcfg), P.run_pipeline(dds, dcfg)


def assert_runs_equal(ref_run, dev_run):
    rmesh, rstats, rstore, rledger = ref_run
    dmesh, dstats, dstore, dledger = dev_run
    got, want = dstore.export(), PC.reference_store_export(rstore)
    assert np.array_equal(got[0], want[0]), (
        f"block sets differ: {len(got[0])} vs {len(want[0])}")
    for name, a, b in zip("dwc", got[1:], want[1:]):
        assert np.array_equal(a, b), f"{name}: {int((a != b).sum())} voxels differ"
    assert dstats.keyframe_count == rstats.keyframe_count
    assert dstats.corrected_entries == rstats.corrected_entries
    assert dstats.retained_pixels == rstats.retained_pixels
    for name in ("blocks_streamed_in", "blocks_streamed_out", "sphere_relocations"):
        assert getattr(dstats, name) == getattr(rstats, name), name
    for a, b in zip(dstats.frames, rstats.frames):
        assert (a.frame, a.blocks_in, a.blocks_out, a.relocations) == \
            (b.frame, b.blocks_in, b.blocks_out, b.relocations)
    assert dledger.K == rledger.K
    for e, f in zip(dledger.entries, rledger.entries):
        assert (e.kf_id, e.anchor_id) == (f.kf_id, f.anchor_id)
        for p, q in ((e.integrated_pose, f.integrated_pose), (e.target_pose, f.target_pose)):
            assert np.array_equal(p.rotation, q.rotation)
            assert np.array_equal(p.translation, q.translation)
        assert np.array_equal(e.kf.depth.cpu().numpy(), f.kf.depth)
        assert np.array_equal(e.kf.weight.cpu().numpy(), f.kf.weight)
        assert np.array_equal(e.kf.color.cpu().numpy(), f.kf.color)
    assert np.array_equal(dmesh.vertices, rmesh.vertices)
    assert np.array_equal(dmesh.colors, rmesh.colors)
    assert np.array_equal(dmesh.triangles, rmesh.triangles)


@pytest.mark.parametrize("mode,kappa,m", [("consecutive_window", 8, 3),
                                          ("topk_baseline", 8, 3),
                                          ("consecutive_window", 1, 20),
                                          ("off", 5, 10)])
def test_pipeline_matches_reference_bitexact(P, small, mode, kappa, m):
    ref_run, dev_run = _run_pair(P, small, "KF_CONST", kappa, m, mode)
    assert_runs_equal(ref_run, dev_run)


def test_pipeline_dvo_strategy_matches_reference(P, small):
    assert_runs_equal(*_run_pair(P, small, "KF_DVO", 20, 4, "consecutive_window"))


# --- the reference's own pipeline tests (tests/test_pipeline.py:106-240) ---


def _cfg(P, **kw):
    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import volume as V

    kind = kw.pop("kind", "KF_CONST")
    kappa = kw.pop("kappa", 8)
    return P.RunConfig(strategy=KF.KeyframeStrategy(kind=kind, kappa=kappa),
                       volume=V.VolumeConfig(voxel_size=0.02, mu=0.06, stream_radius=5.0), **kw)


def test_kf_const_keyframe_count(P, small):
    _, _, ds = small
    for kappa in (1, 7, 20, 100):
        _, stats, _, _ = P.run_pipeline(ds, _cfg(P, kappa=kappa, reintegration_mode="off"))
        assert stats.keyframe_count == math.ceil(ds.n_frames / kappa)


def test_counters_and_finalize(P, small):
    from paper_1709_03763_b200.geometry import pose_distance

    _, _, ds = small
    mesh, stats, store, ledger = P.run_pipeline(ds, _cfg(P, m=3))
    assert stats.blocks_streamed_in == store.blocks_streamed_in
    assert stats.total("blocks_out") == store.blocks_streamed_out
    assert stats.total("relocations") == store.sphere_relocations
    assert stats.corrected_entries > 0
    assert max(pose_distance(e.integrated_pose, e.target_pose) for e in ledger.entries) < 1e-6
    assert stats.retained_pixels == stats.keyframe_count * 64 * 48
    mesh.validate()


def test_end_state_matches_rebuild(P, small):
    from paper_1709_03763_b200 import volume as V

    _, _, ds = small
    cfg = _cfg(P, m=3)
    _, _, store, ledger = P.run_pipeline(ds, cfg)
    rebuilt = V.TwoTierStore(block_capacity=1 << 16)
    for e in ledger.entries:
        V.stream(rebuilt, e.target_pose.translation, cfg.volume)
        V.integrate(rebuilt, e.kf, e.target_pose, cfg.volume)
    dd, dc, dw = V.compare_volumes(store, rebuilt)
    assert dd < 1e-9 and dc < 1e-9 and dw < 1e-9


def test_kf_dvo_breaks_at_flagged_frames(P, small):
    seq, _, ds = small
    _, stats, _, ledger = P.run_pipeline(ds, _cfg(P, kind="KF_DVO", reintegration_mode="off"))
    flagged = {e.at_frame for e in seq.events if e.dvo_kf_flags}
    starts = {entry.kf.members[0] for entry in ledger.entries}
    assert starts == flagged | {1}
    assert stats.keyframe_count == len(starts)


def test_empty_dataset_rejected(P):
    from paper_1709_03763_b200.errors import EmptyInputError

    with pytest.raises(EmptyInputError):
        P.run_pipeline(PC.DeviceDataset([], None, []), _cfg(P))
    with pytest.raises(ValueError):
        P.RunConfig(m=0)
    with pytest.raises(ValueError):
        P.RunConfig(reintegration_mode="sometimes")


# --- BASELINE configs[0] (C1) at full size ----------------------------------


@pytest.mark.slow
def test_c1_demo_room_end_to_end_bitexact(P):
    """C1: 100 frames 640x480 fused into 20 keyframes (KF_CONST, kappa 5),
    1 cm voxels, the frame-100 correction event re-integrating the ledger with
    correct_window(m=20), finalize, marching cubes -- the device pipeline's
    final volume, ledger, counters and mesh equal the reference's run on the
    same frames bit for bit.  Timings go to
    gpurun_out/c1_parity.json (tools/bench_c1.py is the measurement)."""
    import refusion.keyframe_fusion as RKF
    import refusion.pipeline as RP
    import refusion.volume as RV

    from paper_1709_03763_b200 import keyframe_fusion as KF
    from paper_1709_03763_b200 import volume as V

    t0 = time.perf_counter()
    seq = PC.c1_sequence()
    t_render = time.perf_counter() - t0
    rds, dds = PC.reference_dataset(seq), PC.device_dataset(seq)
    vol = dict(voxel_size=0.01, mu=0.06, stream_radius=6.0, hash_buckets=1 << 16)
    rcfg = RP.RunConfig(strategy=RKF.KeyframeStrategy(kind="KF_CONST", kappa=5), m=20,
                        volume=RV.VolumeConfig(**vol), reintegration_mode="consecutive_window")
    dcfg = P.RunConfig(strategy=KF.KeyframeStrategy(kind="KF_CONST", kappa=5), m=20,
                       volume=V.VolumeConfig(**vol), reintegration_mode="consecutive_window",
                       block_capacity=1 << 17)
    t0 = time.perf_counter()
    ref_run = RP.run_pipeline(rds, rcfg)
    t_ref = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev_run = P.run_pipeline(dds, dcfg)
    t_dev = time.perf_counter() - t0
    assert ref_run[1].keyframe_count == 20
    assert ref_run[1].corrected_entries >= 19
    assert_runs_equal(ref_run, dev_run)
    os.makedirs("gpurun_out", exist_ok=True)
    import json

    with open("gpurun_out/c1_parity.json", "w") as fh:
        json.dump({"render_s": t_render, "reference_run_s": t_ref, "device_run_s": t_dev,
                   "reference_correct_ms": ref_run[1].correct_ms,
                   "device_correct_ms": dev_run[1].correct_ms,
                   "corrected_entries": ref_run[1].corrected_entries,
                   "blocks": int(len(dev_run[2].export()[0]))}, fh, indent=1)
