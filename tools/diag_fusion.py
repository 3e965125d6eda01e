"""Host/device profile of fuse_depth on corridor frames (cProfile of the
Python path; the wall time per frame).  Diagnostic only."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from paper_1709_03763_b200 import keyframe_fusion as KF, synth as SY
torch.cuda.set_device(0)
traj = SY.corridor_trajectory(B.N_FRAMES)[:30]
rend = SY.Renderer(SY.corridor_scene(), SY.DEFAULT_INTRINSICS, device=0)
frames = [rend.render(traj[i], seed=7000 + i) for i in range(30)]
intr = SY.DEFAULT_INTRINSICS
KF.detect_blas_order()
def run(n0, n1):
    kf = None
    for i in range(n0, n1):
        fo = KF.FrameObservation(i + 1, frames[i][1], frames[i][0], traj[i])
        if kf is None: kf = KF.new_keyframe(fo, intr)
        KF.fuse_depth(kf, fo)
    torch.cuda.synchronize()
run(0, 5)
t = time.perf_counter(); run(5, 10); print("wall per frame ms", (time.perf_counter() - t) / 5 * 1e3)
cProfile.run("run(10, 30)", "/tmp/fp.out")
pstats.Stats("/tmp/fp.out").sort_stats("cumulative").print_stats(18)
