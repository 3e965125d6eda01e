"""B200-native surface-correction hot path of arXiv 1709.03763 (`refusion`).

Host modules mirror the reference's plugin/operator API:
  kernels        -- the kernel backend plugin point (BACKEND, fuse_block)
  volume         -- voxel-hashed TSDF in HBM (integrate / deintegrate / stream / GC)
  reintegration  -- ledger + window / top-k correction scheduler
  keyframe_fusion-- per-pixel depth / colour fusion into keyframes
All compute runs in librefusion_b200.so (sm_100a CUDA, C ABI in
include/refusion_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
