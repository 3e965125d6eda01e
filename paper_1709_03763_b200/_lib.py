"""ctypes binding of the C ABI in include/refusion_b200.h.

The shared library ``librefusion_b200.so`` (built in-tree by
``__graft_entry__.build()``) holds every CUDA kernel of the hot path.  There
is no fallback: if the library or a CUDA device is missing, ``lib()`` raises
so that nothing silently runs on the CPU.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RF_LIB_PATH") or os.path.join(_HERE, "librefusion_b200.so")

RF_OK = 0
RF_STREAMING_CONTRACT = 1
RF_INCONSISTENT = 2
RF_CAPACITY = 3
RF_INVALID_ARG = 4
RF_CUDA = 5

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_int32_p = ctypes.POINTER(ctypes.c_int32)


class RfConfig(ctypes.Structure):
    _fields_ = [
        ("voxel_size", ctypes.c_double),
        ("mu", ctypes.c_double),
        ("stream_radius", ctypes.c_double),
        ("hash_buckets", ctypes.c_int64),
        ("block_capacity", ctypes.c_int64),
        ("device", ctypes.c_int32),
        ("shard_rank", ctypes.c_int32),
        ("shard_count", ctypes.c_int32),
        ("max_pixels", ctypes.c_int32),
    ]


class RfPose(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3)]


class RfKfView(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_void_p),
        ("weight", ctypes.c_void_p),
        ("color", ctypes.c_void_p),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("ready_event", ctypes.c_void_p),
        ("memo_tag", ctypes.c_uint64),
        ("planes_on_host", ctypes.c_int32),
    ]


class RfOpResult(ctypes.Structure):
    _fields_ = [
        ("blocks_touched", ctypes.c_int64),
        ("voxels_updated", ctypes.c_int64),
        ("n_new", ctypes.c_int64),
    ]


class RfStreamResult(ctypes.Structure):
    _fields_ = [
        ("streamed_in", ctypes.c_int64),
        ("streamed_out", ctypes.c_int64),
        ("relocated", ctypes.c_int64),
    ]


class RfCounters(ctypes.Structure):
    _fields_ = [
        ("blocks_streamed_in", ctypes.c_int64),
        ("blocks_streamed_out", ctypes.c_int64),
        ("sphere_relocations", ctypes.c_int64),
        ("block_count", ctypes.c_int64),
        ("active_count", ctypes.c_int64),
        ("has_center", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("last_center", ctypes.c_double * 3),
    ]


class RfWindowResult(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("failed_entry", ctypes.c_int32),
        ("failed_phase", ctypes.c_int32),
        ("failed_window", ctypes.c_int32),
        ("n_corrected", ctypes.c_int64),
        ("voxels_updated", ctypes.c_int64),
        ("blocks_touched", ctypes.c_int64),
        ("n_new", ctypes.c_int64),
        ("gc_freed", ctypes.c_int64),
    ]


class RfProfile(ctypes.Structure):
    _fields_ = [
        ("fuse_launches", ctypes.c_int64),
        ("fuse_ms", ctypes.c_double),
        ("check_launches", ctypes.c_int64),
        ("check_ms", ctypes.c_double),
        ("footprint_launches", ctypes.c_int64),
        ("footprint_ms", ctypes.c_double),
        ("voxels_updated", ctypes.c_int64),
        ("pixels", ctypes.c_int64),
        ("blocks_touched", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("other_launches", ctypes.c_int64),
        ("other_ms", ctypes.c_double),
        ("integrate_launches", ctypes.c_int64),
        ("integrate_ms", ctypes.c_double),
        ("integrate_voxels", ctypes.c_int64),
        ("integrate_pixels", ctypes.c_int64),
        ("removal_ops", ctypes.c_int64),
        ("removal_ms", ctypes.c_double),
        ("removal_voxels", ctypes.c_int64),
        ("removal_pixels", ctypes.c_int64),
    ]


class RfMemberView(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_void_p),
        ("w_map", ctypes.c_void_p),
        ("color", ctypes.c_void_p),
        ("blur_weight", ctypes.c_void_p),
        ("rel", RfPose),
    ]


class RfSynthPrim(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("center", ctypes.c_double * 3),
        ("size", ctypes.c_double * 3),
        ("albedo", ctypes.c_double * 3),
    ]


class RfSynthRefParams(ctypes.Structure):
    _fields_ = [
        ("z_max", ctypes.c_double),
        ("tol", ctypes.c_double),
        ("ambient", ctypes.c_double),
        ("diffuse", ctypes.c_double),
        ("neg_light", ctypes.c_double * 3),
        ("normal_eps", ctypes.c_double),
        ("steps", ctypes.c_int32),
        ("gemm_order", ctypes.c_int32),
        ("gemv_order", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


class RfSynthGauss(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double * 64), ("r", ctypes.c_int32), ("_pad", ctypes.c_int32)]


_vp = ctypes.c_void_p
_S = ctypes.c_int  # rf_status

# name -> (restype, argtypes); exactly the symbols include/refusion_b200.h declares
SIGNATURES = {
    "rf_volume_create": (_S, [ctypes.POINTER(RfConfig), ctypes.POINTER(_vp)]),
    "rf_volume_destroy": (_S, [_vp]),
    "rf_set_cuda_stream": (_S, [_vp, _vp]),
    "rf_last_error": (ctypes.c_char_p, [_vp]),
    "rf_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rf_block_hash": (ctypes.c_int64, [ctypes.c_int64] * 4),
    "rf_key_owner": (ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32]),
    "rf_stream": (_S, [_vp, c_double_p, ctypes.POINTER(RfStreamResult)]),
    "rf_footprint": (_S, [_vp, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose), c_int64_p,
                          ctypes.c_int64, c_int64_p]),
    "rf_allocate": (_S, [_vp, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose), c_int64_p,
                         ctypes.c_int64, c_int64_p]),
    "rf_integrate": (_S, [_vp, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose),
                          ctypes.POINTER(RfOpResult), c_int64_p, ctypes.c_int64]),
    "rf_deintegrate": (_S, [_vp, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose),
                            ctypes.POINTER(RfOpResult)]),
    "rf_correct": (_S, [_vp, ctypes.c_int32, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose),
                        ctypes.POINTER(RfPose), c_double_p, ctypes.POINTER(RfWindowResult)]),
    "rf_correct_windows": (_S, [_vp, ctypes.c_int32, c_int32_p, ctypes.POINTER(RfKfView),
                                ctypes.POINTER(RfPose), ctypes.POINTER(RfPose), c_double_p,
                                ctypes.POINTER(RfWindowResult)]),
    "rf_garbage_collect": (_S, [_vp, c_int64_p]),
    "rf_total_weight": (_S, [_vp, c_double_p]),
    "rf_counters_get": (_S, [_vp, ctypes.POINTER(RfCounters)]),
    "rf_export_blocks": (_S, [_vp, c_int64_p, c_double_p, ctypes.c_int64, c_int64_p]),
    "rf_import_blocks": (_S, [_vp, c_int64_p, c_double_p, ctypes.c_int64]),
    "rf_snapshot_records": (_S, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, c_int64_p]),
    "rf_grid_index_create": (_S, [_vp, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(_vp),
                                  _vp]),
    "rf_grid_index_query": (_S, [_vp, _vp, ctypes.c_int64, _vp, _vp]),
    "rf_grid_index_destroy": (_S, [_vp]),
    "rf_nn_min_d2": (_S, [c_double_p, ctypes.c_int64, c_double_p, ctypes.c_int64, c_double_p,
                          _vp]),
    "rf_marching_cubes_welded": (_S, [_vp, ctypes.c_double, c_double_p, c_double_p, c_int64_p,
                                      ctypes.c_int64, ctypes.c_int64, c_int64_p, c_int64_p]),
    "rf_marching_cubes": (_S, [_vp, c_double_p, c_double_p, c_int64_p, ctypes.c_int64,
                               ctypes.c_int64, c_int64_p, c_int64_p]),
    "rf_read_blocks": (_S, [_vp, c_int64_p, ctypes.c_int64, c_double_p, c_int32_p]),
    "rf_fuse_block": (_S, [c_double_p, c_double_p, c_double_p] + [ctypes.c_double] * 4
                      + [c_double_p] + [ctypes.c_double] * 7 + [ctypes.c_int32] * 2
                      + [c_double_p] * 3 + [ctypes.c_double] * 2
                      + [ctypes.c_int32, c_int32_p]),
    "rf_depth_weight": (_S, [_vp, ctypes.c_int32, ctypes.c_int32] + [ctypes.c_double] * 5
                        + [ctypes.c_int32, _vp, _vp]),
    "rf_normal_map": (_S, [_vp, ctypes.c_int32, ctypes.c_int32] + [ctypes.c_double] * 4
                      + [_vp, _vp]),
    "rf_depth_sample_weight_normals": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32]
                                       + [ctypes.c_double] * 4 + [_vp, _vp]),
    "rf_fuse_depth": (_S, [_vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32]
                      + [ctypes.c_double] * 4 + [ctypes.POINTER(RfPose), ctypes.c_int32, _vp]),
    "rf_fuse_frame": (_S, [_vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32]
                      + [ctypes.c_double] * 4 + [ctypes.POINTER(RfPose), ctypes.c_int32,
                                                 ctypes.c_double, c_double_p, ctypes.c_int32,
                                                 ctypes.c_double, _vp, _vp, _vp, _vp, _vp]),
    "rf_unsharp_mask": (_S, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_double_p,
                             ctypes.c_int32, ctypes.c_double, _vp, _vp]),
    "rf_grayscale": (_S, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "rf_blurriness": (_S, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "rf_color_prep": (_S, [_vp, ctypes.c_int32, ctypes.c_int32, c_double_p, ctypes.c_int32,
                           ctypes.c_double, _vp, _vp, _vp]),
    "rf_fuse_color": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32] + [ctypes.c_double] * 4
                      + [ctypes.c_int32, ctypes.POINTER(RfMemberView), ctypes.c_double,
                         ctypes.c_int32, _vp, _vp, _vp]),
    "rf_selftest_division": (_S, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                  ctypes.POINTER(ctypes.c_uint64)]),
    "rf_selftest_projection": (_S, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.POINTER(ctypes.c_uint64)]),
    "rf_set_memo_budget": (_S, [_vp, ctypes.c_int64]),
    "rf_route_setup": (_S, [_vp, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(_vp),
                            ctypes.POINTER(ctypes.c_uint64)]),
    "rf_route_connect": (_S, [_vp, ctypes.POINTER(_vp)]),
    "rf_route_ipc_handle": (_S, [_vp, _vp]),
    "rf_route_ipc_open": (_S, [_vp, _vp]),
    "rf_route": (_S, [_vp, ctypes.c_int32, ctypes.POINTER(RfKfView), ctypes.POINTER(RfPose),
                      c_double_p]),
    "rf_shard_sync_setup": (_S, [_vp, ctypes.c_int32, ctypes.POINTER(_vp),
                                 ctypes.POINTER(ctypes.c_uint64)]),
    "rf_shard_sync_connect": (_S, [_vp, ctypes.POINTER(_vp)]),
    "rf_shard_sync_ipc_handle": (_S, [_vp, _vp]),
    "rf_shard_sync_ipc_open": (_S, [_vp, _vp]),
    "rf_reserve": (_S, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "rf_profile_begin": (_S, [_vp]),
    "rf_profile_end": (_S, [_vp, ctypes.POINTER(RfProfile)]),
    "rf_mesh_connect": (_S, [_vp, ctypes.POINTER(_vp), ctypes.c_int32]),
    "rf_mesh_ipc_handle": (_S, [_vp, _vp]),
    "rf_mesh_ipc_open": (_S, [_vp, _vp, c_int64_p]),
    "rf_mesh_blocks": (_S, [_vp, c_int64_p, c_int64_p, c_int64_p, ctypes.c_int64,
                            ctypes.POINTER(ctypes.c_int64)]),
    "rf_synth_depth": (_S, [_vp, ctypes.c_int32, ctypes.POINTER(RfPose)] + [ctypes.c_double] * 4
                       + [ctypes.c_int32] * 2 + [ctypes.POINTER(RfSynthRefParams), _vp, _vp]),
    "rf_synth_color": (_S, [_vp, ctypes.c_int32, ctypes.POINTER(RfPose)] + [ctypes.c_double] * 4
                       + [ctypes.c_int32] * 2 + [ctypes.POINTER(RfSynthRefParams), _vp, _vp,
                                                 _vp]),
    "rf_synth_blur": (_S, [_vp, _vp, ctypes.c_int32, ctypes.c_int32,
                           ctypes.POINTER(RfSynthGauss), _vp]),
}

_lib = None


def load_library(path=LIB_PATH):
    """Load and type the shared library without touching any CUDA device."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The typed library; raises if it is absent or no CUDA device exists."""
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_1709_03763_b200 needs a CUDA device (B200); no CPU fallback exists"
            )
        _lib = load_library()
    return _lib
