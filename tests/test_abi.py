"""CPU checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/refusion_b200.h declares, and the pure-host pieces of
the volume API follow the reference (no device calls)."""

import json
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "refusion_b200.h")
GOLDEN = json.load(open(os.path.join(REPO, "tests", "golden", "volume_golden.json")))


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:rf_status|int64_t|int32_t|const char \*)\s*(rf_\w+)\(",
                                 text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for name in ("rf_volume_create", "rf_integrate", "rf_deintegrate", "rf_correct",
                 "rf_stream", "rf_footprint", "rf_fuse_block", "rf_export_blocks"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_1709_03763_b200 import _lib

    lib = _lib.load_library()
    syms = declared_symbols()
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table and header diverge"
    for name in syms:
        assert getattr(lib, name) is not None


def test_library_is_sm100a_cubin():
    from paper_1709_03763_b200 import _lib

    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_block_hash_host_matches_golden():
    from paper_1709_03763_b200 import volume as V

    for coord, buckets, want in GOLDEN["hash"]:
        assert V.block_hash(coord, buckets) == want


def test_block_hash_c_abi_matches_golden():
    from paper_1709_03763_b200 import _lib

    lib = _lib.load_library()  # pure host function, no device touched
    for coord, buckets, want in GOLDEN["hash"]:
        assert lib.rf_block_hash(*coord, buckets) == want


def test_pack_roundtrip_extremes():
    from paper_1709_03763_b200 import volume as V

    coords = [(0, 0, 0), (-1, -1, -1), ((1 << 20) - 1, -(1 << 20), 5), (123, -456, 789)]
    keys = V.pack_keys(coords)
    assert V.keys_to_coords(keys) == coords
    assert (np.diff(V.pack_keys(sorted(coords))) > 0).all()  # packing preserves order


def test_volume_config_validation():
    from paper_1709_03763_b200 import volume as V

    with pytest.raises(ValueError):
        V.VolumeConfig(voxel_size=0.0)
    with pytest.raises(ValueError):
        V.VolumeConfig(voxel_size=0.01, mu=0.015)
    with pytest.raises(ValueError):
        V.VolumeConfig(voxel_size=0.01, mu=0.06, stream_radius=0.05)
    with pytest.raises(ValueError):
        V.VolumeConfig(hash_buckets=0)


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_1709_03763_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError):
        _lib.lib()


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1709_03763_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "oracle" not in text.replace("oracle/", ""), f
