"""Routed footprints across PROCESSES (rf_route_ipc_handle / rf_route_ipc_open,
connect_shards_distributed): two ranks on the one device of this run, a
gloo process group for the barrier and the status agreement, CUDA IPC for the
inboxes -- the multi-GPU code path with both shards on one GPU.  The union of
the ranks' volumes must equal a single volume bit for bit, and an error on
the shards must surface on both ranks.  Each rank's marching cubes reads its
cross-shard neighbours from the other process's pool (rf_mesh_ipc_open): the
ranks' meshes merged in block order equal the single volume's mesh."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    import scenarios as S

    rng = np.random.default_rng(21)
    frames = [S.wall_frame(S.QVGA_INTR, 1.1 + 0.2 * i, rng=rng, tilt=0.25 * i, noise=0.0015,
                           holes=0.05) for i in range(3)]
    old = [S.SPose(S.rot_z(0.05 * i), [0.02 * i, 0.0, 0.1]) for i in range(3)]
    new = [S.SPose(S.rot_z(0.05 * i + 0.01), [0.02 * i + 0.02, 0.01, 0.1]) for i in range(3)]
    return frames, old, new


def _run(V, S, store, cfg, frames, old, new):
    for f, p in zip(frames, old):
        V.stream(store, p.translation, cfg)
        V.integrate(store, f, p, cfg)
    ents = [S.Entry(f, o.copy(), n.copy()) for f, o, n in zip(frames, old, new)]
    V.correct_windows(store, [[e] for e in ents], cfg, np.array([0.2, 0.0, 0.1]))


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import scenarios as S
    from paper_1709_03763_b200 import volume as V
    from paper_1709_03763_b200.errors import StreamingContractError

    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    store = V.TwoTierStore(block_capacity=1 << 16, shard_rank=rank, shard_count=world)
    V.connect_shards_distributed(store, cfg, image=(320, 240))
    frames, old, new = _scene()
    _run(V, S, store, cfg, frames, old, new)
    keys, d, w, c = store.export()
    from paper_1709_03763_b200 import meshing as M

    dist.barrier()  # both volumes final before either meshes (peer reads)
    mesh = M.marching_cubes(store, cfg)
    mk, mnv, mnt = M.mesh_blocks(store, cfg)
    dist.barrier()  # the peer's pool stays alive until both have meshed
    # a contract error raised on every rank
    err = "none"
    try:
        V.stream(store, np.array([7.5, 0.0, 0.0]), cfg)
        V.integrate(store, frames[0], old[0], cfg)
    except StreamingContractError:
        err = "contract"
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), keys=keys, d=d, w=w, c=c, err=err,
             mv=mesh.vertices, mc=mesh.colors, mt=mesh.triangles, mk=mk, mnv=mnv, mnt=mnt)
    dist.barrier()
    store.close()
    dist.destroy_process_group()


def test_two_process_ipc_routed_equals_single(tmp_path):
    import torch

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    import scenarios as S
    from paper_1709_03763_b200 import volume as V

    torch.cuda.set_device(0)
    cfg = V.VolumeConfig(voxel_size=0.005, mu=0.06, stream_radius=6.0, hash_buckets=1 << 15)
    single = V.TwoTierStore(block_capacity=1 << 16)
    frames, old, new = _scene()
    _run(V, S, single, cfg, frames, old, new)
    want = single.export()
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    keys = np.concatenate([p["keys"] for p in parts])
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(keys[order], want[0])
    for i, name in ((1, "d"), (2, "w"), (3, "c")):
        assert np.array_equal(np.concatenate([p[name] for p in parts])[order], want[i])
    assert all(str(p["err"]) == "contract" for p in parts)
    from paper_1709_03763_b200 import meshing as M

    got = M.merge_shard_meshes([(M.TriangleMesh(p["mv"], p["mc"], p["mt"]), p["mk"], p["mnv"],
                                 p["mnt"]) for p in parts])
    ref = M.marching_cubes(single, cfg)
    assert ref.n_triangles > 100
    assert np.array_equal(got.vertices, ref.vertices)
    assert np.array_equal(got.colors, ref.colors)
    assert np.array_equal(got.triangles, ref.triangles)
