"""CPU, world_size 2 over gloo: the tile-sharded query path assembles exactly the
single-process image. The per-rank evaluator is the oracle (test
infrastructure) on a small scene; on the B200 box the same code runs the fused
GPU query over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_14051_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from conftest import DATA, ORIGIN
    from oracle.oracle import BackboneCfg, Oracle, PhaseModel, load_vtmpl
    from paper_2401_14051_b200 import scenes
    O = Oracle()
    vol = scenes.procedural_cloud(16, 3)
    vs = 2.0 / 16
    tvol = O.build_tvol(vol, vs, ORIGIN, np.array(scenes.LIGHT))
    sc = O.make_scene(vol, tvol, vs, ORIGIN, load_vtmpl(os.path.join(DATA, "diffuse_seed7.vtmpl")),
                      load_vtmpl(os.path.join(DATA, "highlight_seed8.vtmpl")), PhaseModel.hg(0.7),
                      O.phase_table(9, 17, 5, 8))
    cfg = BackboneCfg(seed=0)
    params = O.backbone_init(cfg)

    def eval_fn(rows):
        feats = O.features(sc, rows)
        _, F = O.predict(cfg, params, feats, scenes.config_rows(rows, [0.7], [0.99] * 3))
        return F

    return vol, eval_fn


def _worker(rank, world, port, width, height, tile, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2401_14051_b200 import scenes
    vol, eval_fn = _scene()
    rows = scenes.draw_centers(vol, width * height, 5, scenes.LIGHT)
    img = sharding.query_image(eval_fn, rows, width, height, tile, rank, world)
    if rank == 0:
        np.save(out_path, img.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_rank_pixels_partition():
    for (w, h, t, n) in ((10, 7, 4, 2), (16, 16, 8, 4), (5, 3, 8, 3), (64, 64, 16, 8)):
        parts = [sharding.rank_pixels(w, h, t, r, n) for r in range(n)]
        allp = np.concatenate(parts)
        assert len(allp) == w * h and len(np.unique(allp)) == w * h
        assert sorted(allp.tolist()) == list(range(w * h))


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process(tmp_path):
    width, height, tile = 6, 5, 4
    out = str(tmp_path / "img.npy")
    mp.spawn(_worker, args=(2, _free_port(), width, height, tile, out), nprocs=2, join=True)
    img = np.load(out)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from paper_2401_14051_b200 import scenes
    vol, eval_fn = _scene()
    rows = scenes.draw_centers(vol, width * height, 5, scenes.LIGHT)
    ref = eval_fn(rows)
    assert np.array_equal(img, ref)


# ---- per-light build sharded by z-slab -------------------------------
def test_z_slabs_partition():
    for nz, world in ((16, 2), (17, 3), (5, 8), (128, 8), (1, 4)):
        slabs = sharding.z_slabs(nz, world)
        assert len(slabs) == world and slabs[0][0] == 0 and slabs[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
        sizes = [z1 - z0 for z0, z1 in slabs]
        assert max(sizes) - min(sizes) <= 1


def _slab_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import ORIGIN
    from oracle.oracle import Oracle
    from paper_2401_14051_b200 import scenes
    vol = scenes.procedural_cloud(16, 3)
    # per-rank slab from the oracle (stand-in for sf_build_transmittance_slab on a GPU)
    full = Oracle().build_tvol(vol, 2.0 / 16, ORIGIN, np.array(scenes.LIGHT)).reshape(16, 16, 16)
    z0, z1 = sharding.z_slabs(16, world)[rank]
    got = sharding.gather_slabs(torch.from_numpy(np.ascontiguousarray(full[z0:z1])), 16, rank, world)
    if rank == 0:
        np.save(out_path, np.stack([got.numpy(), full]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_three_rank_gloo_slab_gather(tmp_path):
    out = str(tmp_path / "tvol.npy")
    mp.spawn(_slab_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    got, full = np.load(out)
    assert np.array_equal(got, full)
