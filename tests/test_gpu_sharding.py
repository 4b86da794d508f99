"""The multi-GPU path on the real kernels: two processes (world 2, gloo, host-staged collectives)
on the one visible B200 run sharding.relight_sharded (each rank builds a z-slab of the
transmittance volume with sf_build_transmittance_slab, the slabs are all-gathered into the
scene's own storage) and sharding.query_image (each rank queries its 32x32 image tiles with the
fused query, the radiance tiles are all-gathered). The image and the volume must be
bit-identical to the single-process Scene.relight + query (results do not depend
on how the work is split, inc/parallel.h:16-17). No rank's kernels wait on another's: the
collectives run on the host, so two ranks on one device is a valid stand-in for two GPUs here."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W, H, TILE = 64, 48, 16


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(precision_name):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import paper_2401_14051_b200 as sf
    from paper_2401_14051_b200 import scenes
    vol = scenes.procedural_cloud(64, 4)
    g = sf.DensityGrid.from_array(vol, 2.0 / 64, (-1.0, -1.0, -1.0))
    pyr = sf.DensityPyramid(g)
    data = os.path.join(ROOT, "paper_2401_14051_b200", "data")
    d = sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl"))
    h = sf.load_template(os.path.join(data, "highlight_seed8.vtmpl"))
    light = scenes.rotating_light(3, 32)
    scene = sf.Scene(g, sf.build_transmittance_volume(pyr, scenes.LIGHT), d, h, sf.PhaseModel.hg(0.7),
                     sf.PhaseTable(64, 128, 32, 16))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((0.7,), (0.99,) * 3)
    rows = scenes.draw_centers(vol, W * H, 9, light)
    prec = sf.BF16 if precision_name == "bf16" else sf.FP32
    fast = prec == sf.BF16

    def eval_fn(r):
        rd = torch.from_numpy(np.ascontiguousarray(r)).cuda()
        F = torch.empty((len(r), 3), dtype=torch.float64, device="cuda")
        sf.query(scene, net, med, rd, prec, F_out=F)
        return F
    return sf, scene, pyr, light, rows, eval_fn, fast


def _worker(rank, world, port, precision_name, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sf, scene, pyr, light, rows, eval_fn, fast = _setup(precision_name)
    from paper_2401_14051_b200 import sharding
    sharding.relight_sharded(scene, pyr, light, rank, world, fast=fast)
    img = sharding.query_image(eval_fn, rows, W, H, TILE, rank, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "img.npy"), img.cpu().numpy())
        np.save(os.path.join(out_dir, "tvol.npy"), scene.tvol_storage().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("precision_name", ["fp32", "bf16"])
def test_two_ranks_bit_identical(tmp_path, precision_name):
    import torch
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, precision_name, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    sf, scene, pyr, light, rows, eval_fn, fast = _setup(precision_name)
    scene.relight(pyr, light, fast=fast)
    want = eval_fn(rows).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(np.load(tmp_path / "tvol.npy"), scene.tvol_storage().cpu().numpy())
    assert np.array_equal(np.load(tmp_path / "img.npy"), want)
