"""Multi-GPU sharding of shading-point queries and of the per-light build.

Every query is independent given the replicated inputs (density volume,
transmittance feature volume, phase table, templates, network weights), so the
image is split into square tiles dealt round-robin to the ranks (one process per
GPU); each rank runs the fused query on its tiles and the per-tile radiance is
gathered once per frame — the only exchange of the path. No collective touches
the data path itself (weak scaling when every rank owns a fixed number of tiles).

The per-light build (graded transmittance + combiner) is needed whole on every GPU but is
embarrassingly parallel per voxel: each rank builds a z-slab of the level-0 transmittance
feature volume (sf_build_transmittance_slab: level 0 marched for the slab plus a halo,
coarser levels redundantly) and one all_gather assembles the volume on every rank
(build_tvol_sharded) — bit-identical to the single-GPU build.

Works with any torch.distributed backend: NCCL over NVLink on the B200 box, gloo
for the CPU tests (tests/test_sharding_gloo.py).
"""
from __future__ import annotations

import numpy as np


def tile_ids(width: int, height: int, tile: int):
    """Row-major tile grid; returns (n_tiles_x, n_tiles_y)."""
    return (width + tile - 1) // tile, (height + tile - 1) // tile


def rank_pixels(width: int, height: int, tile: int, rank: int, world: int) -> np.ndarray:
    """Pixel indices (row-major, y * width + x) owned by `rank`: tiles t with t % world == rank,
    each tile's pixels in row-major order, tiles in increasing order."""
    ntx, nty = tile_ids(width, height, tile)
    out = []
    for t in range(rank, ntx * nty, world):
        ty, tx = divmod(t, ntx)
        y0, x0 = ty * tile, tx * tile
        ys = np.arange(y0, min(y0 + tile, height))
        xs = np.arange(x0, min(x0 + tile, width))
        out.append((ys[:, None] * width + xs[None, :]).reshape(-1))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def shard_sizes(width: int, height: int, tile: int, world: int):
    return [len(rank_pixels(width, height, tile, r, world)) for r in range(world)]


def gather_radiance(local, width: int, height: int, tile: int, rank: int, world: int, group=None):
    """Assemble the full [height*width, 3] radiance on every rank from per-rank tiles.

    `local` is a torch tensor [n_local, 3] (CUDA with NCCL, CPU with gloo) in the
    pixel order of rank_pixels(..., rank, world). Ranks own different pixel counts
    at the image border, so shards are padded to the largest before all_gather.
    """
    import torch
    import torch.distributed as dist

    sizes = shard_sizes(width, height, tile, world)
    pad = max(sizes)
    dev = _comm_device(local.device, group)
    buf = torch.zeros((pad, local.shape[1]), dtype=local.dtype, device=dev)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    full = torch.empty((width * height, local.shape[1]), dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = torch.as_tensor(rank_pixels(width, height, tile, r, world), device=local.device)
        full[idx] = parts[r][: sizes[r]].to(local.device)
    return full


def _comm_device(dev, group=None):
    """Where a collective's buffers live: the tensor's device for NCCL, the host for gloo (CPU
    tests, and the multi-process GPU tests that share one device)."""
    import torch
    import torch.distributed as dist

    return torch.device("cpu") if dist.get_backend(group) == "gloo" else dev


def query_image(eval_fn, queries, width: int, height: int, tile: int, rank: int, world: int, group=None):
    """Run `eval_fn(rows) -> [n, 3]` on this rank's tiles of the per-pixel query rows
    ([height*width, 9]) and gather the image. `eval_fn` is the fused GPU query
    (paper_2401_14051_b200.query bound to a scene/net) in production, anything with the
    same contract in tests."""
    import torch

    mine = rank_pixels(width, height, tile, rank, world)
    local = eval_fn(queries[mine])
    if not isinstance(local, torch.Tensor):
        local = torch.as_tensor(np.ascontiguousarray(local))
    return gather_radiance(local, width, height, tile, rank, world, group)


def z_slabs(nz: int, world: int):
    """Contiguous z-row ranges [z0, z1) per rank, sizes differing by at most one row."""
    base, extra = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((z, z + n))
        z += n
    return out


def gather_slabs(local, nz: int, rank: int, world: int, group=None):
    """All-gather per-rank z-slabs [z1-z0, ny, nx] into the full [nz, ny, nx] volume on every rank
    (slabs padded to the largest; NCCL over NVLink on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    slabs = z_slabs(nz, world)
    pad = max(z1 - z0 for z0, z1 in slabs)
    buf = torch.zeros((pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=_comm_device(local.device, group))
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: z1 - z0] for r, (z0, z1) in enumerate(slabs)], dim=0).to(local.device)


def build_tvol_sharded(pyramid, light, rank: int, world: int, weights=None, cfg=None, group=None, fast=False):
    """build_transmittance_volume with the level-0 work split by z-slab over the ranks of `group`;
    returns the TransmittanceFeatureVolume (identical on every rank)."""
    import torch

    from . import api

    g0 = pyramid.level(0)
    nx, ny, nz = g0.dims
    z0, z1 = z_slabs(nz, world)[rank]
    local = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device="cuda")
    api.build_transmittance_slab(pyramid, light, z0, z1, weights, cfg, out=local, fast=fast)
    full = gather_slabs(local, nz, rank, world, group)
    return api.TransmittanceFeatureVolume.from_values(full.contiguous(), g0.voxel_size(), g0.origin(), light, weights)


def relight_sharded(scene, pyramid, light, rank: int, world: int, weights=None, cfg=None, group=None, fast=False,
                    stream=None):
    """Scene.relight with the per-light build split by z-slab over the ranks of `group`: every rank
    builds its slab (sf_build_transmittance_slab, bit-identical rows), one all_gather assembles the
    volume straight into the scene's own storage, and the query records are refreshed — the
    result is bit-identical to scene.relight(pyramid, light) on every rank."""
    import torch
    import torch.distributed as dist

    from . import api

    g0 = pyramid.level(0)
    nx, ny, nz = g0.dims
    slabs = z_slabs(nz, world)
    pad = max(z1 - z0 for z0, z1 in slabs)
    z0, z1 = slabs[rank]
    dev = torch.device("cuda", torch.cuda.current_device())
    even = all(z1_ - z0_ == pad for z0_, z1_ in slabs)
    store = scene.tvol_storage()
    if world > 1 and dist.get_backend(group) == "gloo":  # host-staged gather (CPU collectives)
        local = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=dev)
        api.build_transmittance_slab(pyramid, light, z0, z1, weights, cfg, out=local, fast=fast, stream=stream)
        torch.cuda.synchronize()
        store.copy_(gather_slabs(local.cpu(), nz, rank, world, group))
        scene.commit_tvol(light, stream=stream)
        return scene
    if even:
        # equal slabs: gather in place, rank r's rows land at [r*pad, (r+1)*pad)
        local = store[z0:z1]
        api.build_transmittance_slab(pyramid, light, z0, z1, weights, cfg, out=local, fast=fast, stream=stream)
        if world > 1:
            dist.all_gather_into_tensor(store, local, group=group)  # in place: local is store's slice
    else:
        buf = torch.empty((pad, ny, nx), dtype=torch.float32, device=dev)
        api.build_transmittance_slab(pyramid, light, z0, z1, weights, cfg, out=buf[: z1 - z0], fast=fast, stream=stream)
        full = torch.empty((world * pad, ny, nx), dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(full, buf, group=group)
        for r, (a, b) in enumerate(slabs):
            store[a:b].copy_(full[r * pad: r * pad + (b - a)])
    scene.commit_tvol(light, stream=stream)
    return scene
