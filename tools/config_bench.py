"""Sustained throughput of configurations C3 and C5 on one GPU, with the
per-stage device breakdown; writes one JSON line per config.

C5: 256^3 static noise volume, light rotated about +Y, the transmittance volume rebuilt
    every frame, 1280x720 = 921,600 queries per frame (bf16); sustained queries/s over the
    frames INCLUDING the per-frame build. Stages: pyramid (once), transmittance, sample+sort,
    backbone.
C3: 256^3 smoke plume (70% empty), 4 lights (tvol rebuilt per light), 512x512 = 262,144
    queries per light, F = sum_l I_l F_l.

usage: python tools/config_bench.py [--frames 8] [--grid 256]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_14051_b200 as sf  # noqa: E402
from paper_2401_14051_b200 import configs, scenes  # noqa: E402
from paper_2401_14051_b200._lib import profile_read  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=8)
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--c4", action="store_true", help="also run C4 (512^3 per-voxel albedo/g, 1920x1080 queries)")
ap.add_argument("--only-c4", action="store_true")
ap.add_argument("--exact-build", action="store_true", help="FP64 reference march for the tvol (default: FP32 march)")
a = ap.parse_args()
FAST = not a.exact_build
N = a.grid
data = os.path.join(os.path.dirname(sf.__file__), "data")
dt = sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl"))
ht = sf.load_template(os.path.join(data, "highlight_seed8.vtmpl"))
table = sf.PhaseTable(64, 128, 32, 16)
net = sf.make_backbone(sf.BackboneConfig(seed=0))
stream = torch.cuda.current_stream()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def stage_split():
    st = profile_read()
    return {k: round(v[0], 3) for k, v in st.items() if v[1]}


def run_c4():
    # C4: 512^3 mixed medium, per-voxel albedo in [0.9, 0.999] and HG g in [0.3, 0.9] sampled at p
    # (scenes.sample_media), 1920x1080 = 2,073,600 queries, one light; frame = tvol build + query
    n4 = 512
    t0 = time.perf_counter()
    dens, alb, gg = scenes.mixed_medium_large(n4, 4)
    t_gen = time.perf_counter() - t0
    g4 = sf.DensityGrid.from_array(dens, 2.0 / n4, (-1.0, -1.0, -1.0))
    nq4 = 1920 * 1080
    rows4 = scenes.draw_centers(dens, nq4, 31, scenes.LIGHT)
    media = torch.from_numpy(scenes.sample_media(alb, gg, rows4)).cuda()
    rows4 = torch.from_numpy(rows4).cuda()
    F4 = torch.empty((nq4, 3), dtype=torch.float64, device="cuda")
    pyr4 = sf.DensityPyramid(g4, stream=stream)
    res = []
    for it in range(3):
        tv4, t_tv = timed(lambda: sf.build_transmittance_volume(pyr4, scenes.LIGHT, stream=stream, fast=FAST))
        sc4 = sf.Scene(g4, tv4, dt, ht, sf.PhaseModel.hg(0.6), table)
        _, t_q = timed(lambda: sf.query_media(sc4, net, rows4, media, sf.BF16, F_out=F4, stream=stream))
        if it > 0:
            res.append((t_tv, t_q))
    tv_ms = float(np.mean([x[0] for x in res]))
    q_ms = float(np.mean([x[1] for x in res]))
    print(json.dumps({"config": "C4", "grid": n4, "queries_per_frame": nq4, "frame_ms": tv_ms + q_ms,
                      "transmittance_ms": tv_ms, "query_ms": q_ms, "query_only_qps": nq4 / (q_ms * 1e-3),
                      "per_query_media": "g, albedo sampled at p (trilinear of the per-voxel grids)",
                      "scene_gen_s_host": round(t_gen, 1), "build": "fp64 march" if not FAST else "fp32 march",
                      "gpus": 1}))


if a.only_c4:
    run_c4()
    sys.exit(0)

# ---------------- C5
vol = scenes.noise_volume(N, 5)
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
nq = 1280 * 720
rows = torch.from_numpy(scenes.draw_centers(vol, nq, 21, scenes.LIGHT)).cuda()
F = torch.empty((nq, 3), dtype=torch.float64, device="cuda")
med = sf.MediumParams((0.7,), (0.99,) * 3)
model = sf.PhaseModel.hg(0.7)
pyr, t_pyr = timed(lambda: sf.DensityPyramid(g, stream=stream))
pyr, t_pyr = timed(lambda: sf.DensityPyramid(g, stream=stream))  # warm (module load, pool)
frames = []
sf.lib.sf_profile_enable(1)
profile_read()
for f in range(a.frames + 1):
    light = scenes.rotating_light(f, 32)
    tv, t_tv = timed(lambda: sf.build_transmittance_volume(pyr, light, stream=stream, fast=FAST))
    sc = sf.Scene(g, tv, dt, ht, model, table)
    r = rows.clone()
    r[:, 6:] = torch.tensor(np.asarray(light) / np.linalg.norm(light), device="cuda")
    _, t_q = timed(lambda: sf.query(sc, net, med, r, sf.BF16, F_out=F, stream=stream))
    if f > 0:  # frame 0 warms up
        frames.append((t_tv, t_q))
    else:
        profile_read()
stages = stage_split()
sf.lib.sf_profile_enable(0)
tv_ms = float(np.mean([x[0] for x in frames]))
q_ms = float(np.mean([x[1] for x in frames]))
frame_ms = tv_ms + q_ms
print(json.dumps({"config": "C5", "grid": N, "queries_per_frame": nq, "frames": a.frames,
                  "sustained_qps": nq / (frame_ms * 1e-3), "frame_ms": frame_ms, "transmittance_ms": tv_ms,
                  "query_ms": q_ms, "query_only_qps": nq / (q_ms * 1e-3), "pyramid_ms_once": t_pyr,
                  "query_stage_ms_per_frame": {k: v / a.frames for k, v in stages.items()},
                  "dtype": "bf16 network", "build": "fp64 march" if not FAST else "fp32 march", "gpus": 1}))

# ---------------- C3
vol = scenes.smoke_plume(N, 3)
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
pyr = sf.DensityPyramid(g, stream=stream)
lights, inten = scenes.c3_lights()
nq = 512 * 512
rows = scenes.draw_centers(vol, nq, 23, lights[0])
med = sf.MediumParams((0.5,), (0.95,) * 3)
model = sf.PhaseModel.hg(0.5)
for it in range(2):  # warm, then timed
    t0 = time.perf_counter()
    tot_tv = tot_q = 0.0
    total = torch.zeros((nq, 3), dtype=torch.float64, device="cuda")
    for light, I in zip(lights, inten):
        tv, t_tv = timed(lambda: sf.build_transmittance_volume(pyr, light, stream=stream, fast=FAST))
        sc = sf.Scene(g, tv, dt, ht, model, table)
        r = torch.from_numpy(configs.with_light(rows, light)).cuda()
        Fl = torch.empty((nq, 3), dtype=torch.float64, device="cuda")
        _, t_q = timed(lambda: sf.query(sc, net, med, r, sf.BF16, F_out=Fl, stream=stream))
        total += I * Fl
        tot_tv += t_tv
        tot_q += t_q
print(json.dumps({"config": "C3", "grid": N, "lights": len(lights), "queries_per_light": nq,
                  "empty_voxels": float(np.mean(vol == 0)),
                  "frame_ms": tot_tv + tot_q, "transmittance_ms_per_light": tot_tv / len(lights),
                  "query_ms_per_light": tot_q / len(lights),
                  "sustained_qps": len(lights) * nq / ((tot_tv + tot_q) * 1e-3), "gpus": 1}))

if a.c4:
    run_c4()
