"""One (or a few) C5 frames for ncu captures: pyramid once, then per frame the FP32-march
transmittance build, scene records and the fp16 (default) or bf16 query of 921,600 shading points.

usage: python tools/profile_c5.py [--frames 1] [--grid 256] [--queries 921600]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_14051_b200 as sf  # noqa: E402
from paper_2401_14051_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=1)
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--queries", type=int, default=1280 * 720)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16"])
ap.add_argument("--profile-last", action="store_true", help="cudaProfilerStart/Stop around the last frame only")
a = ap.parse_args()
N = a.grid
vol = scenes.noise_volume(N, 5)
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
rows = torch.from_numpy(scenes.draw_centers(vol, a.queries, 21, scenes.LIGHT)).cuda()
data = os.path.join(os.path.dirname(sf.__file__), "data")
dt = sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl"))
ht = sf.load_template(os.path.join(data, "highlight_seed8.vtmpl"))
table = sf.PhaseTable(64, 128, 32, 16)
net = sf.make_backbone(sf.BackboneConfig(seed=0))
F = torch.empty((a.queries, 3), dtype=torch.float64, device="cuda")
pyr = sf.DensityPyramid(g)
sc = sf.Scene(g, sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=not a.exact), dt, ht, sf.PhaseModel.hg(0.7),
              table)
for f in range(a.frames):  # the bench's per-frame path: relight + query
    if a.profile_last and f == a.frames - 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    light = scenes.rotating_light(f, 32)
    sc.relight(pyr, light, fast=not a.exact)
    rows[:, 6:] = torch.tensor(np.asarray(light) / np.linalg.norm(light), device="cuda")
    sf.query(sc, net, sf.MediumParams((0.7,), (0.99,) * 3), rows, sf.FP16 if a.precision == "fp16" else sf.BF16, F_out=F)
torch.cuda.synchronize()
if a.profile_last:
    torch.cuda.profiler.stop()
print("ok", float(F.mean()))
