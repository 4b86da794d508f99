"""Per-light transmittance builds for ncu launch lists: the C5 noise volume under the first C5 light
and the C3 plume under its four lights (production FP32 build; --exact: FP64).
usage: python tools/profile_build.py [--exact] [--grid 256] [--which c5,c3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_14051_b200 as sf  # noqa: E402
from paper_2401_14051_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--exact", action="store_true")
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--which", default="c5,c3")
a = ap.parse_args()
N = a.grid
for which in a.which.split(","):
    vol = scenes.noise_volume(N, 5) if which == "c5" else scenes.smoke_plume(N, 3)
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0)))
    lights = [scenes.rotating_light(0, 32)] if which == "c5" else scenes.c3_lights()[0]
    for L in lights:
        sf.build_transmittance_volume(pyr, L, fast=not a.exact)
torch.cuda.synchronize()
print("ok")
