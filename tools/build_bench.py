"""Per-light transmittance build time (exact FP64 and FP32 march) at 128^3 and 256^3."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
out = {}
for N in (128, 256):
    vol = scenes.fractal_ellipsoid(N, 1) if N == 128 else scenes.noise_volume(N, 5)
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0)))
    for fast in (False, True):
        sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3): sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast)
        torch.cuda.synchronize(); out[f"{N}_{'fp32' if fast else 'fp64'}_ms"] = round((time.perf_counter() - t) / 3 * 1e3, 3)
print(json.dumps(out))
