"""Time build_transmittance_volume and Scene.relight at 256^3 (C5 volume): wall and device ms."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.noise_volume(256, 5)
g = sf.DensityGrid.from_array(vol, 2.0 / 256, (-1.0, -1.0, -1.0))
pyr = sf.DensityPyramid(g)
data = os.path.join(os.path.dirname(sf.__file__), "data")
res = {}
for fast in (True, False):
    for it in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); e0.record()
        tv = sf.build_transmittance_volume(pyr, scenes.rotating_light(it, 32), fast=fast)
        e1.record(); torch.cuda.synchronize()
        res.setdefault(f"build_{int(fast)}", []).append((round((time.perf_counter() - t) * 1e3, 3), round(e0.elapsed_time(e1), 3)))
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
for fast in (True, False):
    for it in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); e0.record()
        sc.relight(pyr, scenes.rotating_light(it, 32), fast=fast)
        e1.record(); torch.cuda.synchronize()
        res.setdefault(f"relight_{int(fast)}", []).append((round((time.perf_counter() - t) * 1e3, 3), round(e0.elapsed_time(e1), 3)))
print(json.dumps(res))
