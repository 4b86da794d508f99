"""FP32-sum (production) vs FP64 (exact) transmittance build on a cheap synthetic volume at large
grids: max |dT| per grid (the bound tests/test_gpu_parity.py states). usage: python tools/fast_vs_exact_large.py 256 512"""
import os, sys, time, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes


def blobs(n):
    x = np.linspace(-1.0, 1.0, n, dtype=np.float32)
    f = 0.5 + 0.5 * np.sin(7 * x)[None, None, :] * np.cos(5 * x)[None, :, None] * np.sin(3 * x + 1)[:, None, None]
    return np.ascontiguousarray(np.where(f > 0.45, 2.0 * f, 0.0).astype(np.float32))


for n in map(int, sys.argv[1:]):
    vol = blobs(n)
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / n, (-1.0, -1.0, -1.0)))
    t = time.time()
    exact = sf.build_transmittance_volume(pyr, scenes.LIGHT).values.values()
    t1 = time.time()
    fast = sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=True).values.values()
    t2 = time.time()
    d = np.abs(fast - exact)
    print(json.dumps({"n": n, "max_dT": float(d.max()), "p999": float(np.quantile(d[::7, ::5, ::3], 0.999)),
                      "exact_s": t1 - t, "fast_s": t2 - t1, "T_min": float(exact.min()), "occupied": float((vol > 0).mean())}))
