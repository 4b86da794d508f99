"""A/B the graded-transmittance march (SF_GRADED=0) against the shared tap lists (SF_GRADED=1):
per-level graded fields and the combined volume, exact (FP64) and production (FP32) builds,
on a 64^3 cloud, a non-cubic 64x32x16 grid and the 256^3 C5 noise volume under several lights;
plus build times at 256^3 (median of 5).
usage: python tools/ab_taps.py"""
import json
import os
import subprocess
import sys

code = r'''
import os, sys, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
res = {}
outs = {}
lights = [scenes.LIGHT, scenes.rotating_light(5, 32), scenes.rotating_light(13, 32), (0.0, -1.0, 0.0), (0.0, 0.0, 1.0),
          (1.0, 0.0, 0.0), (0.6, 0.7, -0.4), (-0.3, 0.2, 0.9)]
cases = [("c1", scenes.procedural_cloud(64, 0)), ("nc", scenes.procedural_cloud(64, 2)[:16, :32, :]),
         ("c5", scenes.noise_volume(256, 5))]
for name, vol in cases:
    nz, ny, nx = vol.shape
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / nx, (-1.0, -1.0, -1.0)))
    for li, L in enumerate(lights if name != "c5" else lights[:3]):
        for fast in (False, True):
            tv = sf.build_transmittance_volume(pyr, L, fast=fast)
            outs[f"{name}_{li}_{int(fast)}"] = tv.values.values().ravel()
            if name != "c5":
                for lev in range(pyr.level_count()):
                    vs = 2.0 / nx * 2 ** lev
                    if not fast:
                        outs[f"{name}_{li}_g{lev}"] = sf.graded_transmittance(pyr, lev, L, 0.6, 0.5 * vs).values.values().ravel()
    if name == "c5":
        for fast in (False, True):
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                t = time.perf_counter(); sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast); torch.cuda.synchronize()
                ts.append(time.perf_counter() - t)
            res[f"build_256_{'fp32' if fast else 'fp64'}_ms"] = round(sorted(ts)[2] * 1e3, 3)
np.savez(sys.argv[1], **outs)
print(json.dumps(res))
'''
out = {}
for mode in ("0", "1"):
    env = dict(os.environ, SF_GRADED=mode)
    r = subprocess.run([sys.executable, "-c", code, f"/tmp/abt_{mode}.npz"], env=env, capture_output=True, text=True)
    out[f"mode{mode}"] = r.stdout.strip() or r.stderr[-2000:]
import numpy as np  # noqa: E402

A, B = np.load("/tmp/abt_0.npz"), np.load("/tmp/abt_1.npz")
worst = {}
for k in A.files:
    a, b = A[k], B[k]
    ulp = np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
    worst[k] = {"max_abs": float(np.abs(a - b).max()), "max_ulp": int(ulp.max()), "frac_equal": float(np.mean(a == b))}
out["exact_builds_max_ulp"] = max(v["max_ulp"] for k, v in worst.items() if not k.endswith("_1"))
out["exact_builds_min_frac_equal"] = min(v["frac_equal"] for k, v in worst.items() if not k.endswith("_1"))
out["fast_builds_max_abs"] = max(v["max_abs"] for k, v in worst.items() if k.endswith("_1"))
out["fast_vs_exact_taps_max_abs"] = max(float(np.abs(B[k] - B[k[:-2] + "_0"]).max()) for k in B.files if k.endswith("_1"))
out["detail"] = worst
print(json.dumps(out, indent=1))
