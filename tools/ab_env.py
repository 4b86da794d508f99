"""A/B two environment settings of the library on the transmittance build: every output of
builds (exact and FP32, identity and random combiner, full and 3-slab) on a 64^3 cloud, a
non-cubic 64x32x16 grid and the 256^3 C5 volume under several lights, compared bit for bit;
plus median build times at 256^3.
usage: python tools/ab_env.py "SF_BUILD_V1=1" ""      (A env, B env; space-separated K=V)"""
import json
import os
import subprocess
import sys

code = r'''
import os, sys, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes, sharding
res, outs = {}, {}
lights = [scenes.LIGHT, scenes.rotating_light(5, 32), scenes.rotating_light(13, 32), (0.0, -1.0, 0.0), (0.6, 0.7, -0.4)]
cases = [("c1", scenes.procedural_cloud(64, 0)), ("nc", scenes.procedural_cloud(64, 2)[:16, :32, :]),
         ("c5", scenes.noise_volume(256, 5))]
for name, vol in cases:
    nz, ny, nx = vol.shape
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / nx, (-1.0, -1.0, -1.0)))
    L = pyr.level_count()
    rng = np.random.default_rng(3)
    k = rng.uniform(-0.2, 0.2, (L, 27)).astype(np.float32); k[:, 13] += 1
    wr = sf.CombinerWeights(k, np.full(L, 1.0 / L, np.float32))
    for li, lt in enumerate(lights if name != "c5" else lights[:2]):
        for fast in (False, True):
            for wn, w in (("id", None), ("rnd", wr)):
                outs[f"{name}_{li}_{int(fast)}_{wn}"] = sf.build_transmittance_volume(pyr, lt, w, fast=fast).values.values().ravel()
            if name == "c1":
                parts = [sf.build_transmittance_slab(pyr, lt, z0, z1, wr, fast=fast) for z0, z1 in sharding.z_slabs(nz, 3)]
                outs[f"{name}_{li}_{int(fast)}_slab"] = np.concatenate(parts).ravel()
    if name == "c5":
        for fast in (False, True):
            sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast); torch.cuda.synchronize()
            ts = []
            for _ in range(7):
                t = time.perf_counter(); sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast); torch.cuda.synchronize()
                ts.append(time.perf_counter() - t)
            res[f"build_256_{'fp32' if fast else 'fp64'}_ms"] = round(sorted(ts)[3] * 1e3, 3)
np.savez(sys.argv[1], **outs)
print(json.dumps(res))
'''
out = {}
for tag, spec in (("A", sys.argv[1]), ("B", sys.argv[2])):
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", code, f"/tmp/abe_{tag}.npz"], env=env, capture_output=True, text=True)
    out[tag] = (spec, r.stdout.strip() or r.stderr[-2000:])
import numpy as np  # noqa: E402

A, B = np.load("/tmp/abe_A.npz"), np.load("/tmp/abe_B.npz")
diff = {}
for k in A.files:
    a, b = A[k], B[k]
    if not np.array_equal(a, b):
        ulp = np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
        diff[k] = {"max_abs": float(np.abs(a - b).max()), "max_ulp": int(ulp.max()), "frac_equal": float(np.mean(a == b))}
out["arrays"] = len(A.files)
out["bit_identical"] = not diff
out["differences"] = diff
print(json.dumps(out, indent=1))
