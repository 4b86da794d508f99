"""A/B two library builds on the production (FP32-march; AB_EXACT=1: the FP64 march) transmittance build: bit identity
on a 128^3 cloud and a 256^3 noise volume, and the build time at 256^3.
usage: python tools/ab_build.py OTHER.so"""
import os, subprocess, sys, json
code = r'''
import os, sys, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
FAST = os.environ.get("AB_EXACT") is None
res = {}
outs = []
for N, vol in ((128, scenes.fractal_ellipsoid(128, 1)), (256, scenes.noise_volume(256, 5))):
    pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0)))
    tv = sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=FAST)
    outs.append(tv.values.values().ravel())
    if N == 256:
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t = time.perf_counter(); sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=FAST); torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        res["build_256_ms"] = round(sorted(ts)[2] * 1e3, 3)
np.save(sys.argv[1], np.concatenate(outs))
print(json.dumps(res))
'''
out = {}
for name, lib in (("tree", ""), ("other", sys.argv[1])):
    env = dict(os.environ)
    if lib:
        env["SF_B200_LIB"] = os.path.abspath(lib)
    r = subprocess.run([sys.executable, "-c", code, f"/tmp/abb_{name}.npy"], env=env, capture_output=True, text=True)
    out[name] = r.stdout.strip() or r.stderr[-400:]
import numpy as np
A, B = np.load("/tmp/abb_tree.npy"), np.load("/tmp/abb_other.npy")
out["bit_identical"] = bool(np.array_equal(A, B))
out["max_abs_diff"] = float(np.abs(A - B).max())
print(json.dumps(out))
