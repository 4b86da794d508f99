"""A/B library builds on the C5 per-frame rebuild (Scene.relight at 256^3, FP32-sum tap build):
device ms per relight (median of 4 lights x 3) and whether the transmittance volumes are identical
to the first arm's. usage: python tools/ab_build.py NAME=LIB[@K=V,...] ...  (LIB "tree" = in-tree)"""
import json, os, subprocess, sys
import numpy as np

code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
N = int(os.environ.get("AB_GRID", "256"))
vol = scenes.noise_volume(N, 5)
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
pyr = sf.DensityPyramid(g)
data = os.path.join(os.path.dirname(sf.__file__), "data")
outs, ms = [], []
for it in range(3):
    for k in (0, 5, 11, 22):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tv = sf.build_transmittance_volume(pyr, scenes.rotating_light(k, 32), fast=True)
        b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        if it == 2:
            outs.append(tv.values.values())
np.save(sys.argv[1], np.stack(outs))
print(json.dumps({"ms_median": sorted(ms[4:])[len(ms[4:]) // 2], "ms_all": [round(x, 3) for x in ms]}))
'''

first = None
for arg in sys.argv[1:]:
    name, spec = arg.split("=", 1)
    lib, _, envs = spec.partition("@")
    env = dict(os.environ)
    if lib != "tree":
        env["SF_B200_LIB"] = os.path.abspath(lib)
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    out = f"/tmp/abb_{name}.npy"
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True)
    res = {"arm": name, "result": r.stdout.strip() or r.stderr[-600:]}
    if os.path.exists(out):
        T = np.load(out)
        if first is None:
            first = T
        res["identical_to_first"] = bool(np.array_equal(T, first))
    print(json.dumps(res), flush=True)
