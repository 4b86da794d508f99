"""A/B Scene.relight (the per-frame build at 256^3, FP32 taps) under env settings: device ms per
relight (median over 8 lights x 3) and whether every relit volume is identical to the first arm's.
usage: python tools/ab_relight.py NAME=tree[@K=V,...] ..."""
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
sc = sf.Scene(g, sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=True), sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
ms, outs = [], []
for it in range(3):
    for k in range(0, 32, 4):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sc.relight(pyr, scenes.rotating_light(k, 32), fast=True)
        b.record(); torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        if it == 2:
            outs.append(sc.tvol_storage().cpu().numpy().copy())
np.save(sys.argv[1], np.stack(outs))
m = sorted(ms[8:])
print(json.dumps({"ms_median": m[len(m) // 2], "ms_min": m[0]}))
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
    out = f"/tmp/abr_{name}.npy"
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True)
    res = {"arm": name, "result": r.stdout.strip() or r.stderr[-600:]}
    if os.path.exists(out):
        T = np.load(out)
        if first is None:
            first = T
        res["identical_to_first"] = bool(np.array_equal(T, first))
    print(json.dumps(res), flush=True)
