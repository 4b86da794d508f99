"""A/B library builds on the C4 query (per-query media, full-table phase lookups): 512^3 mixed medium
(AB_GRID to shrink it), 2,073,600 fp16 queries; device ms per query call (median of 5) and F identity with
the first arm. usage: python tools/ab_c4.py NAME=LIB[@K=V,...] ...   (LIB "tree" = the in-tree build)"""
import json, os, subprocess, sys
import numpy as np

code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
N = int(os.environ.get("AB_GRID", "512"))
vol, alb, gg = scenes.mixed_medium_large(N, 4)
rows = scenes.draw_centers(vol, 1920 * 1080, 31, scenes.LIGHT)
media = torch.from_numpy(scenes.sample_media(alb, gg, rows)).cuda()
rows = torch.from_numpy(rows).cuda()
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT, fast=True), sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.6), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0))
F = torch.empty((len(rows), 3), dtype=torch.float64, device="cuda")
for _ in range(2): sf.query_media(sc, net, rows, media, sf.FP16, F_out=F)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    a.record(); sf.query_media(sc, net, rows, media, sf.FP16, F_out=F); b.record(); torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
from paper_2401_14051_b200._lib import profile_read
sf.lib.sf_profile_enable(1); profile_read()
sf.query_media(sc, net, rows, media, sf.FP16, F_out=F); torch.cuda.synchronize()
st = {k: round(v[0], 3) for k, v in profile_read().items() if v[1]}
np.save(sys.argv[1], F.cpu().numpy())
print(json.dumps({"ms": sorted(ms)[2], "stages": st}))
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
    out = f"/tmp/abc4_{name}.npy"
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True)
    res = {"arm": name, "result": r.stdout.strip() or r.stderr[-600:]}
    if os.path.exists(out):
        F = np.load(out)
        if first is None:
            first = F
        res["identical_to_first"] = bool(np.array_equal(F, first))
    print(json.dumps(res), flush=True)
