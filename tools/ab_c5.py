"""A/B two library builds (or env settings) on the C5 frame query (921,600 bf16 queries on the
256^3 noise volume, Morton-ordered): device ms per query call (median of 5 x 10) and F identity.
usage: python tools/ab_c5.py OTHER.so   (AB_ENV_OTHER="K=V,..." for the other arm; AB_PREC=fp16|bf16)"""
import json, os, subprocess, sys
code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.noise_volume(256, 5)
c = torch.from_numpy(scenes.draw_centers(vol, 1280 * 720, 21, scenes.LIGHT)).cuda()
g = sf.DensityGrid.from_array(vol, 2.0 / 256, (-1.0, -1.0, -1.0))
pyr = sf.DensityPyramid(g)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=True), sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.7,), (0.99,) * 3)
F = torch.empty((len(c), 3), dtype=torch.float64, device="cuda")
PREC = sf.FP16 if os.environ.get("AB_PREC", "fp16") == "fp16" else sf.BF16
for _ in range(3): sf.query(sc, net, med, c, PREC, F_out=F)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    a.record()
    for _ in range(10): sf.query(sc, net, med, c, PREC, F_out=F)
    b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b) / 10)
from paper_2401_14051_b200._lib import profile_read
sf.lib.sf_profile_enable(1); profile_read()
for _ in range(10): sf.query(sc, net, med, c, PREC, F_out=F)
torch.cuda.synchronize()
st = {k: round(v[0] / 10, 4) for k, v in profile_read().items() if v[1]}
sf.lib.sf_profile_enable(0)
np.save(sys.argv[1], F.cpu().numpy())
print(json.dumps({"ms": sorted(ms)[2], "stages": st}))
'''

def main():
    out = {}
    for name, lib in (("tree", ""), ("other", sys.argv[1])):
        env = dict(os.environ)
        if lib:
            env["SF_B200_LIB"] = os.path.abspath(lib)
            for kv in filter(None, os.environ.get("AB_ENV_OTHER", "").split(",")):
                k, v = kv.split("=", 1)
                env[k] = v
        r = subprocess.run([sys.executable, "-c", code, f"/tmp/abc5_{name}.npy"], env=env, capture_output=True,
                           text=True)
        out[name] = r.stdout.strip() or r.stderr[-400:]
    import numpy as np
    A, B = np.load("/tmp/abc5_tree.npy"), np.load("/tmp/abc5_other.npy")
    out["bit_identical"] = bool(np.array_equal(A, B))
    out["max_abs_diff"] = float(np.abs(A - B).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
