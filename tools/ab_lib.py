"""A/B two library builds on the C2 bf16 query: F bit-identity and device time per step.
usage: python tools/ab_lib.py OTHER.so  (the in-tree build is the other arm).
AB_ENV_OTHER="K=V,K2=V2" sets environment variables for the other arm only (OTHER.so may then be
the in-tree library itself, for an A/B of a runtime switch)."""
import os, subprocess, sys, json
code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.fractal_ellipsoid(128, 1)
c = torch.from_numpy(scenes.draw_centers(vol, 65536, 11, scenes.LIGHT)).cuda()
g = sf.DensityGrid.from_array(vol, 2.0 / 128, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
F = torch.empty((65536, 3), dtype=torch.float64, device="cuda")
for _ in range(5): sf.query(sc, net, med, c, sf.BF16, F_out=F)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    a.record()
    for _ in range(50): sf.query(sc, net, med, c, sf.BF16, F_out=F)
    b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b) / 50)
np.save(sys.argv[1], F.cpu().numpy())
print(json.dumps({"ms": sorted(ms)[2]}))
'''
out = {}
for name, lib in (("tree", ""), ("other", sys.argv[1])):
    env = dict(os.environ)
    if lib:
        env["SF_B200_LIB"] = os.path.abspath(lib)
        for kv in filter(None, os.environ.get("AB_ENV_OTHER", "").split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
    r = subprocess.run([sys.executable, "-c", code, f"/tmp/ab_{name}.npy"], env=env, capture_output=True, text=True)
    out[name] = r.stdout.strip() or r.stderr[-400:]
import numpy as np
A, B = np.load("/tmp/ab_tree.npy"), np.load("/tmp/ab_other.npy")
out["bit_identical"] = bool(np.array_equal(A, B))
out["max_abs_diff"] = float(np.abs(A - B).max())
print(json.dumps(out))
