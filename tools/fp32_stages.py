"""Per-stage device times of the FP32 exact query path at C1 (64^3, 4,096 queries) and C2 sizes."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
from paper_2401_14051_b200._lib import profile_read
data = os.path.join(os.path.dirname(sf.__file__), "data")
dt, ht = sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl"))
net = sf.make_backbone(sf.BackboneConfig(seed=0))
out = {}
for name, vol, n, g_, a_ in (("C1", scenes.procedural_cloud(64, 0), 4096, 0.7, 0.99), ("C2", scenes.fractal_ellipsoid(128, 1), 65536, 0.85, 0.999)):
    N = vol.shape[0]
    g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
    sc = sf.Scene(g, tv, dt, ht, sf.PhaseModel.hg(g_), sf.PhaseTable(64, 128, 32, 16))
    med = sf.MediumParams((g_,), (a_,) * 3)
    c = torch.from_numpy(scenes.draw_centers(vol, n, 5, scenes.LIGHT)).cuda()
    F = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    for _ in range(2): sf.query(sc, net, med, c, sf.FP32, F_out=F)
    torch.cuda.synchronize(); sf.lib.sf_profile_enable(1); profile_read()
    for _ in range(3): sf.query(sc, net, med, c, sf.FP32, F_out=F)
    torch.cuda.synchronize(); st = profile_read(); sf.lib.sf_profile_enable(0)
    out[name] = {k: round(v[0] / 3, 3) for k, v in st.items() if v[1]}
    out[name]["qps_M"] = round(n / (sum(v[0] for v in st.values()) / 3 * 1e-3) / 1e6, 2)
print(json.dumps(out))
