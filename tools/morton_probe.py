"""Does spatial (Morton) order of the query rows speed up k_sample_sort? (host-side pre-sort probe)"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
from paper_2401_14051_b200._lib import profile_read

def morton(c, n=128):
    v = np.clip(((c[:, :3] + 1.0) * 0.5 * n).astype(np.int64), 0, n - 1)
    key = np.zeros(len(c), np.int64)
    for b in range(7):
        for a in range(3):
            key |= ((v[:, a] >> b) & 1) << (3 * b + a)
    return np.argsort(key, kind="stable")

vol = scenes.fractal_ellipsoid(128, 1)
rows = scenes.draw_centers(vol, 65536, 11, scenes.LIGHT)
g = sf.DensityGrid.from_array(vol, 2.0 / 128, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
for name, order in (("random", np.arange(len(rows))), ("morton", morton(rows))):
    c = torch.from_numpy(np.ascontiguousarray(rows[order])).cuda()
    F = torch.empty((65536, 3), dtype=torch.float64, device="cuda")
    for _ in range(3): sf.query(sc, net, med, c, sf.BF16, F_out=F)
    torch.cuda.synchronize(); sf.lib.sf_profile_enable(1); profile_read()
    for _ in range(10): sf.query(sc, net, med, c, sf.BF16, F_out=F)
    torch.cuda.synchronize(); st = profile_read(); sf.lib.sf_profile_enable(0)
    print(name, json.dumps({k: round(v[0] / 10, 4) for k, v in st.items() if v[1]}))
