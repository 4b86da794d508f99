"""One C5 frame query (tools/ab_c5.py's workload) after warm-up: for ncu captures of the query kernels."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.noise_volume(256, 5)
c = torch.from_numpy(scenes.draw_centers(vol, 1280 * 720, 21, scenes.LIGHT)).cuda()
g = sf.DensityGrid.from_array(vol, 2.0 / 256, (-1.0, -1.0, -1.0))
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT, fast=True), sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.7,), (0.99,) * 3)
F = torch.empty((len(c), 3), dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("BB_REPS", "2"))): sf.query(sc, net, med, c, sf.FP16, F_out=F)
torch.cuda.synchronize()
print("ok")
