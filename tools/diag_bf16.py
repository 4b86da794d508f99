import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
from conftest import DATA, ORIGIN
vol = scenes.procedural_cloud(64, 2)
g = sf.DensityGrid.from_array(vol, 2.0 / 64, ORIGIN)
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
tm = (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))
table = sf.PhaseTable(64, 128, 32, 16)
rows = scenes.draw_centers(vol, 777, 5, scenes.LIGHT)
for name, ts, lit in (("lit", 1.0, True), ("ts2.5", 2.5, False), ("both", 2.5, True)):
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), table, template_scale=ts)
    net = sf.make_backbone(sf.BackboneConfig(seed=7, literal_attention=lit))
    med = sf.MediumParams((0.5,), (0.9, 0.8, 0.7))
    y32 = np.empty((777, 3), np.float32); y16 = np.empty((777, 3), np.float32)
    sf.query(scene, net, med, rows, sf.FP32, y_out=y32); sf.query(scene, net, med, rows, sf.BF16, y_out=y16)
    dy = np.abs(y16 - y32)
    print(name, "y32 range", y32.min(), y32.max(), "max dy", dy.max(), "p99", np.quantile(dy, 0.99), "rel max", (dy / np.maximum(np.abs(y32), 1)).max())
net = sf.make_backbone(sf.BackboneConfig(seed=7))
scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), table)
y32 = np.empty((777, 3), np.float32); y16 = np.empty((777, 3), np.float32)
sf.query(scene, net, sf.MediumParams((0.5,), (0.9, 0.8, 0.7)), rows, sf.FP32, y_out=y32); sf.query(scene, net, sf.MediumParams((0.5,), (0.9, 0.8, 0.7)), rows, sf.BF16, y_out=y16)
print("seed7 learned ts1", y32.max(), np.abs(y16-y32).max())
