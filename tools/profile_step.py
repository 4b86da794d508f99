"""One C2 query step for ncu captures: python tools/profile_step.py [--precision bf16|fp32] [--steps N]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_14051_b200 as sf  # noqa: E402
from paper_2401_14051_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="bf16")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--n", type=int, default=65536)
a = ap.parse_args()
vol = scenes.fractal_ellipsoid(128, 1)
centers = scenes.draw_centers(vol, a.n, 11, scenes.LIGHT)
g = sf.DensityGrid.from_array(vol, 2.0 / 128, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
scene = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")),
                 sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85),
                 sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0))
med = sf.MediumParams((0.85,), (0.999,) * 3)
prec = sf.BF16 if a.precision == "bf16" else sf.FP32
import torch  # noqa: E402
qd = torch.from_numpy(centers).cuda()  # device-resident rows, as bench.py's `value` leg
Fd = torch.empty((len(centers), 3), dtype=torch.float64, device="cuda")
for _ in range(a.steps):
    sf.query(scene, net, med, qd, prec, F_out=Fd)
torch.cuda.synchronize()
print("ok", float(Fd.mean()))
