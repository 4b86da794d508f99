"""Time the C2 bf16 query (device in/out) for several SF_PIPE_TILES values (one process each)."""
import os, subprocess, sys
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
ref = F.clone()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): sf.query(sc, net, med, c, sf.BF16, F_out=F)
b.record(); torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 50, "same": bool(torch.equal(F, ref)), "F": float(F.sum())}))
'''
for v in sys.argv[1:] or ["0", "64", "128", "256"]:
    env = dict(os.environ, SF_PIPE_TILES=v)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(v, r.stdout.strip() or r.stderr[-800:])
