"""Time the bf16 query stages under SF_DEBUG_SAMPLE_SORT variants (one process per variant; the library
must be built with SF_NVCC_EXTRA=-DSF_SAMPLE_SORT_DEBUG, else the switches are compiled out)."""
import os, subprocess, sys, json
code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
from paper_2401_14051_b200._lib import profile_read
C5 = os.environ.get("AB_C5") is not None
N = 256 if C5 else 128
vol = scenes.noise_volume(256, 5) if C5 else scenes.fractal_ellipsoid(128, 1)
c = torch.from_numpy(scenes.draw_centers(vol, 921600 if C5 else 65536, 21 if C5 else 11, scenes.LIGHT)).cuda()
g = sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
F = torch.empty((len(c), 3), dtype=torch.float64, device="cuda")
for _ in range(3): sf.query(sc, net, med, c, sf.FP16, F_out=F)
torch.cuda.synchronize(); sf.lib.sf_profile_enable(1); profile_read()
for _ in range(10): sf.query(sc, net, med, c, sf.FP16, F_out=F)
torch.cuda.synchronize(); st = profile_read()
print(json.dumps({k: v[0] / 10 for k, v in st.items() if v[1]}))
'''
for mode in sys.argv[1:] or ["0", "1", "2", "4", "6", "7"]:
    env = dict(os.environ, SF_DEBUG_SAMPLE_SORT=mode)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(mode, r.stdout.strip() or r.stderr[-500:])
