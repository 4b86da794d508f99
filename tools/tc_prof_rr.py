"""Per-phase cycle breakdown of k_backbone_rr, CTA 0 / thread 0 (SF_DEBUG_TC=1), on the C5 frame query
(tools/ab_c5.py's workload). Phases: wait_mma, wait_big, wait_small, barrier+issue, FC-1 epilogue,
FC-2 epilogue (+attention), misc, tail. Needs a -DSF_TC_PROFILE build (see tools/tc_prof.py)."""
import ctypes, os, sys
os.environ.setdefault("SF_DEBUG_TC", "1")
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
for _ in range(3): sf.query(sc, net, med, c, sf.FP16, F_out=F)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)()
sf.lib.sf_debug_tc_profile(buf)
R = 5
for _ in range(R): sf.query(sc, net, med, c, sf.FP16, F_out=F)
torch.cuda.synchronize()
sf.lib.sf_debug_tc_profile(buf)
names = ["wait_mma", "wait_big", "wait_small", "bar+issue", "epi_fc1", "epi_fc2", "pre_acq", "pre_wait", "total", "chains_end", "tail"]
# two launches per query call (chunks): per CTA-0 run
print({n: int(buf[i] / R / 2) for i, n in enumerate(names)})
