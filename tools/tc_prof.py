"""Per-phase cycle breakdown of tensor-core backbone CTA 0 (SF_DEBUG_TC=1; needs a library built with
SF_NVCC_EXTRA=-DSF_TC_PROFILE, e.g. tools/build_variant.py variants/prof.so -DSF_TC_PROFILE + SF_B200_LIB)."""
import ctypes, os, sys
os.environ["SF_DEBUG_TC"] = sys.argv[1] if len(sys.argv) > 1 else "1"
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
for _ in range(3): sf.query(sc, net, med, c, sf.BF16, F_out=F)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)()
sf.lib.sf_debug_tc_profile(buf)
for _ in range(5): sf.query(sc, net, med, c, sf.BF16, F_out=F)
torch.cuda.synchronize()
sf.lib.sf_debug_tc_profile(buf)
names = ["wait_full1", "mma_fc1", "epi_fc1", "wait_full2", "issue_fc2", "attention", "wait_fc2", "epi_fc2+loop", "total"]
v = [buf[i] / 5 for i in range(16)]
print({n: int(x) for n, x in zip(names, v)}, "per-layer-step avg (36 layers):", {n: int(x / 36) for n, x in zip(names[:7], v[:7])})
print("fc2 epilogue split (per layer):", {k: int(v[i] / 36) for k, i in (("tmem_ld", 9), ("math", 10), ("store", 11))})
n_mma = max(v[13], 1)
print("run_mma per call (cycles):", {k: int(v[i] / n_mma) for k, i in (("sync", 9), ("prefetch", 10), ("issue", 11), ("wait", 12))}, "calls", n_mma)
