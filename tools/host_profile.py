"""Where the fixed per-call host time of sf.query goes (n = 128, device I/O)."""
import os, sys, time, json, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
from paper_2401_14051_b200._lib import lib, ptr, stream_ptr
vol = scenes.fractal_ellipsoid(64, 1)
g = sf.DensityGrid.from_array(vol, 2.0 / 64, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
n = 128
qd = torch.from_numpy(scenes.draw_centers(vol, n, 11, scenes.LIGHT)).cuda()
Fd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
m = med.to_c()
qp, fp = ptr(qd), ptr(Fd)
out = {}
def bench(name, fn, k=300):
    for _ in range(10): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); out[name] = (time.perf_counter() - t) / k * 1e6
bench("python_wrapper_us", lambda: sf.query(sc, net, med, qd, sf.BF16, F_out=Fd))
bench("raw_ctypes_us", lambda: lib.sf_query(sc._h, net._h, C.byref(m), n, qp, 1, fp, None, None))
bench("launch_count_us", lambda: lib.sf_launch_count())
x = torch.empty(1, device="cuda")
bench("torch_tiny_kernel_us", lambda: x.add_(1))
bench("raw_ctypes_fp32_us", lambda: lib.sf_query(sc._h, net._h, C.byref(m), n, qp, 0, fp, None, None))
print(json.dumps(out))
