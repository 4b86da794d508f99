"""Fixed per-call cost of sf.query (host wall time) for tiny batches, host and device I/O."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.fractal_ellipsoid(64, 1)
g = sf.DensityGrid.from_array(vol, 2.0 / 64, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
out = {}
for n in (128, 65536):
    c = scenes.draw_centers(vol, n, 11, scenes.LIGHT)
    q = torch.from_numpy(c).pin_memory().numpy()
    F = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    for _ in range(5): sf.query(sc, net, med, q, sf.BF16, F_out=F)
    t = time.perf_counter()
    for _ in range(100): sf.query(sc, net, med, q, sf.BF16, F_out=F)
    out[f"host_io_n{n}_ms"] = (time.perf_counter() - t) * 10
    qd = torch.from_numpy(c).cuda(); Fd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    for _ in range(5): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(100): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd)
    torch.cuda.synchronize()
    out[f"device_io_n{n}_ms"] = (time.perf_counter() - t) * 10
print(json.dumps(out))
