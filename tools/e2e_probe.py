"""Time sf.query with pinned host rows in / host F out (the bench e2e leg) against device
buffers, one side at a time (where does the end-to-end gap come from?)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
vol = scenes.fractal_ellipsoid(128, 1)
c = scenes.draw_centers(vol, 65536, 11, scenes.LIGHT)
g = sf.DensityGrid.from_array(vol, 2.0 / 128, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")), sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.85), sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0)); med = sf.MediumParams((0.85,), (0.999,) * 3)
stream = torch.cuda.current_stream()
q = torch.from_numpy(c).pin_memory().numpy()
F = torch.empty((65536, 3), dtype=torch.float64).pin_memory().numpy()
qd = torch.from_numpy(c).cuda(); Fd = torch.empty((65536, 3), dtype=torch.float64, device="cuda")
out = {}
for name, (qi, fo) in {"host": (q, F), "host_in": (q, Fd), "host_out": (qd, F), "device": (qd, Fd)}.items():
    for _ in range(3): sf.query(sc, net, med, qi, sf.BF16, F_out=fo, stream=stream)
    torch.cuda.synchronize()
    reps = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(40): sf.query(sc, net, med, qi, sf.BF16, F_out=fo, stream=stream)
        b.record(stream); torch.cuda.synchronize()
        reps.append(a.elapsed_time(b) / 40)
    out[name] = round(sorted(reps)[3], 4)
print(json.dumps(out))
