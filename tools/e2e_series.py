"""Wall time per sf.query call (pinned host I/O) over 1,500 consecutive calls right after a
stretch of device-only work, in blocks of 50: when does the end-to-end path reach its steady
state, and is the slow phase time- or call-count-based?"""
import os, sys, time, json
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
for phase in range(2):
    for _ in range(300): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd, stream=stream)  # device-only stretch
    torch.cuda.synchronize()
    if phase == 1: time.sleep(1.0)  # plus an idle second
    w = []
    t0 = time.perf_counter()
    for _ in range(1500):
        t = time.perf_counter()
        sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream)
        w.append((time.perf_counter() - t) * 1e3)
    w = np.array(w).reshape(30, 50)
    out[f"phase{phase}"] = {"block_median_ms": [round(float(x), 3) for x in np.median(w, 1)],
                            "total_s": round(time.perf_counter() - t0, 3)}
print(json.dumps(out))
