"""Diagnose the two states of the synchronous e2e path: per 50-call block, the median wall
time per call, the GPU span per call (events around the call), a pinned 4.7 MB H2D and a
1.6 MB D2H copy time, and the device-only query time."""
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
mode = sys.argv[1] if len(sys.argv) > 1 else "torch"  # torch: torch pin_memory; sf: sf.pinned_empty
if mode == "sf":
    q = sf.pinned_empty(c.shape); q[:] = c
    F = sf.pinned_empty((65536, 3))
    hbuf = sf.pinned_empty((4718592,), np.uint8)
    hb = torch.from_numpy(hbuf)
else:
    q = torch.from_numpy(c).pin_memory().numpy()
    F = torch.empty((65536, 3), dtype=torch.float64).pin_memory().numpy()
    hb = torch.empty(4718592, dtype=torch.uint8).pin_memory()
qd = torch.from_numpy(c).cuda(); Fd = torch.empty((65536, 3), dtype=torch.float64, device="cuda")
db = torch.empty(4718592, dtype=torch.uint8, device="cuda")
def ev(): return torch.cuda.Event(enable_timing=True)
rows = []
for blk in range(8):
    wall, span = [], []
    for _ in range(50):
        a, b = ev(), ev()
        a.record(stream)
        t = time.perf_counter()
        sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream)
        wall.append((time.perf_counter() - t) * 1e3)
        b.record(stream); b.synchronize()
        span.append(a.elapsed_time(b))
    a, b = ev(), ev(); a.record(stream)
    for _ in range(10): db.copy_(hb, non_blocking=True)
    b.record(stream); b.synchronize(); h2d = a.elapsed_time(b) / 10
    a, b = ev(), ev(); a.record(stream)
    for _ in range(10): hb[:1572864].copy_(db[:1572864], non_blocking=True)
    b.record(stream); b.synchronize(); d2h = a.elapsed_time(b) / 10
    a, b = ev(), ev(); a.record(stream)
    for _ in range(10): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd, stream=stream)
    b.record(stream); b.synchronize(); dev = a.elapsed_time(b) / 10
    rows.append([blk, round(float(np.median(wall)), 3), round(float(np.median(span)), 3), round(h2d * 1e3, 1),
                 round(d2h * 1e3, 1), round(dev, 3)])
print(json.dumps({"mode": mode, "cols": ["block", "wall_ms", "gpu_span_ms", "h2d_4.7MB_us", "d2h_1.6MB_us", "device_ms"], "rows": rows}))
