"""Per-call wall time distribution of sf.query with pinned host rows in / host F out (the
bench e2e leg): is the end-to-end gap per-call host overhead or device time?"""
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
out = {}
for rep in range(3):
    for _ in range(3): sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream)
    w = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(100):
        t = time.perf_counter()
        sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream)
        w.append((time.perf_counter() - t) * 1e3)
    b.record(stream); torch.cuda.synchronize()
    w = np.array(w)
    out[f"rep{rep}"] = {"event_ms_per_call": round(a.elapsed_time(b) / 100, 4),
                        "wall_p10": round(float(np.percentile(w, 10)), 4), "wall_p50": round(float(np.median(w)), 4),
                        "wall_p90": round(float(np.percentile(w, 90)), 4), "wall_max": round(float(w.max()), 4)}
# fixed cost: tiny batch
qs, Fs = q[:128].copy(), F[:128].copy()
qs = torch.from_numpy(qs).pin_memory().numpy(); Fs = torch.from_numpy(Fs).pin_memory().numpy()
for _ in range(5): sf.query(sc, net, med, qs, sf.BF16, F_out=Fs, stream=stream)
t = time.perf_counter()
for _ in range(200): sf.query(sc, net, med, qs, sf.BF16, F_out=Fs, stream=stream)
out["tiny_wall_ms"] = round((time.perf_counter() - t) / 200 * 1e3, 4)
print(json.dumps(out))
