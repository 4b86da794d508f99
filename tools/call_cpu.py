"""Host-side cost of one sf.query call: CPU time of the asynchronous device-pointer call
(submission only), and the Python wrapper alone (ctypes argument marshalling)."""
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
qd = torch.from_numpy(c).cuda(); Fd = torch.empty((65536, 3), dtype=torch.float64, device="cuda")
out = {}
for _ in range(5): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd, stream=stream)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    t = time.perf_counter(); sf.query(sc, net, med, qd, sf.BF16, F_out=Fd, stream=stream); ts.append(time.perf_counter() - t)
    torch.cuda.synchronize()
out["async_device_call_us_p50"] = round(float(np.median(ts)) * 1e6, 1)
q = sf.pinned_empty(c.shape); q[:] = c; F = sf.pinned_empty((65536, 3))
for _ in range(5): sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream)
ts = []
for _ in range(50):
    t = time.perf_counter(); sf.query(sc, net, med, q, sf.BF16, F_out=F, stream=stream); ts.append(time.perf_counter() - t)
out["sync_host_call_us_p50"] = round(float(np.median(ts)) * 1e6, 1)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(20): sf.query(sc, net, med, qd, sf.BF16, F_out=Fd, stream=stream)
b.record(stream); torch.cuda.synchronize()
out["device_ms"] = round(a.elapsed_time(b) / 20, 4)
m = med.to_c()
import ctypes as C
from paper_2401_14051_b200._lib import ptr, stream_ptr
ts = []
for _ in range(200):
    t = time.perf_counter(); _ = (ptr(q), ptr(F), stream_ptr(stream), med.to_c()); ts.append(time.perf_counter() - t)
out["python_marshalling_us"] = round(float(np.median(ts)) * 1e6, 2)
print(json.dumps(out))
