"""Debug: production sampler pools vs the reference on an odd non-cubic grid."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2401_14051_b200 as sf
from oracle.oracle import Reference, PhaseModel
from test_gpu_reference_live import slice_pools, DT, HT
from conftest import LIGHT
R = Reference(); R.set_threads(os.cpu_count())
case = sys.argv[1] if len(sys.argv) > 1 else "odd"
rng = np.random.default_rng(7)
if case == "odd":
    nx, ny, nz, vs = 33, 20, 17, 0.0625
    origin = np.array([-1.0, -0.6, -0.5])
elif case == "cubic_off":   # cubic, origin offset
    nx, ny, nz, vs = 32, 32, 32, 0.0625
    origin = np.array([-1.0, -0.6, -0.5])
elif case == "odd_std":     # odd dims, standard origin
    nx, ny, nz, vs = 33, 20, 17, 0.0625
    origin = np.array([-1.0, -1.0, -1.0])
else:
    nx, ny, nz, vs = 32, 32, 32, 0.0625
    origin = np.array([-1.0, -1.0, -1.0])
vol = rng.uniform(0.0, 1.0, (nz, ny, nx)).astype(np.float32)
tvol = rng.uniform(0.05, 1.0, (nz, ny, nx)).astype(np.float32)
if case == "c2":
    from paper_2401_14051_b200 import scenes
    nx = ny = nz = 128
    vs = 2.0 / 128
    origin = np.array([-1.0, -1.0, -1.0])
    vol = scenes.fractal_ellipsoid(128, 1)
    tvol = R.build_tvol(vol, vs, origin, LIGHT)
hi = origin + vs * np.array([nx, ny, nz])
n = 512
p = origin + rng.uniform(0.0, 1.0, (n, 3)) * (hi - origin)
faces = "--faces" in sys.argv
if faces:
    for k in range(0, 96):
        a = k % 3
        p[k, a] = origin[a] if k % 2 else hi[a]
w = rng.normal(size=(n, 3)); w /= np.linalg.norm(w, axis=1, keepdims=True)
rows = np.concatenate([p, w, np.broadcast_to(LIGHT, (n, 3))], axis=1)
if case == "c2":
    from paper_2401_14051_b200 import scenes
    rows = scenes.draw_centers(vol, 65536, 11, scenes.LIGHT)[:1024]
    n = len(rows)
tab = R.phase_table(64, 128, 32, 16)
G = 0.85 if case == "c2" else 0.7
ctx = R.make_ctx(vol, tvol, vs, origin, DT, HT, PhaseModel.hg(G), tab)
feats = R.features(ctx, rows, 194, 72)
want = slice_pools(feats)
g = sf.DensityGrid.from_array(vol, vs, origin)
tv = sf.TransmittanceFeatureVolume.from_values(tvol, vs, origin, LIGHT)
d, h = sf.load_template(DT), sf.load_template(HT)
gt = sf.PhaseTable(64, 128, 32, 16)
scene = sf.Scene(g, tv, d, h, sf.PhaseModel.hg(G), gt)
net = sf.make_backbone(sf.BackboneConfig(seed=0))
got = sf.debug_query_pools(scene, net, sf.MediumParams((G,), (0.99,) * 3), rows)
# exact path features
fd = sf.sample_features(rows, d, g, tv, sf.PhaseModel.hg(G), gt)
fh = sf.sample_features(rows, h, g, tv, sf.PhaseModel.hg(G), gt)
fx = np.concatenate([fd.reshape(n, -1), fh.reshape(n, -1)], axis=1)
print(case, "faces" if faces else "", "exact-path feature max abs err", np.abs(fx - feats).max())
names = ["mean_d", "mean_p", "mean_t", "max_d", "max_p", "max_t"]
for k in range(6):
    e = np.abs(got[..., k] - want[..., k]) / np.maximum(np.abs(want[..., k]), 1e-6 * np.abs(want[..., k]).max())
    qi, li = np.unravel_index(np.argmax(e), e.shape)
    print(f"{names[k]}: max rel {e.max():.3e} at q {qi} layer {li}: got {got[qi, li, k]:.7g} want {want[qi, li, k]:.7g}"
          f"  frac>1e-5 {np.mean(e > 1e-5):.4f}  p={rows[qi,:3]}")

# worst density feature of the worst max_d query
e = np.abs(got[..., 3] - want[..., 3]) / np.maximum(np.abs(want[..., 3]), 1e-6 * np.abs(want[..., 3]).max())
qi, li = np.unravel_index(np.argmax(e), e.shape)
print("worst max_d query", qi, "layer", li, "row", rows[qi])
counts = [6, 8, 12, 16, 24, 32, 48, 48, 32, 16, 16, 8]
st = sum(counts[:li]) if li < 8 else 194 * 3 + sum(counts[8:li])
nk = 194 if li < 8 else 72
c = counts[li]
dens_ref = feats[qi, st: st + c] if li < 8 else feats[qi, 3 * 194 + (st - 3 * 194): 3 * 194 + (st - 3 * 194) + c]
print("ref density features of that layer:", np.sort(dens_ref)[::-1][:6])
print("got max", got[qi, li, 3], "want", want[qi, li, 3])
