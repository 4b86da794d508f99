"""Artifact formats of the reference, for drop-in I/O.

All little-endian (src/wire.h), byte-compatible with the reference's writers:

* ``.vgrid``  — DensityGrid: ``VGRD``, u32 version 1, u32 nx ny nz, f32 voxel_size,
  f32 origin xyz, f32 values x-fastest (src/volume_grid.cpp:175-238).
* ``.vfeat``  — FeatureTable: ``VFEA``, u32 version 1, u32 n_centers nd nh g_res a_res h_res
  levels, f64 lambda template_scale, per center the diffuse then the highlight
  SampleFeatureBlock (f64 p, omega, light; f32 density[n], transmittance[n], phase[n]),
  the phase table f32 values, per level 27 f32 kernel taps + f32 scale
  (src/feature_pipeline.cpp:248-338).
* ``.vnet``   — Backbone<float>: ``VNET``, u32 version 1, 64-byte SHA-256 hex of the config
  JSON, u32 json length + JSON, u32 param count, per param u32 name length + name, u32 rank,
  u32 dims, f32 values, in walk_params order (src/neural.cpp:493-549,
  src/predictor.cpp:62-109, 276-306, 631-649).
* ``.vtmpl``  — SamplingTemplate JSON: api.load_template / save_template.

Loads validate like the reference (magic, version, dims, finiteness, digest) and raise
ScatterfieldError with the reference's Errc.
"""
from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import dataclass, field

import numpy as np

from . import api
from ._lib import ScatterfieldError

# Errc ordinal + 1 (include/scatterfield_b200.h sf_status)
_IO, _MALFORMED, _BAD_DIMS, _BAD_VALUE, _TRUNCATED, _SHAPE, _PROVENANCE = 1, 2, 3, 4, 5, 7, 8


def _err(code, msg):
    return ScatterfieldError(code, msg)


class _Reader:
    def __init__(self, data: bytes, what: str):
        self.b, self.o, self.what = data, 0, what

    def take(self, n, code=_TRUNCATED):
        if self.o + n > len(self.b):
            raise _err(code, f"{self.what}: truncated")
        v = self.b[self.o:self.o + n]
        self.o += n
        return v

    def u32(self, code=_TRUNCATED):
        return struct.unpack("<I", self.take(4, code))[0]

    def f32(self, code=_TRUNCATED):
        return struct.unpack("<f", self.take(4, code))[0]

    def f64(self, code=_TRUNCATED):
        return struct.unpack("<d", self.take(8, code))[0]

    def f32s(self, n, code=_TRUNCATED):
        return np.frombuffer(self.take(4 * n, code), "<f4").astype(np.float32)


def _read(path, what):
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise _err(_IO, f"{what}: cannot open '{path}'") from e


# ---------------------------------------------------------------------------- .vgrid
def load_density_array(path):
    """load_density -> (values [nz, ny, nx] f32, voxel_size, origin) on the host."""
    r = _Reader(_read(path, "load_density"), "load_density")
    if r.take(4, _MALFORMED) != b"VGRD":
        raise _err(_MALFORMED, f"load_density: bad magic in '{path}'")
    if r.u32(_MALFORMED) != 1:
        raise _err(_MALFORMED, "load_density: unsupported version")
    dims = [r.u32(_MALFORMED) for _ in range(3)]
    vs = r.f32(_MALFORMED)
    origin = tuple(float(r.f32(_MALFORMED)) for _ in range(3))
    for d in dims:
        if d == 0 or d > (1 << 16) or d & (d - 1):
            raise _err(_BAD_DIMS, "load_density: dims must be powers of two")
    if not (vs > 0.0 and np.isfinite(vs)):
        raise _err(_BAD_VALUE, "load_density: voxel_size must be positive")
    nx, ny, nz = dims
    vals = r.f32s(nx * ny * nz).reshape(nz, ny, nx)
    if not np.all(np.isfinite(vals)):
        raise _err(_BAD_VALUE, "load_density: non-finite density")
    if np.any(vals < 0):
        raise _err(_BAD_VALUE, "load_density: negative density")
    return vals, float(vs), origin


def load_density(path) -> api.DensityGrid:
    """load_density (src/volume_grid.cpp:175-222) straight into a device DensityGrid.
    As the reference, voxel size and origin are the file's f32 values widened to f64."""
    vals, vs, origin = load_density_array(path)
    return api.DensityGrid.from_array(vals, vs, origin)


def save_density_array(values, voxel_size, origin, path):
    v = np.ascontiguousarray(values, np.float32)
    nz, ny, nx = v.shape
    if min(nx, ny, nz) <= 0 or not (voxel_size > 0):
        raise _err(_BAD_DIMS, "save_density: invalid grid")
    with open(path, "wb") as f:
        f.write(b"VGRD" + struct.pack("<4I", 1, nx, ny, nz) + struct.pack("<4f", voxel_size, *origin))
        f.write(v.astype("<f4").tobytes())


def save_density(grid: api.DensityGrid, path):
    """save_density (src/volume_grid.cpp:224-238)."""
    save_density_array(grid.values(), grid.voxel_size(), grid.origin(), path)


# ---------------------------------------------------------------------------- .vfeat
@dataclass
class FeatureTable:
    """FeatureTable (inc/feature_pipeline.h:63-70) on the host: per center the query row
    (p, omega, light) and the diffuse / highlight blocks [n, 3, points] as
    (density, transmittance, phase)."""

    centers: np.ndarray        # [n, 9] f64
    diffuse: np.ndarray        # [n, 3, nd] f32
    highlight: np.ndarray      # [n, 3, nh] f32
    phase_table: np.ndarray    # [G, A, H] f32
    kernels: np.ndarray        # [L, 27] f32
    scales: np.ndarray         # [L] f32
    lambda_: float = 0.6
    template_scale: float = 1.0
    extra: dict = field(default_factory=dict)

    def features(self):
        """[n, 3 (nd + nh)] rows in the sf_predict / sf_sample_features layout."""
        n = len(self.centers)
        return np.concatenate([self.diffuse.reshape(n, -1), self.highlight.reshape(n, -1)], axis=1)


def save_feature_table(t: FeatureTable, path):
    n = len(t.centers)
    if len(t.diffuse) != n or len(t.highlight) != n:
        raise _err(_SHAPE, "save_feature_table: center count mismatch")
    nd = t.diffuse.shape[2] if n else 0
    nh = t.highlight.shape[2] if n else 0
    G, A, H = t.phase_table.shape
    L = len(t.scales)
    out = [b"VFEA", struct.pack("<8I", 1, n, nd, nh, G, A, H, L), struct.pack("<2d", t.lambda_, t.template_scale)]
    c = np.ascontiguousarray(t.centers, "<f8")
    for i in range(n):
        for blk in (t.diffuse[i], t.highlight[i]):
            out.append(c[i].tobytes())
            out.append(np.ascontiguousarray(blk, "<f4").tobytes())
    out.append(np.ascontiguousarray(t.phase_table, "<f4").tobytes())
    kern = np.ascontiguousarray(t.kernels, "<f4")
    sc = np.ascontiguousarray(t.scales, "<f4")
    for li in range(L):
        out.append(kern[li].tobytes() + sc[li:li + 1].tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(out))


def load_feature_table(path) -> FeatureTable:
    r = _Reader(_read(path, "load_feature_table"), "load_feature_table")
    if r.take(4, _MALFORMED) != b"VFEA":
        raise _err(_MALFORMED, "load_feature_table: bad magic")
    if r.u32(_MALFORMED) != 1:
        raise _err(_MALFORMED, "load_feature_table: unsupported version")
    n, nd, nh, G, A, H, L = (r.u32(_MALFORMED) for _ in range(7))
    lam, ts = r.f64(_MALFORMED), r.f64(_MALFORMED)
    centers = np.zeros((n, 9))
    dif = np.zeros((n, 3, nd), np.float32)
    hil = np.zeros((n, 3, nh), np.float32)
    for i in range(n):
        for k, (blk, m) in enumerate(((dif, nd), (hil, nh))):
            row = np.frombuffer(r.take(72), "<f8")
            if k == 0:
                centers[i] = row
            blk[i] = r.f32s(3 * m).reshape(3, m)
    table = r.f32s(G * A * H).reshape(G, A, H)
    kern = np.zeros((L, 27), np.float32)
    sc = np.zeros(L, np.float32)
    for li in range(L):
        kern[li] = r.f32s(27)
        sc[li] = r.f32()
    return FeatureTable(centers, dif, hil, table, kern, sc, lam, ts)


def precompute_tables(centers, diffuse: api.SamplingTemplate, highlight: api.SamplingTemplate,
                      density: api.DensityGrid, tvol: api.TransmittanceFeatureVolume, model: api.PhaseModel,
                      table: api.PhaseTable, weights: api.CombinerWeights = None, cfg: api.FeatureConfig = None):
    """precompute_tables (src/feature_pipeline.cpp:213-246) on the GPU: both templates'
    feature blocks for every center, with the table / combiner / lambda / scale it was built with."""
    cfg = cfg or api.FeatureConfig()
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 9)
    fd = api.sample_features(c, diffuse, density, tvol, model, table, cfg.template_scale)
    fh = api.sample_features(c, highlight, density, tvol, model, table, cfg.template_scale)
    n = len(c)
    w = weights or tvol.weights or api.CombinerWeights.identity(1)
    return FeatureTable(c, fd.reshape(n, 3, -1), fh.reshape(n, 3, -1), table.values(),
                        np.asarray(w.kernels, np.float32), np.asarray(w.scales, np.float32), cfg.lambda_,
                        cfg.template_scale)


# ---------------------------------------------------------------------------- .vnet
_TAU = ("density", "phase", "trans")


def param_layout(cfg: api.BackboneConfig):
    """walk_params (src/predictor.cpp:62-109): [(name, shape)] in canonical order."""
    out = []
    W, M, Hh = cfg.width, cfg.merge_width, cfg.head_width
    for kind, counts in (("d", cfg.diffuse_counts), ("h", cfg.highlight_counts)):
        for tau in _TAU:
            base = f"{kind}/{tau}"
            out += [(base + "/init/W", (W, 7)), (base + "/init/b", (W,))]
            for i, cnt in enumerate(counts):
                blk = f"{base}/blk{i}"
                if not cfg.literal_attention:
                    out += [(blk + "/att/W1", (4, 8)), (blk + "/att/b1", (4,)), (blk + "/att/W2", (3, 4)),
                            (blk + "/att/b2", (3,))]
                out += [(blk + "/fc1/W", (W, W + cnt + 2)), (blk + "/fc1/b", (W,)), (blk + "/fc2/W", (W, W)),
                        (blk + "/fc2/b", (W,))]
    for tau in _TAU:
        out += [(f"merge/{tau}/W", (M, 2 * W)), (f"merge/{tau}/b", (M,))]
    out += [("merge/cross/W", (M, 3 * M)), ("merge/cross/b", (M,))]
    for l, (o, i) in enumerate(((Hh, M), (Hh, Hh), (3, Hh))):
        out += [(f"head/{l}/W", (o, i)), (f"head/{l}/b", (o,))]
    return out


def config_json(cfg: api.BackboneConfig) -> str:
    """BackboneConfig::to_json (src/predictor.cpp:276-287): nlohmann dump, keys sorted, compact."""
    return cfg.to_json()


def write_network(cfg: api.BackboneConfig, params, path):
    """save_network (src/neural.cpp:493-511) of walk_params-ordered flat parameters."""
    js = config_json(cfg).encode()
    params = np.asarray(params, np.float32)
    out = [b"VNET", struct.pack("<I", 1), hashlib.sha256(js).hexdigest().encode(), struct.pack("<I", len(js)), js]
    layout = param_layout(cfg)
    out.append(struct.pack("<I", len(layout)))
    off = 0
    for name, shape in layout:
        n = int(np.prod(shape))
        nb = name.encode()
        out.append(struct.pack("<I", len(nb)) + nb + struct.pack("<I", len(shape)) +
                   struct.pack(f"<{len(shape)}I", *shape))
        out.append(np.ascontiguousarray(params[off:off + n], "<f4").tobytes())
        off += n
    if off != len(params):
        raise _err(_SHAPE, "save_backbone: parameter count mismatch")
    with open(path, "wb") as f:
        f.write(b"".join(out))


def read_network(path):
    """load_network + the layout checks of load_backbone (src/neural.cpp:513-549,
    src/predictor.cpp:635-649) on the host: (BackboneConfig, flat f32 params)."""
    r = _Reader(_read(path, "load_network"), "load_network")
    if r.take(4, _MALFORMED) != b"VNET":
        raise _err(_MALFORMED, f"not a network file: {path}")
    if r.u32(_MALFORMED) != 1:
        raise _err(_MALFORMED, "unsupported network version")
    digest = r.take(64).decode()
    js = r.take(r.u32()).decode()
    if hashlib.sha256(js.encode()).hexdigest() != digest:
        raise _err(_PROVENANCE, f"architecture digest mismatch in {path}")
    try:
        j = json.loads(js)
        cfg = api.BackboneConfig(diffuse_counts=tuple(j["diffuse_counts"]),
                                 highlight_counts=tuple(j["highlight_counts"]), width=int(j["width"]),
                                 merge_width=int(j["merge_width"]), head_width=int(j["head_width"]),
                                 gamma=float(j["gamma"]), seed=int(j["seed"]),
                                 literal_attention=bool(j["literal_attention"]))
    except (KeyError, ValueError, TypeError) as e:
        raise _err(_MALFORMED, f"backbone config: {e}") from e
    layout = param_layout(cfg)
    if r.u32() != len(layout):
        raise _err(_SHAPE, "network file parameter count mismatch")
    vals = []
    for name, shape in layout:
        got = r.take(r.u32()).decode()
        dims = tuple(r.u32() for _ in range(r.u32()))
        if got != name or dims != tuple(shape):
            raise _err(_SHAPE, f"network file parameter layout mismatch: {got}")
        vals.append(r.f32s(int(np.prod(dims))))
    return cfg, np.concatenate(vals)


def save_backbone(net: api.Backbone, path):
    """save_backbone (src/predictor.cpp:631-633)."""
    write_network(net.config, net.params(), path)


def load_backbone(path) -> api.Backbone:
    """load_backbone (src/predictor.cpp:635-649) into a device Backbone."""
    cfg, params = read_network(path)
    return api.make_backbone(cfg, params=params)
