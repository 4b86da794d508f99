"""Python mirror of the reference's per-shading-point API (scatterfield::core).

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/core/include/scatterfield/*.h), implemented over the C ABI
of libsf_b200.so: every call runs on the GPU; there is no CPU path. Failures
raise ``ScatterfieldError`` carrying the reference ``Errc`` name.

Batched forms replace the reference's per-object calls where the reference
loops (``sample_features`` per center -> one call for many queries), with the
per-query results laid out exactly like the reference's objects.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import (SfBackboneConfig, SfMediumParams, SfPhaseModel, ScatterfieldError, check, dvec, lib,
                   ptr, stream_ptr)

DIFFUSE, HIGHLIGHT = 0, 1
FP32, BF16, FP16 = 0, 1, 2


def _arr(a, dtype):
    """Host numpy copy in C order unless `a` is a (contiguous) torch tensor."""
    if hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------- grids
class DensityGrid:
    """DensityGrid (inc/volume_grid.h:17-58), device resident. values: [nz, ny, nx]."""

    def __init__(self, nx, ny=None, nz=None, voxel_size=1.0, origin=(0.0, 0.0, 0.0), values=None,
                 _handle=None, _owner=None, _owned=False):
        self._owner = _owner
        if _handle is not None:
            self._h = _handle
            self._owned = _owned
            return
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        h = C.c_void_p()
        v = None if values is None else _arr(values, np.float32)
        check(lib.sf_grid_create(nx, ny, nz, float(voxel_size), dvec(origin), ptr(v), C.byref(h)))
        self._h = h
        self._owned = True

    @staticmethod
    def from_array(values, voxel_size, origin):
        nz, ny, nx = values.shape
        return DensityGrid(nx, ny, nz, voxel_size, origin, values)

    def _info(self):
        dims = (C.c_int * 3)()
        vs = C.c_double()
        o = (C.c_double * 3)()
        check(lib.sf_grid_info(self._h, dims, C.byref(vs), o))
        return tuple(dims), vs.value, tuple(o)

    @property
    def dims(self):
        return self._info()[0]

    def nx(self):
        return self.dims[0]

    def ny(self):
        return self.dims[1]

    def nz(self):
        return self.dims[2]

    def voxel_size(self):
        return self._info()[1]

    def origin(self):
        return self._info()[2]

    def bounds(self):
        (nx, ny, nz), vs, o = self._info()
        return (o, (o[0] + nx * vs, o[1] + ny * vs, o[2] + nz * vs))

    def device_ptr(self):
        return lib.sf_grid_device_ptr(self._h)

    def values(self, stream=None):
        nx, ny, nz = self.dims
        out = np.empty((nz, ny, nx), np.float32)
        check(lib.sf_grid_download(self._h, ptr(out), stream_ptr(stream)))
        return out

    def sample_trilinear(self, pts, stream=None):
        """DensityGrid::sample_trilinear (src/volume_grid.cpp:40-62) for [n,3] points."""
        pts = _arr(pts, np.float64).reshape(-1, 3) if not hasattr(pts, "data_ptr") else pts
        n = pts.shape[0]
        out = np.empty(n, np.float64)
        check(lib.sf_grid_sample_trilinear(self._h, n, ptr(pts), ptr(out), stream_ptr(stream)))
        return out

    def __del__(self):
        if getattr(self, "_owned", False) and self._h:
            lib.sf_grid_destroy(self._h)
            self._h = None


class DensityPyramid:
    """DensityPyramid (inc/volume_grid.h:62-72): 8-child FP64 mean down to 1^3."""

    def __init__(self, finest: DensityGrid, stream=None):
        h = C.c_void_p()
        check(lib.sf_pyramid_build(finest._h, C.byref(h), stream_ptr(stream)))
        self._h = h

    def level_count(self):
        return lib.sf_pyramid_level_count(self._h)

    def level(self, i) -> DensityGrid:
        if not 0 <= i < self.level_count():
            raise ScatterfieldError(6, "pyramid: level out of range")
        return DensityGrid(0, _handle=C.c_void_p(lib.sf_pyramid_level(self._h, i)), _owner=self)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_pyramid_destroy(self._h)
            self._h = None


def build_pyramid(grid: DensityGrid, stream=None) -> DensityPyramid:
    return DensityPyramid(grid, stream)


# ------------------------------------------------------------------- transmittance
@dataclass
class FeatureConfig:
    """FeatureConfig (inc/feature_pipeline.h:72-80)."""

    lambda_: float = 0.6
    step_scale: float = 0.5
    template_scale: float = 1.0
    phase_g_res: int = 64
    phase_angle_res: int = 128
    phase_aperture_res: int = 32
    phase_quad_nodes: int = 16


@dataclass
class CombinerWeights:
    """CombinerWeights (inc/feature_pipeline.h:30-36): [L,27] kernels + [L] scales."""

    kernels: np.ndarray
    scales: np.ndarray

    @staticmethod
    def identity(level_count):
        k = np.zeros((level_count, 27), np.float32)
        k[:, 13] = 1.0
        return CombinerWeights(k, np.full(level_count, np.float32(1.0 / level_count), np.float32))

    def level_count(self):
        return len(self.kernels)


class GradedTransmittanceField:
    """GradedTransmittanceField (inc/feature_pipeline.h:21-26)."""

    def __init__(self, level, light_dir, lambda_, values: DensityGrid):
        self.level, self.light_dir, self.lambda_, self.values = level, light_dir, lambda_, values


def _normalize(v):
    v = [float(x) for x in v]
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


def graded_transmittance(pyramid: DensityPyramid, level, light, lambda_, step, stream=None):
    """graded_transmittance (src/feature_pipeline.cpp:37-68)."""
    h = C.c_void_p()
    check(lib.sf_graded_transmittance(pyramid._h, level, dvec(light), float(lambda_), float(step), C.byref(h),
                                      stream_ptr(stream)))
    return GradedTransmittanceField(level, _normalize(light), lambda_, DensityGrid(0, _handle=h, _owned=True))


def conv3_replicate(grid: DensityGrid, kernel, stream=None) -> DensityGrid:
    """conv3_replicate (src/feature_pipeline.cpp:70-92)."""
    k = np.ascontiguousarray(kernel, np.float32).reshape(27)
    h = C.c_void_p()
    check(lib.sf_conv3_replicate(grid._h, ptr(k), C.byref(h), stream_ptr(stream)))
    return DensityGrid(0, _handle=h, _owned=True)


class TransmittanceFeatureVolume:
    """TransmittanceFeatureVolume (inc/feature_pipeline.h:38-47); sample() = 1 outside."""

    def __init__(self, handle, light_dir, weights: CombinerWeights):
        self._h = handle
        self.light_dir = light_dir
        self.weights = weights
        self.values = DensityGrid(0, _handle=C.c_void_p(lib.sf_tvol_values(handle)), _owner=self)

    @staticmethod
    def from_values(values, voxel_size, origin, light_dir, weights: CombinerWeights = None):
        """Construct from explicit level-0 values (the reference struct's public members)."""
        v = _arr(values, np.float32)
        nz, ny, nx = v.shape
        h = C.c_void_p()
        check(lib.sf_tvol_from_values(nx, ny, nz, float(voxel_size), dvec(origin), ptr(v), dvec(light_dir),
                                      C.byref(h)))
        return TransmittanceFeatureVolume(h, _normalize(light_dir), weights)

    def sample(self, pts):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        lo, hi = self.values.bounds()
        inside = np.all((pts >= lo) & (pts <= hi), axis=1)
        v = self.values.sample_trilinear(pts)
        return np.where(inside, v, 1.0)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_tvol_destroy(self._h)
            self._h = None


def combine_transmittance(fields, weights: CombinerWeights, stream=None):
    """combine_transmittance (src/feature_pipeline.cpp:94-128)."""
    if len(fields) == 0:
        raise ScatterfieldError(6, "combine_transmittance: no fields")
    if weights.level_count() != len(fields) or len(weights.scales) != len(fields):
        raise ScatterfieldError(7, "combine_transmittance: weight/level mismatch")
    l0 = fields[0].light_dir
    for f in fields:
        if math.dist(f.light_dir, l0) > 1e-9:
            raise ScatterfieldError(6, "combine_transmittance: mismatched light directions")
    arr = (C.c_void_p * len(fields))(*[f.values._h.value for f in fields])
    k = np.ascontiguousarray(weights.kernels, np.float32)
    s = np.ascontiguousarray(weights.scales, np.float32)
    h = C.c_void_p()
    check(lib.sf_combine_transmittance(arr, len(fields), ptr(k), ptr(s), dvec(l0), C.byref(h), stream_ptr(stream)))
    return TransmittanceFeatureVolume(h, l0, weights)


BUILD_FP32_MARCH = 1


def build_transmittance_volume(pyramid: DensityPyramid, light, weights: CombinerWeights = None,
                               cfg: FeatureConfig = None, stream=None, fast: bool = False):
    """build_transmittance_volume (src/feature_pipeline.cpp:200-211). fast=True marches in FP32
    (the production build for the bf16 query path, ~1e-6 relative optical depth)."""
    cfg = cfg or FeatureConfig()
    weights = weights or CombinerWeights.identity(pyramid.level_count())
    if weights.level_count() != pyramid.level_count():
        raise ScatterfieldError(7, "combine_transmittance: weight/level mismatch")
    k = np.ascontiguousarray(weights.kernels, np.float32)
    s = np.ascontiguousarray(weights.scales, np.float32)
    h = C.c_void_p()
    check(lib.sf_build_transmittance_volume_ex(pyramid._h, dvec(light), ptr(k), ptr(s), float(cfg.lambda_),
                                               float(cfg.step_scale), BUILD_FP32_MARCH if fast else 0, C.byref(h),
                                               stream_ptr(stream)))
    return TransmittanceFeatureVolume(h, _normalize(light), weights)


def build_transmittance_slab(pyramid: DensityPyramid, light, z0: int, z1: int, weights: CombinerWeights = None,
                             cfg: FeatureConfig = None, out=None, stream=None, fast: bool = False):
    """Level-0 rows [z0, z1) of build_transmittance_volume, bit-identical to the full build's
    rows (the per-light build sharded by z-slab). `out`: a CUDA tensor
    [(z1-z0), ny, nx] float32 to fill in place (stays on the device), else returns numpy."""
    cfg = cfg or FeatureConfig()
    weights = weights or CombinerWeights.identity(pyramid.level_count())
    if weights.level_count() != pyramid.level_count():
        raise ScatterfieldError(7, "combine_transmittance: weight/level mismatch")
    k = np.ascontiguousarray(weights.kernels, np.float32)
    s = np.ascontiguousarray(weights.scales, np.float32)
    g0 = pyramid.level(0)
    nx, ny, _ = g0.dims
    dst = out if out is not None else np.empty((max(z1 - z0, 0), ny, nx), np.float32)
    check(lib.sf_build_transmittance_slab(pyramid._h, dvec(light), ptr(k), ptr(s), float(cfg.lambda_),
                                          float(cfg.step_scale), BUILD_FP32_MARCH if fast else 0, int(z0), int(z1),
                                          ptr(dst), stream_ptr(stream)))
    return dst


def light_entry_point(bounds, p, light):
    """light_entry_point (src/feature_pipeline.cpp:130-137)."""
    out = (C.c_double * 3)()
    check(lib.sf_light_entry_point(dvec(bounds[0]), dvec(bounds[1]), dvec(p), dvec(light), out))
    return tuple(out)


# -------------------------------------------------------------------------- phase
@dataclass
class PhaseModel:
    """PhaseModel (inc/phase.h:13-41): kind 0 isotropic, 1 HG, 2 multi-HG."""

    kind: int = 0
    lobes: tuple = ((1.0, 0.0),)  # (weight, g)

    @staticmethod
    def isotropic():
        return PhaseModel(0, ((1.0, 0.0),))

    @staticmethod
    def hg(g):
        m = PhaseModel(1, ((1.0, float(g)),))
        m.validate()
        return m

    @staticmethod
    def multi_hg(lobes):
        m = PhaseModel(2, tuple((float(w), float(g)) for w, g in lobes))
        m.validate()
        return m

    def validate(self):
        if not self.lobes:
            raise ScatterfieldError(4, "phase: model has no lobes")
        s = 0.0
        for w, g in self.lobes:
            if not w >= 0.0:
                raise ScatterfieldError(4, "phase: lobe weight must be nonnegative")
            if not -1.0 < g < 1.0:
                raise ScatterfieldError(4, "phase: asymmetry must lie in (-1, 1)")
            s += w
        if abs(s - 1.0) > 1e-9:
            raise ScatterfieldError(4, "phase: lobe weights must sum to 1")

    def to_c(self):
        m = SfPhaseModel()
        m.kind = self.kind
        m.n_lobes = len(self.lobes)
        for i, (w, g) in enumerate(self.lobes):
            m.weight[i], m.g[i] = w, g
        return m


class PhaseTable:
    """PhaseTable (inc/phase.h:72-99): [g][angle][aperture] cap integrals, built on the GPU."""

    def __init__(self, g_res=64, angle_res=128, aperture_res=32, quad_nodes=16, stream=None, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        check(lib.sf_phase_table_build(g_res, angle_res, aperture_res, quad_nodes, C.byref(h), stream_ptr(stream)))
        self._h = h

    @staticmethod
    def from_values(g_res, angle_res, aperture_res, values):
        v = np.ascontiguousarray(values, np.float32).reshape(-1)
        if v.size != g_res * angle_res * aperture_res:
            raise ScatterfieldError(7, "phase table: value count mismatch")
        h = C.c_void_p()
        check(lib.sf_phase_table_from_values(g_res, angle_res, aperture_res, ptr(v), C.byref(h)))
        return PhaseTable(_handle=h)

    def dims(self):
        d = (C.c_int * 3)()
        check(lib.sf_phase_table_info(self._h, d))
        return tuple(d)

    def values(self):
        g, a, h = self.dims()
        out = np.empty((g, a, h), np.float32)
        check(lib.sf_phase_table_download(self._h, ptr(out), None))
        return out

    def lookup_hg(self, g, angle, half_angle):
        g, a, h = (np.ascontiguousarray(np.atleast_1d(x), np.float64) for x in (g, angle, half_angle))
        out = np.empty(len(g), np.float64)
        check(lib.sf_phase_table_lookup_hg(self._h, len(g), ptr(g), ptr(a), ptr(h), ptr(out), None))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_phase_table_destroy(self._h)
            self._h = None


# ----------------------------------------------------------------------- templates
@dataclass
class TemplateLayer:
    index: int
    radius: float
    cap_radius: float
    points: np.ndarray  # [n, 3] f64


@dataclass
class SamplingTemplate:
    """SamplingTemplate (inc/templates.h:18-34)."""

    kind: int
    seed: int
    layers: list
    gen_distance: float = 0.0
    cone_half_angle: float = 0.0
    _h: object = field(default=None, repr=False)

    def total_points(self):
        return sum(len(l.points) for l in self.layers)

    def counts(self):
        return [len(l.points) for l in self.layers]

    def handle(self):
        if self._h is None:
            counts = np.array(self.counts(), np.int32)
            pts = np.ascontiguousarray(np.concatenate([l.points for l in self.layers]).reshape(-1, 3), np.float64)
            caps = np.array([l.cap_radius for l in self.layers], np.float64)
            h = C.c_void_p()
            check(lib.sf_template_create(self.kind, len(counts), ptr(counts), ptr(pts), ptr(caps),
                                         float(self.gen_distance), float(self.cone_half_angle), C.byref(h)))
            self._h = h
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_template_destroy(self._h)
            self._h = None


def load_template(path) -> SamplingTemplate:
    """.vtmpl JSON (src/templates.cpp:286-328)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise ScatterfieldError(1, f"load_template: cannot open '{path}'") from e
    except json.JSONDecodeError as e:
        raise ScatterfieldError(2, f"load_template: {e}") from e
    try:
        kind = {"diffuse": DIFFUSE, "highlight": HIGHLIGHT}.get(j["kind"])
        if kind is None:
            raise ScatterfieldError(4, f"load_template: unknown kind '{j['kind']}'")
        layers = []
        for jl in j["layers"]:
            pts = np.array(jl["points"], np.float64).reshape(-1, 3)
            if len(pts) != jl["count"]:
                raise ScatterfieldError(5, "load_template: point count mismatch")
            layers.append(TemplateLayer(int(jl["index"]), float(jl["radius"]), float(jl["cap_radius"]), pts))
        return SamplingTemplate(kind, int(j["seed"]), layers,
                                float(j.get("gen_distance", 0.0)) if kind == HIGHLIGHT else 0.0,
                                float(j.get("cone_half_angle", 0.0)) if kind == HIGHLIGHT else 0.0)
    except KeyError as e:
        raise ScatterfieldError(2, f"load_template: missing key {e}") from e


def save_template(tmpl: SamplingTemplate, path):
    """.vtmpl JSON writer (src/templates.cpp:258-284); floats round-trip exactly."""
    j = {"kind": "diffuse" if tmpl.kind == DIFFUSE else "highlight", "seed": tmpl.seed}
    if tmpl.kind == HIGHLIGHT:
        j["gen_distance"] = tmpl.gen_distance
        j["cone_half_angle"] = tmpl.cone_half_angle
    j["layers"] = [{"index": l.index, "radius": l.radius, "cap_radius": l.cap_radius, "count": len(l.points),
                    "points": [[float(c) for c in p] for p in l.points]} for l in tmpl.layers]
    with open(path, "w") as f:
        json.dump(j, f, indent=2)
        f.write("\n")


def place_template(tmpl: SamplingTemplate, p, omega, entry, template_scale=1.0):
    """place_template + placed_cap_radii (src/templates.cpp:207-256), batched over [n,3] rows."""
    p, omega, entry = (np.ascontiguousarray(np.atleast_2d(a), np.float64) for a in (p, omega, entry))
    n, t = len(p), tmpl.total_points()
    pts = np.empty((n, t, 3), np.float64)
    caps = np.empty((n, t), np.float64)
    check(lib.sf_place_template(tmpl.handle(), n, ptr(p), ptr(omega), ptr(entry), float(template_scale),
                                ptr(pts), ptr(caps), None))
    return pts, caps


def sample_features(queries, tmpl: SamplingTemplate, density: DensityGrid, tvol: TransmittanceFeatureVolume,
                    model: PhaseModel, table: PhaseTable, template_scale=1.0, out=None, stream=None):
    """sample_features (src/feature_pipeline.cpp:139-172) for [n,9] query rows (p, omega, l).

    Returns [n, 3, npts] float32 = {density, transmittance, phase} per query."""
    q = _arr(queries, np.float64)
    n = q.shape[0] if hasattr(q, "shape") else len(q)
    if out is None:
        out = np.empty((n, 3, tmpl.total_points()), np.float32)
    m = model.to_c()
    check(lib.sf_sample_features(density._h, tvol._h, tmpl.handle(), C.byref(m), table._h, float(template_scale),
                                 n, ptr(q), ptr(out), stream_ptr(stream)))
    return out


# ------------------------------------------------------------------------ backbone
@dataclass
class BackboneConfig:
    """BackboneConfig (inc/predictor.h:33-46)."""

    diffuse_counts: tuple = (6, 8, 12, 16, 24, 32, 48, 48)
    highlight_counts: tuple = (32, 16, 16, 8)
    width: int = 32
    merge_width: int = 64
    head_width: int = 64
    gamma: float = 4.0
    seed: int = 1
    literal_attention: bool = False

    def to_c(self):
        c = SfBackboneConfig()
        c.n_diffuse_layers, c.n_highlight_layers = len(self.diffuse_counts), len(self.highlight_counts)
        for i, v in enumerate(self.diffuse_counts):
            c.diffuse_counts[i] = v
        for i, v in enumerate(self.highlight_counts):
            c.highlight_counts[i] = v
        c.width, c.merge_width, c.head_width = self.width, self.merge_width, self.head_width
        c.gamma, c.seed, c.literal_attention = self.gamma, self.seed, int(self.literal_attention)
        return c

    def to_json(self):
        """Canonical JSON digested into .vnet (src/predictor.cpp:276-288; nlohmann key order)."""
        return json.dumps({"diffuse_counts": list(self.diffuse_counts), "gamma": self.gamma,
                           "head_width": self.head_width, "highlight_counts": list(self.highlight_counts),
                           "literal_attention": self.literal_attention, "merge_width": self.merge_width,
                           "seed": self.seed, "width": self.width}, separators=(",", ":"))


class Backbone:
    """Backbone<float> (inc/predictor.h:53-56) with device-resident parameters."""

    def __init__(self, config: BackboneConfig, params=None):
        self.config = config
        c = config.to_c()
        h = C.c_void_p()
        p = None if params is None else _arr(params, np.float32)
        check(lib.sf_backbone_create(C.byref(c), ptr(p), C.byref(h)))
        self._h = h

    def param_count(self):
        return lib.sf_backbone_param_count(self._h)

    def params(self):
        out = np.empty(self.param_count(), np.float32)
        check(lib.sf_backbone_download_params(self._h, ptr(out), None))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_backbone_destroy(self._h)
            self._h = None


def make_backbone(config: BackboneConfig, params=None) -> Backbone:
    """make_backbone<float> (src/predictor.cpp:308-329): He-uniform init seeded by config.seed."""
    return Backbone(config, params)


def angle_between(a, b):
    """angle_between (inc/math.h:53-56), same FP64 operation order."""
    dot = a[0] * b[0] + a[1] * b[1] + a[2] * b[2]
    c = dot / math.sqrt((a[0] * a[0] + a[1] * a[1] + a[2] * a[2]) * (b[0] * b[0] + b[1] * b[1] + b[2] * b[2]))
    return math.acos(min(1.0, max(-1.0, c)))


@dataclass
class ConfigParams:
    """ConfigParams (inc/predictor.h:20-27)."""

    g_params: tuple
    albedo: tuple
    alpha: float = 0.0

    def row(self):
        g = list(self.g_params)[:3] + [0.0] * (3 - min(3, len(self.g_params)))
        return [float(len(self.g_params))] + g + [float(x) for x in self.albedo] + [float(self.alpha)]


def make_config(albedo, phase: PhaseModel, omega, light_dir, material_g_count=None) -> ConfigParams:
    """make_config (src/predictor.cpp:261-274) without the material-class check."""
    phase.validate()
    if phase.kind == 0:
        g = (0.0,) * (material_g_count or 1)
    else:
        g = tuple(g for _, g in phase.lobes)
    return ConfigParams(g, tuple(albedo), angle_between(omega, light_dir))


def config_rows(cfgs):
    return np.array([c.row() for c in cfgs], np.float64).reshape(-1, 8)


def predict(net: Backbone, features, config8, precision=FP32, stream=None):
    """predict_y + decode_prediction over a batch (src/predictor.cpp:389-409, 531-543).

    features: [n, 3*(nd+nh)] rows (diffuse block then highlight block);
    config8: [n, 8] rows (n_g, g0..g2, albedo.xyz, alpha). Returns (y f32 [n,3], F f64 [n,3])."""
    f = _arr(features, np.float32)
    c8 = _arr(config8, np.float64)
    n = c8.shape[0]
    y = np.empty((n, 3), np.float32)
    F = np.empty((n, 3), np.float64)
    check(lib.sf_predict(net._h, n, ptr(f), ptr(c8), precision, ptr(y), ptr(F), stream_ptr(stream)))
    return y, F


def predict_y(net: Backbone, diffuse_block, highlight_block, cfg: ConfigParams, precision=FP32):
    """predict_y (src/predictor.cpp:389-396) for one center; blocks are [3, n] arrays."""
    row = np.concatenate([np.asarray(diffuse_block, np.float32).reshape(-1),
                          np.asarray(highlight_block, np.float32).reshape(-1)])[None]
    y, _ = predict(net, row, config_rows([cfg]), precision)
    return tuple(float(v) for v in y[0])


def decode_prediction(y, albedo, gamma):
    """decode_prediction (src/predictor.cpp:406-409): F = eta^gamma * expm1(y)."""
    for a in albedo:
        if not 0.0 < a < 1.0:
            raise ScatterfieldError(4, "albedo components must lie in (0,1)")
    return tuple(math.pow(a, gamma) * math.expm1(v) for a, v in zip(albedo, y))


def encode_label(F, albedo, gamma):
    """encode_label (src/predictor.cpp:398-404)."""
    for f in F:
        if not f >= 0.0:
            raise ScatterfieldError(4, "labels must be nonnegative")
    for a in albedo:
        if not 0.0 < a < 1.0:
            raise ScatterfieldError(4, "albedo components must lie in (0,1)")
    return tuple(math.log(f / math.pow(a, gamma) + 1.0) for f, a in zip(F, albedo))


# --------------------------------------------------------------------- fused query
class Scene:
    """Bound inputs of the per-shading-point query (what render_neural holds while baking,
    src/predictor.cpp:585-614): density, transmittance feature volume, both templates,
    phase model and table, template scale."""

    def __init__(self, density: DensityGrid, tvol: TransmittanceFeatureVolume, diffuse: SamplingTemplate,
                 highlight: SamplingTemplate, model: PhaseModel, table: PhaseTable, template_scale=1.0):
        self._keep = (density, tvol, diffuse, highlight, table)
        m = model.to_c()
        h = C.c_void_p()
        check(lib.sf_scene_create(density._h, tvol._h, diffuse.handle(), highlight.handle(), C.byref(m), table._h,
                                  float(template_scale), C.byref(h)))
        self._h = h
        self.model = model

    def relight(self, pyramid: DensityPyramid, light, weights: CombinerWeights = None, cfg: FeatureConfig = None,
                fast: bool = False, stream=None):
        """Rebuild the scene's transmittance feature volume for `light` (build_transmittance_volume,
        src/feature_pipeline.cpp:200-211, as render_neural runs it per call, src/predictor.cpp:593-599)
        into the scene's own storage, asynchronously on `stream`. `pyramid` is the density's."""
        cfg = cfg or FeatureConfig()
        weights = weights or CombinerWeights.identity(pyramid.level_count())
        if weights.level_count() != pyramid.level_count():
            raise ScatterfieldError(7, "combine_transmittance: weight/level mismatch")
        k = np.ascontiguousarray(weights.kernels, np.float32)
        sc = np.ascontiguousarray(weights.scales, np.float32)
        check(lib.sf_scene_relight(self._h, pyramid._h, dvec(light), ptr(k), ptr(sc), float(cfg.lambda_),
                                   float(cfg.step_scale), BUILD_FP32_MARCH if fast else 0, stream_ptr(stream)))
        self._pyramid = pyramid
        self.light = _normalize(light)
        return self

    def tvol_storage(self):
        """The scene's own transmittance storage as a CUDA tensor view [nz, ny, nx] float32 (for a
        volume assembled outside the library, e.g. gathered z-slabs); then commit_tvol(light)."""
        import torch
        p = C.c_void_p()
        check(lib.sf_scene_tvol_storage(self._h, C.byref(p)))
        nx, ny, nz = self._keep[0].dims

        class _Cai:
            __cuda_array_interface__ = {"shape": (nz, ny, nx), "typestr": "<f4", "data": (p.value, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_Cai(), device="cuda")

    def commit_tvol(self, light, stream=None):
        check(lib.sf_scene_commit_tvol(self._h, dvec(light), stream_ptr(stream)))
        self.light = _normalize(light)
        return self

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sf_scene_destroy(self._h)
            self._h = None


@dataclass
class MediumParams:
    """The medium part of ConfigParams (g list, albedo)."""

    g: tuple
    albedo: tuple

    def to_c(self):
        m = SfMediumParams()
        m.n_g = len(self.g)
        for i, v in enumerate(self.g):
            m.g[i] = v
        for i, v in enumerate(self.albedo):
            m.albedo[i] = v
        return m


class _HostBlock:
    def __init__(self, p):
        self.p = p

    def __del__(self):
        if self.p:
            lib.sf_host_free(C.c_void_p(self.p))
            self.p = None


class PinnedArray(np.ndarray):
    """numpy array over an sf_host_alloc block; views keep the block alive through .base."""
    _block = None


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """Page-locked host array for the host-memory query path (sf_host_alloc: huge-page backed,
    registered with CUDA), so rows in / F out move at PCIe speed from the first call."""
    dt = np.dtype(dtype)
    nbytes = max(int(np.prod(shape)), 1) * dt.itemsize
    h = C.c_void_p()
    check(lib.sf_host_alloc(nbytes, C.byref(h)))
    block = _HostBlock(h.value)
    buf = (C.c_char * nbytes).from_address(h.value)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape).view(PinnedArray)
    arr._block = block
    return arr


def query(scene: Scene, net: Backbone, medium: MediumParams, queries, precision=FP32, F_out=None, y_out=None,
          stream=None):
    """The fused per-shading-point hot path: features for both templates, make_config,
    backbone forward and decode for [n,9] query rows (p, omega, l).

    Host arrays in -> host arrays out; CUDA tensors in/out stay on the device."""
    q = _arr(queries, np.float64)
    n = q.shape[0]
    if F_out is None:
        F_out = np.empty((n, 3), np.float64)
    m = medium.to_c()
    check(lib.sf_query(scene._h, net._h, C.byref(m), n, ptr(q), precision, ptr(F_out), ptr(y_out),
                       stream_ptr(stream)))
    return F_out


def debug_query_pools(scene: Scene, net: Backbone, medium: MediumParams, queries, stream=None):
    """The production sampler's fp32 per-layer pools (slice_layers' mean / max per feature type,
    src/predictor.cpp:153-191) for [n,9] query rows: [n, n_layers, 6] = mean d, p, t, max d, p, t."""
    q = _arr(queries, np.float64)
    n = q.shape[0]
    nl = len(net.config.diffuse_counts) + len(net.config.highlight_counts)
    out = np.empty((nl, n, 8), np.float32)
    m = medium.to_c()
    check(lib.sf_debug_query_pools(scene._h, net._h, C.byref(m), n, ptr(q), ptr(out), stream_ptr(stream)))
    return np.ascontiguousarray(out[:, :, :6].transpose(1, 0, 2))


def query_media(scene: Scene, net: Backbone, queries, media, precision=FP32, F_out=None, y_out=None, stream=None):
    """query() with a per-query medium: media [n, 4] = (g, albedo r, g, b), each query using
    PhaseModel.hg(g) for its phase features and ConfigParams(g=(g,), albedo) (config C4)."""
    q = _arr(queries, np.float64)
    md = _arr(media, np.float64)
    n = q.shape[0]
    if md.shape[0] != n or md.shape[-1] != 4:
        raise ScatterfieldError(7, "query_media: media must be [n, 4]")
    if F_out is None:
        F_out = np.empty((n, 3), np.float64)
    check(lib.sf_query_media(scene._h, net._h, n, ptr(q), ptr(md), precision, ptr(F_out), ptr(y_out),
                             stream_ptr(stream)))
    return F_out


# ------------------------------------------------------------------ image entry point
@dataclass
class Camera:
    """Camera (inc/camera.h:17-35): position, look_at, up, vertical fov in degrees, resolution."""

    position: tuple
    look_at: tuple = (0.0, 0.0, 0.0)
    up: tuple = (0.0, 1.0, 0.0)
    vfov: float = 40.0
    width: int = 64
    height: int = 64


@dataclass
class RenderOptions:
    """RenderOptions (inc/rte.h:145-148)."""

    step_scale: float = 0.5
    background: tuple = (0.0, 0.0, 0.0)


MATERIAL_CLASSES = {"air": 0, "gas": 1, "solid_liquid": 2, "skin": 3}


def bake_field(scene: Scene, net: Backbone, medium: MediumParams, camera_position, precision=FP32, out=None,
               stream=None):
    """bake_field (src/predictor.cpp:559-581) over the scene's density grid: F at every occupied
    voxel centre with omega toward the voxel from the camera, l = the scene tvol's light.
    Returns [3, nz, ny, nx] float32 (0 at empty voxels); `out` may be a CUDA tensor."""
    dens = scene._keep[0]
    nx, ny, nz = dens.dims
    if out is None:
        out = np.empty((3, nz, ny, nx), np.float32)
    m = medium.to_c()
    check(lib.sf_bake_field(scene._h, net._h, C.byref(m), dvec(camera_position), precision, ptr(out),
                            stream_ptr(stream)))
    return out


def render_volume(grid: DensityGrid, sigma_t, albedo, camera: Camera, field=None, opts: RenderOptions = None,
                  material_class="gas", out=None, stream=None):
    """render_volume (src/rte.cpp:407-447) with the baked field as the in-scatter provider
    (field None: F = 0). Returns the [height, width, 3] float32 image (ImageF::rgb)."""
    opts = opts or RenderOptions()
    if out is None:
        out = np.empty((camera.height, camera.width, 3), np.float32)
    f = None if field is None else _arr(field, np.float32)
    mc = MATERIAL_CLASSES[material_class] if isinstance(material_class, str) else int(material_class)
    check(lib.sf_render_volume(grid._h, dvec(sigma_t), dvec(albedo), mc, dvec(camera.position), dvec(camera.look_at),
                               dvec(camera.up), float(camera.vfov), int(camera.width), int(camera.height), ptr(f),
                               float(opts.step_scale), dvec(opts.background), ptr(out), stream_ptr(stream)))
    return out


def render_neural(grid: DensityGrid, light, camera: Camera, net: Backbone, table: PhaseTable,
                  diffuse: SamplingTemplate, highlight: SamplingTemplate, model: PhaseModel, medium: MediumParams,
                  sigma_t=(1.0, 1.0, 1.0), material_class="gas", weights: CombinerWeights = None,
                  cfg: FeatureConfig = None, opts: RenderOptions = None, precision=FP32, stream=None):
    """render_neural (src/predictor.cpp:585-614): build the transmittance feature volume for
    `light`, bake F on the density lattice, march the image."""
    cfg = cfg or FeatureConfig()
    opts = opts or RenderOptions()
    pyr = DensityPyramid(grid, stream=stream)
    tvol = build_transmittance_volume(pyr, light, weights, cfg, stream=stream)
    scene = Scene(grid, tvol, diffuse, highlight, model, table, cfg.template_scale)
    field = bake_field(scene, net, medium, camera.position, precision, stream=stream)
    return render_volume(grid, sigma_t, medium.albedo, camera, field, opts, material_class, stream=stream)
