"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-ends for the two CPU checkers of the B200 product:

* ``Oracle``  — oracle/_build/libsf_oracle.so, the plain-C restatement
  (oracle/sf_oracle.c) of the reference hot path.
* ``Reference`` — oracle/_ref/libsf_ref.so, the UNMODIFIED reference core
  (/root/reference/proj/core/src/*.cpp) compiled in place by oracle/Makefile and
  driven through oracle/ref_driver.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference / cpu_baseline
leg import this module. The product (paper_2401_14051_b200) never does.

Array conventions (shared with the product):
  grid      float32 [nz, ny, nx] (x fastest, inc/volume_grid.h:28-33)
  centers   float64 [Q, 9]  = p, omega, light
  cfg8      float64 [Q, 8]  = n_g, g0, g1, g2, albedo.xyz, alpha
  features  float32 [Q, 3*(nd+nh)] = diffuse{density,trans,phase}, highlight{...}
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsf_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def pyramid_dims(nx, ny, nz):
    dims = [(nx, ny, nz)]
    while max(dims[-1]) > 1:
        x, y, z = dims[-1]
        dims.append((max(1, x // 2), max(1, y // 2), max(1, z // 2)))
    return dims


@dataclass
class Template:
    """A SamplingTemplate as flat arrays (inc/templates.h:18-34)."""

    kind: str  # "diffuse" | "highlight"
    counts: np.ndarray  # int32 [n_layers]
    points: np.ndarray  # float64 [n_points, 3]
    caps: np.ndarray  # float64 [n_layers]  layer cap_radius
    radii: np.ndarray  # float64 [n_layers]
    gen_distance: float = 0.0
    cone_half_angle: float = 0.0
    seed: int = 0


def load_vtmpl(path) -> Template:
    """Parse the reference's .vtmpl JSON (src/templates.cpp:258-328)."""
    import json

    with open(path) as f:
        j = json.load(f)
    layers = j["layers"]
    pts = [p for l in layers for p in l["points"]]
    return Template(
        kind=j["kind"],
        counts=np.array([len(l["points"]) for l in layers], np.int32),
        points=np.array(pts, np.float64).reshape(-1, 3),
        caps=np.array([l["cap_radius"] for l in layers], np.float64),
        radii=np.array([l["radius"] for l in layers], np.float64),
        gen_distance=float(j.get("gen_distance", 0.0)),
        cone_half_angle=float(j.get("cone_half_angle", 0.0)),
        seed=int(j["seed"]),
    )


class OrScene(C.Structure):
    _fields_ = [
        ("density", C.c_void_p), ("tvol", C.c_void_p),
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("vs", C.c_double), ("origin", C.c_double * 3),
        ("nl_d", C.c_int), ("counts_d", C.c_void_p), ("pts_d", C.c_void_p), ("caps_d", C.c_void_p),
        ("nl_h", C.c_int), ("counts_h", C.c_void_p), ("pts_h", C.c_void_p), ("caps_h", C.c_void_p),
        ("gen_distance", C.c_double),
        ("phase_kind", C.c_int), ("n_lobes", C.c_int),
        ("lobe_w", C.c_double * 3), ("lobe_g", C.c_double * 3),
        ("table", C.c_void_p), ("g_res", C.c_int), ("a_res", C.c_int), ("h_res", C.c_int),
        ("template_scale", C.c_double),
    ]


class OrBackboneCfg(C.Structure):
    _fields_ = [
        ("nl_d", C.c_int), ("counts_d", C.c_int * 16),
        ("nl_h", C.c_int), ("counts_h", C.c_int * 16),
        ("width", C.c_int), ("merge_width", C.c_int), ("head_width", C.c_int),
        ("literal", C.c_int), ("gamma", C.c_double), ("seed", C.c_uint64),
    ]


@dataclass
class BackboneCfg:
    """BackboneConfig (inc/predictor.h:33-46); defaults as the reference."""

    diffuse_counts: tuple = (6, 8, 12, 16, 24, 32, 48, 48)
    highlight_counts: tuple = (32, 16, 16, 8)
    width: int = 32
    merge_width: int = 64
    head_width: int = 64
    gamma: float = 4.0
    seed: int = 1
    literal_attention: bool = False

    def to_c(self):
        c = OrBackboneCfg()
        c.nl_d = len(self.diffuse_counts)
        c.nl_h = len(self.highlight_counts)
        for i, v in enumerate(self.diffuse_counts):
            c.counts_d[i] = v
        for i, v in enumerate(self.highlight_counts):
            c.counts_h[i] = v
        c.width, c.merge_width, c.head_width = self.width, self.merge_width, self.head_width
        c.literal = int(self.literal_attention)
        c.gamma = self.gamma
        c.seed = self.seed
        return c


@dataclass
class PhaseModel:
    """PhaseModel (inc/phase.h:13-41): kind 0 isotropic, 1 HG, 2 multi-HG."""

    kind: int
    weights: tuple = (1.0,)
    gs: tuple = (0.0,)

    @staticmethod
    def hg(g):
        return PhaseModel(1, (1.0,), (float(g),))

    @staticmethod
    def isotropic():
        return PhaseModel(0, (1.0,), (0.0,))

    @staticmethod
    def multi_hg(lobes):
        return PhaseModel(2, tuple(w for w, _ in lobes), tuple(g for _, g in lobes))


class Oracle:
    """The plain-C restatement (oracle/sf_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.L = C.CDLL(path)
        L.or_sample_trilinear.restype = C.c_double
        L.or_sample_trilinear.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p]
        L.or_pyramid.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, C.POINTER(C.c_int), C.c_void_p]
        L.or_graded.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, C.c_int, _f64p,
                                C.c_double, C.c_double, _f32p]
        L.or_conv3.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        L.or_build_tvol.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p,
                                    C.c_double, C.c_double, C.c_void_p, C.c_void_p, _f32p]
        L.or_gauss_legendre.argtypes = [C.c_int, _f64p, _f64p]
        L.or_phase_table.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        L.or_lookup_hg.restype = C.c_double
        L.or_lookup_hg.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.or_light_entry_point.argtypes = [_f64p, _f64p, _f64p, _f64p, _f64p]
        L.or_features.argtypes = [C.POINTER(OrScene), C.c_int64, _f64p, _f32p]
        L.or_place_highlight.argtypes = [C.POINTER(OrScene), _f64p, _f64p, _f64p, _f64p, _f64p]
        L.or_backbone_param_count.restype = C.c_int64
        L.or_backbone_param_count.argtypes = [C.POINTER(OrBackboneCfg)]
        L.or_backbone_init.argtypes = [C.POINTER(OrBackboneCfg), _f32p]
        L.or_predict.argtypes = [C.POINTER(OrBackboneCfg), _f32p, C.c_int64, _f32p, _f64p, _f64p, _f64p]
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]

    # -- volume -------------------------------------------------------------
    def sample_trilinear(self, grid, vs, origin, p):
        nz, ny, nx = grid.shape
        return self.L.or_sample_trilinear(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                                          _c(p, np.float64))

    def pyramid(self, grid):
        nz, ny, nx = grid.shape
        dims = pyramid_dims(nx, ny, nz)
        out = np.zeros(sum(a * b * c for a, b, c in dims), np.float32)
        n = C.c_int()
        self.L.or_pyramid(_c(grid, np.float32), nx, ny, nz, out, C.byref(n), None)
        levels, off = [], 0
        for (x, y, z) in dims:
            levels.append(out[off:off + x * y * z].reshape(z, y, x))
            off += x * y * z
        return levels

    def graded(self, grid, vs, origin, level, light, lam, step):
        nz, ny, nx = grid.shape
        x, y, z = pyramid_dims(nx, ny, nz)[level]
        out = np.zeros(x * y * z, np.float32)
        rc = self.L.or_graded(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64), level,
                              _c(light, np.float64), lam, step, out)
        assert rc == 0
        return out.reshape(z, y, x)

    def conv3(self, field, k27):
        nz, ny, nx = field.shape
        out = np.zeros_like(field, dtype=np.float32)
        self.L.or_conv3(_c(field, np.float32), nx, ny, nz, _c(k27, np.float32), out)
        return out

    def build_tvol(self, grid, vs, origin, light, lam=0.6, step_scale=0.5, kernels=None, scales=None):
        nz, ny, nx = grid.shape
        out = np.zeros(grid.shape, np.float32)
        k = None if kernels is None else _c(kernels, np.float32)
        s = None if scales is None else _c(scales, np.float32)
        self.L.or_build_tvol(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                             _c(light, np.float64), lam, step_scale,
                             None if k is None else k.ctypes.data, None if s is None else s.ctypes.data, out)
        return out

    # -- phase --------------------------------------------------------------
    def gauss_legendre(self, n):
        x, w = np.zeros(n), np.zeros(n)
        self.L.or_gauss_legendre(n, x, w)
        return x, w

    def phase_table(self, g_res=64, a_res=128, h_res=32, nodes=16):
        out = np.zeros(g_res * a_res * h_res, np.float32)
        self.L.or_phase_table(g_res, a_res, h_res, nodes, out)
        return out.reshape(g_res, a_res, h_res)

    def lookup_hg(self, table, g, angle, half):
        gr, ar, hr = table.shape
        return self.L.or_lookup_hg(_c(table, np.float32), gr, ar, hr, g, angle, half)

    def light_entry_point(self, lo, hi, p, light):
        out = np.zeros(3)
        self.L.or_light_entry_point(_c(lo, np.float64), _c(hi, np.float64), _c(p, np.float64),
                                    _c(light, np.float64), out)
        return out

    # -- features -----------------------------------------------------------
    def make_scene(self, grid, tvol, vs, origin, dt: Template, ht: Template, model: PhaseModel, table,
                   template_scale=1.0):
        keep = []

        def ptr(a, dt_):
            a = _c(a, dt_)
            keep.append(a)
            return a.ctypes.data

        s = OrScene()
        nz, ny, nx = grid.shape
        s.density, s.tvol = ptr(grid, np.float32), ptr(tvol, np.float32)
        s.nx, s.ny, s.nz, s.vs = nx, ny, nz, vs
        for i in range(3):
            s.origin[i] = origin[i]
        s.nl_d, s.counts_d, s.pts_d, s.caps_d = (len(dt.counts), ptr(dt.counts, np.int32),
                                                 ptr(dt.points, np.float64), ptr(dt.caps, np.float64))
        s.nl_h, s.counts_h, s.pts_h, s.caps_h = (len(ht.counts), ptr(ht.counts, np.int32),
                                                 ptr(ht.points, np.float64), ptr(ht.caps, np.float64))
        s.gen_distance = ht.gen_distance
        s.phase_kind, s.n_lobes = model.kind, len(model.gs)
        for i, (w, g) in enumerate(zip(model.weights, model.gs)):
            s.lobe_w[i], s.lobe_g[i] = w, g
        s.table = ptr(table, np.float32)
        s.g_res, s.a_res, s.h_res = table.shape
        s.template_scale = template_scale
        s._keep = keep
        return s

    def features(self, scene, centers):
        centers = _c(centers, np.float64).reshape(-1, 9)
        nd = int(np.sum(np.ctypeslib.as_array(C.cast(scene.counts_d, C.POINTER(C.c_int)), (scene.nl_d,))))
        nh = int(np.sum(np.ctypeslib.as_array(C.cast(scene.counts_h, C.POINTER(C.c_int)), (scene.nl_h,))))
        out = np.zeros((len(centers), 3 * (nd + nh)), np.float32)
        rc = self.L.or_features(C.byref(scene), len(centers), centers, out)
        if rc != 0:
            raise ValueError("or_features: entry coincides with p")
        return out

    # -- backbone -----------------------------------------------------------
    def backbone_init(self, cfg: BackboneCfg):
        c = cfg.to_c()
        n = self.L.or_backbone_param_count(C.byref(c))
        out = np.zeros(n, np.float32)
        self.L.or_backbone_init(C.byref(c), out)
        return out

    def predict(self, cfg: BackboneCfg, params, feats, cfg8):
        feats = _c(feats, np.float32)
        cfg8 = _c(cfg8, np.float64).reshape(-1, 8)
        q = len(cfg8)
        y, F = np.zeros((q, 3)), np.zeros((q, 3))
        c = cfg.to_c()
        self.L.or_predict(C.byref(c), _c(params, np.float32), q, feats, cfg8, y, F)
        return y, F


class Reference:
    """The unmodified reference core compiled in place (oracle/_ref/libsf_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_get_threads.restype = C.c_int
        L.ref_generate_medium.argtypes = [C.c_int, C.c_int, C.c_uint64, _f32p]
        L.ref_pyramid.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f32p, C.POINTER(C.c_int)]
        L.ref_graded.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, C.c_int, _f64p,
                                 C.c_double, C.c_double, _f32p]
        L.ref_conv3.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_build_tvol.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f64p, C.c_double,
                                     C.c_double, C.c_void_p, C.c_void_p, _f32p]
        L.ref_phase_table.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        L.ref_lookup_hg.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int64, _f64p, _f64p, _f64p, _f64p]
        L.ref_gen_template.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_char_p]
        L.ref_draw_centers.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, C.c_int, C.c_uint64,
                                       _f64p, _f64p]
        L.ref_ctx_new.restype = C.c_void_p
        L.ref_ctx_new.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, _f32p, C.c_char_p,
                                  C.c_char_p, C.c_int, C.c_int, _f64p, _f64p, _f32p, C.c_int, C.c_int, C.c_int,
                                  C.c_double]
        L.ref_ctx_free.argtypes = [C.c_void_p]
        L.ref_ctx_features.argtypes = [C.c_void_p, C.c_int64, _f64p, _f32p]
        L.ref_backbone_new.restype = C.c_void_p
        L.ref_backbone_new.argtypes = [C.c_uint64, C.c_int, _i32p, C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_double]
        L.ref_backbone_free.argtypes = [C.c_void_p]
        L.ref_backbone_param_count.restype = C.c_int64
        L.ref_backbone_param_count.argtypes = [C.c_void_p]
        L.ref_backbone_get_params.argtypes = [C.c_void_p, _f32p]
        L.ref_backbone_set_params.argtypes = [C.c_void_p, _f32p]
        L.ref_backbone_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_predict.argtypes = [C.c_void_p, C.c_int64, _f32p, _f64p, _f64p, _f64p]
        L.ref_time_queries.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, _f64p, _f64p, _f64p,
                                       C.POINTER(C.c_double)]
        L.ref_save_density.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, _f64p, C.c_char_p]
        L.ref_load_density.argtypes = [C.c_char_p, _f64p, C.c_void_p]
        L.ref_save_feature_table.argtypes = [C.c_void_p, C.c_int64, _f64p, C.c_int, C.c_double, C.c_char_p]
        L.ref_render_neural.argtypes = [C.c_void_p, C.c_void_p, _f64p, _f64p, C.c_int, _f64p, _f64p, _f64p, _f64p,
                                        C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, _f64p, C.c_void_p,
                                        C.c_void_p, _f32p]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def set_threads(self, n):
        self.L.ref_set_threads(int(n))

    def generate_medium(self, kind, dims, seed):
        out = np.zeros(dims ** 3, np.float32)
        self._check(self.L.ref_generate_medium(kind, dims, seed, out))
        return out.reshape(dims, dims, dims)

    def pyramid(self, grid, vs=1.0, origin=(0, 0, 0)):
        nz, ny, nx = grid.shape
        dims = pyramid_dims(nx, ny, nz)
        out = np.zeros(sum(a * b * c for a, b, c in dims), np.float32)
        n = C.c_int()
        self._check(self.L.ref_pyramid(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64), out,
                                       C.byref(n)))
        levels, off = [], 0
        for (x, y, z) in dims:
            levels.append(out[off:off + x * y * z].reshape(z, y, x))
            off += x * y * z
        return levels

    def graded(self, grid, vs, origin, level, light, lam, step):
        nz, ny, nx = grid.shape
        x, y, z = pyramid_dims(nx, ny, nz)[level]
        out = np.zeros(x * y * z, np.float32)
        self._check(self.L.ref_graded(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64), level,
                                      _c(light, np.float64), lam, step, out))
        return out.reshape(z, y, x)

    def conv3(self, field, k27):
        nz, ny, nx = field.shape
        out = np.zeros(field.shape, np.float32)
        self._check(self.L.ref_conv3(_c(field, np.float32), nx, ny, nz, _c(k27, np.float32), out))
        return out

    def build_tvol(self, grid, vs, origin, light, lam=0.6, step_scale=0.5, kernels=None, scales=None):
        nz, ny, nx = grid.shape
        out = np.zeros(grid.shape, np.float32)
        k = None if kernels is None else _c(kernels, np.float32)
        s = None if scales is None else _c(scales, np.float32)
        self._check(self.L.ref_build_tvol(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                                          _c(light, np.float64), lam, step_scale,
                                          None if k is None else k.ctypes.data,
                                          None if s is None else s.ctypes.data, out))
        return out

    def phase_table(self, g_res=64, a_res=128, h_res=32, nodes=16):
        out = np.zeros(g_res * a_res * h_res, np.float32)
        self._check(self.L.ref_phase_table(g_res, a_res, h_res, nodes, out))
        return out.reshape(g_res, a_res, h_res)

    def lookup_hg(self, table, g, angle, half):
        g, angle, half = (_c(np.atleast_1d(a), np.float64) for a in (g, angle, half))
        out = np.zeros(len(g))
        gr, ar, hr = table.shape
        self._check(self.L.ref_lookup_hg(_c(table, np.float32), gr, ar, hr, len(g), g, angle, half, out))
        return out

    def gen_template(self, kind, seed, path, gen_distance=1.0, cone_half_angle=5.0 * np.pi / 180.0):
        self._check(self.L.ref_gen_template(0 if kind == "diffuse" else 1, seed, gen_distance,
                                            cone_half_angle, str(path).encode()))

    def draw_centers(self, grid, vs, origin, count, seed, light):
        nz, ny, nx = grid.shape
        out = np.zeros((count, 9))
        self._check(self.L.ref_draw_centers(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                                            count, seed, _c(light, np.float64), out))
        return out

    def make_ctx(self, grid, tvol, vs, origin, dt_path, ht_path, model: PhaseModel, table, template_scale=1.0):
        nz, ny, nx = grid.shape
        w = np.zeros(3)
        g = np.zeros(3)
        w[: len(model.weights)] = model.weights
        g[: len(model.gs)] = model.gs
        gr, ar, hr = table.shape
        ctx = self.L.ref_ctx_new(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                                 _c(tvol, np.float32), str(dt_path).encode(), str(ht_path).encode(),
                                 model.kind, len(model.gs), w, g, _c(table, np.float32), gr, ar, hr,
                                 template_scale)
        if not ctx:
            raise RuntimeError(self.L.ref_last_error().decode())
        return ctx

    def features(self, ctx, centers, nd, nh):
        centers = _c(centers, np.float64).reshape(-1, 9)
        out = np.zeros((len(centers), 3 * (nd + nh)), np.float32)
        self._check(self.L.ref_ctx_features(ctx, len(centers), centers, out))
        return out

    def backbone(self, cfg: BackboneCfg):
        d = np.array(cfg.diffuse_counts, np.int32)
        h = np.array(cfg.highlight_counts, np.int32)
        b = self.L.ref_backbone_new(cfg.seed, int(cfg.literal_attention), d, len(d), h, len(h), cfg.width,
                                    cfg.merge_width, cfg.head_width, cfg.gamma)
        if not b:
            raise RuntimeError(self.L.ref_last_error().decode())
        return b

    def backbone_params(self, b):
        out = np.zeros(self.L.ref_backbone_param_count(b), np.float32)
        self.L.ref_backbone_get_params(b, out)
        return out

    def predict(self, b, feats, cfg8):
        cfg8 = _c(cfg8, np.float64).reshape(-1, 8)
        q = len(cfg8)
        y, F = np.zeros((q, 3)), np.zeros((q, 3))
        self._check(self.L.ref_predict(b, q, _c(feats, np.float32), cfg8, y, F))
        return y, F

    def time_queries(self, ctx, b, centers, cfg8):
        centers = _c(centers, np.float64).reshape(-1, 9)
        cfg8 = _c(cfg8, np.float64).reshape(-1, 8)
        F = np.zeros((len(centers), 3))
        secs = C.c_double()
        self._check(self.L.ref_time_queries(ctx, b, len(centers), centers, cfg8, F, C.byref(secs)))
        return secs.value, F

    def render_neural(self, ctx, b, sigma_t, albedo, material_class, light, cam_pos, look_at, up, vfov, w, h,
                      lam=0.6, step_scale=0.5, background=(0.0, 0.0, 0.0), kernels=None, scales=None):
        """render_neural (src/predictor.cpp:585-614) with the FeatureTable combiner `kernels` [L,27] /
        `scales` [L] (None: the identity combiner): [h, w, 3] f32."""
        out = np.zeros((h, w, 3), np.float32)
        v = lambda a: _c(a, np.float64)  # noqa: E731
        k = None if kernels is None else _c(kernels, np.float32)
        s = None if scales is None else _c(scales, np.float32)
        self._check(self.L.ref_render_neural(ctx, b, v(sigma_t), v(albedo), int(material_class), v(light),
                                             v(cam_pos), v(look_at), v(up), float(vfov), int(w), int(h), lam,
                                             step_scale, v(background), None if k is None else k.ctypes.data,
                                             None if s is None else s.ctypes.data, out))
        return out

    def save_density(self, grid, vs, origin, path):
        nz, ny, nx = grid.shape
        self._check(self.L.ref_save_density(_c(grid, np.float32), nx, ny, nz, vs, _c(origin, np.float64),
                                            str(path).encode()))

    def load_density(self, path):
        info = np.zeros(7)
        self._check(self.L.ref_load_density(str(path).encode(), info, None))
        nx, ny, nz = (int(v) for v in info[:3])
        out = np.zeros((nz, ny, nx), np.float32)
        self._check(self.L.ref_load_density(str(path).encode(), info, out.ctypes.data))
        return out, info[3], info[4:7]

    def save_feature_table(self, ctx, centers, levels, lam, path):
        centers = _c(centers, np.float64).reshape(-1, 9)
        self._check(self.L.ref_save_feature_table(ctx, len(centers), centers, int(levels), float(lam),
                                                  str(path).encode()))

    def save_backbone(self, b, path):
        self._check(self.L.ref_backbone_save(b, str(path).encode()))
