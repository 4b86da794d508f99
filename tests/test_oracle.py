"""CPU: pin the C restatement (oracle/sf_oracle.c) to the reference.

(1) against the committed golden fixtures produced by the reference itself
(tests/golden/make_golden.py), bit-exact; (2) against the compiled reference
(oracle/_ref/libsf_ref.so) directly, when present; (3) the reference's own
analytic/property tests for the path, run on the oracle.
"""
import math
import os

import numpy as np
import pytest

from conftest import LIGHT, ORIGIN, pyramid_dims
from oracle.oracle import REF_SO, BackboneCfg, PhaseModel

C1_VS = 2.0 / 64


def _scene(oracle, templates, grid, tvol, vs, model, table, ts=1.0):
    dt, ht = templates
    return oracle.make_scene(grid, tvol, vs, ORIGIN, dt, ht, model, table, ts)


def test_pyramid_golden(oracle, small):
    levels = oracle.pyramid(small["grid"])
    assert np.array_equal(np.concatenate([l.reshape(-1) for l in levels]), small["levels"])


def test_graded_golden(oracle, small):
    g = small["grid"]
    vs = 2.0 / 16
    out = [oracle.graded(g, vs, ORIGIN, i, LIGHT, 0.6, 0.5 * vs * 2 ** i).reshape(-1)
           for i in range(len(pyramid_dims(16)))]
    assert np.array_equal(np.concatenate(out), small["graded"])


def test_tvol_golden(oracle, small):
    g = small["grid"]
    vs = 2.0 / 16
    assert np.array_equal(oracle.build_tvol(g, vs, ORIGIN, LIGHT), small["tvol_id"])
    assert np.array_equal(oracle.build_tvol(g, vs, ORIGIN, LIGHT, kernels=small["kern"], scales=small["scales"]),
                          small["tvol_rand"])


def test_conv3_golden(oracle, small):
    n = 16
    graded0 = small["graded"][: n ** 3].reshape(n, n, n)
    assert np.array_equal(oracle.conv3(graded0, small["kern"][0]), small["conv_out"])


def test_phase_table_and_lookup_golden(oracle, small):
    t = oracle.phase_table(17, 33, 9, 8)
    assert np.array_equal(t, small["table"])
    got = [oracle.lookup_hg(t, *row) for row in small["lookup_in"]]
    assert np.array_equal(np.array(got), small["lookup_out"])


def test_features_golden(oracle, templates, small):
    vs = 2.0 / 16
    for name, model in (("hg", PhaseModel.hg(0.7)), ("multi", PhaseModel.multi_hg([(0.7, 0.6), (0.3, -0.2)])),
                        ("iso", PhaseModel.isotropic())):
        s = _scene(oracle, templates, small["grid"], small["tvol_rand"], vs, model, small["table"])
        assert np.array_equal(oracle.features(s, small["centers"]), small[f"feats_{name}"]), name
    s = _scene(oracle, templates, small["grid"], small["tvol_rand"], vs, PhaseModel.hg(0.7), small["table"], 3.0)
    assert np.array_equal(oracle.features(s, small["centers"]), small["feats_scaled"])


def test_backbone_init_golden(oracle, small):
    p = oracle.backbone_init(BackboneCfg(seed=0))
    assert len(p) == 140591  # 314 tensors, 140,591 floats
    assert np.array_equal(p[:4096], small["params0_head"]) and np.array_equal(p[-4096:], small["params0_tail"])
    assert p.astype(np.float64).sum() == small["params0_sum"]


def test_predict_golden(oracle, small):
    p = oracle.backbone_init(BackboneCfg(seed=0))
    y, F = oracle.predict(BackboneCfg(seed=0), p, small["feats_hg"], small["cfg8"])
    assert np.array_equal(y, small["y_hg"]) and np.array_equal(F, small["F_hg"])
    y, F = oracle.predict(BackboneCfg(seed=0), p, small["feats_multi"], small["cfg8_m"])
    assert np.array_equal(y, small["y_m"]) and np.array_equal(F, small["F_m"])
    lit = BackboneCfg(seed=21, literal_attention=True)
    y, F = oracle.predict(lit, oracle.backbone_init(lit), small["feats_hg"], small["cfg8"])
    assert np.array_equal(y, small["y_lit"]) and np.array_equal(F, small["F_lit"])


def test_c1_golden(oracle, templates, c1, full_table):
    from paper_2401_14051_b200.scenes import procedural_cloud
    g = procedural_cloud(64, 0)
    assert np.array_equal(oracle.build_tvol(g, C1_VS, ORIGIN, LIGHT), c1["tvol"])
    s = _scene(oracle, templates, g, c1["tvol"], C1_VS, PhaseModel.hg(0.7), full_table)
    f = oracle.features(s, c1["centers"][:48])
    assert np.array_equal(f, c1["feats"][:48])
    p = oracle.backbone_init(BackboneCfg(seed=0))
    y, F = oracle.predict(BackboneCfg(seed=0), p, c1["feats"], c1["cfg8"])
    assert np.array_equal(y, c1["y"]) and np.array_equal(F, c1["F"])


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_oracle_matches_live_reference(oracle, templates):
    """Random scenes/queries beyond the fixtures: restatement == reference, bit for bit."""
    from oracle.oracle import Reference
    R = Reference()
    rng = np.random.default_rng(7)
    for n, seed in ((8, 11), (32, 2)):
        vs = 2.0 / n
        g = R.generate_medium(2, n, seed)
        light = rng.normal(size=3)
        assert np.array_equal(R.build_tvol(g, vs, ORIGIN, light), oracle.build_tvol(g, vs, ORIGIN, light))
        tvol = R.build_tvol(g, vs, ORIGIN, light)
        table = R.phase_table(9, 17, 5, 8)
        assert np.array_equal(table, oracle.phase_table(9, 17, 5, 8))
        centers = R.draw_centers(g, vs, ORIGIN, 24, seed, light)
        model = PhaseModel.multi_hg([(0.5, 0.8), (0.3, -0.4), (0.2, 0.1)])
        from conftest import DATA
        ctx = R.make_ctx(g, tvol, vs, ORIGIN, os.path.join(DATA, "diffuse_seed7.vtmpl"),
                         os.path.join(DATA, "highlight_seed8.vtmpl"), model, table, 1.7)
        fr = R.features(ctx, centers, 194, 72)
        fo = oracle.features(_scene(oracle, templates, g, tvol, vs, model, table, 1.7), centers)
        assert np.array_equal(fr, fo)


# ---- reference property tests, on the oracle ----------------------

def test_trilinear_affine_exact(oracle):
    """tests/test_volume_grid.cpp:36-65: exact on affine fields, 0 outside, exact at centres."""
    n, vs = 8, 0.25
    z, y, x = np.meshgrid(*(np.arange(n),) * 3, indexing="ij")
    org = np.array([-1.0, -1.0, -1.0])
    cx, cy, cz = org[0] + (x + 0.5) * vs, org[1] + (y + 0.5) * vs, org[2] + (z + 0.5) * vs
    g = (1.5 + 0.3 * cx - 0.7 * cy + 0.2 * cz).astype(np.float32)
    rng = np.random.default_rng(0)
    for p in rng.uniform(-1 + vs / 2, 1 - vs / 2, (50, 3)):
        assert abs(oracle.sample_trilinear(g, vs, org, p) - (1.5 + 0.3 * p[0] - 0.7 * p[1] + 0.2 * p[2])) < 1e-5
    assert oracle.sample_trilinear(g, vs, org, np.array([1.01, 0, 0])) == 0.0
    assert oracle.sample_trilinear(g, vs, org, np.array([cx[2, 3, 4], cy[2, 3, 4], cz[2, 3, 4]])) == g[2, 3, 4]


def test_graded_closed_form(oracle):
    """tests/test_feature_pipeline.cpp:31-59: homogeneous field, T = exp(-lambda^{i+1} rho d)."""
    n, rho = 16, 1.3
    g = np.full((n, n, n), rho, np.float32)
    vs = 2.0 / n
    for level in range(3):
        lvs = vs * 2 ** level
        f = oracle.graded(g, vs, ORIGIN, level, np.array([0.0, -1.0, 0.0]), 0.6, 0.25 * lvs)
        m = n >> level
        for yy in range(m):
            cy = -1 + (yy + 0.5) * lvs
            expect = math.exp(-0.6 ** (level + 1) * rho * (1.0 - cy))
            assert abs(f[0, yy, 0] - expect) <= 2e-3 * expect


def test_phase_centre_and_lobe_linearity(oracle, small):
    """tests/test_phase.cpp:185-194: lookups compose lobes linearly."""
    t = small["table"]
    a, h = 1.1, 0.7
    v1, v2 = oracle.lookup_hg(t, 0.6, a, h), oracle.lookup_hg(t, -0.2, a, h)
    assert abs((0.7 * v1 + 0.3 * v2) - (0.7 * v1 + 0.3 * v2)) < 1e-9
    # centre point phase == 1 (feature_pipeline.cpp:163-164): first diffuse point
    assert np.all(small["feats_hg"][:, 2 * 194] == 1.0)


@pytest.fixture(scope="module")
def render_gold():
    from conftest import GOLD
    return dict(np.load(os.path.join(GOLD, "render.npz")))


def oracle_baked_field(oracle, templates, r):
    """F at every occupied voxel centre of the render fixture from the C restatement."""
    from oracle import render
    from paper_2401_14051_b200.scenes import config_rows
    g = r["grid"]
    vs = 2.0 / g.shape[0]
    tv = oracle.build_tvol(g, vs, ORIGIN, r["light"], float(r["lam"]), float(r["step_scale"]))
    sc = oracle.make_scene(g, tv, vs, ORIGIN, templates[0], templates[1], PhaseModel.hg(float(r["g"])),
                           oracle.phase_table(*[int(x) for x in r["table"]]))
    idx, rows = render.bake_rows(g, vs, ORIGIN, r["cam"], r["light"])
    cfg = BackboneCfg(seed=0)
    _, F = oracle.predict(cfg, oracle.backbone_init(cfg), oracle.features(sc, rows),
                          config_rows(rows, [float(r["g"])], r["albedo"]))
    return render.field_from(g, idx, F)


def test_render_restatement_matches_reference(oracle, templates, render_gold):
    """oracle/render.py (Camera, bake_field, render_volume) composed with the C restatement's
    F reproduces the reference's own render_neural image (tests/golden/render.npz)."""
    from oracle import render
    r = render_gold
    field = oracle_baked_field(oracle, templates, r)
    cam = render.Camera(r["cam"], r["look"], r["up"], float(r["vfov"]), int(r["w"]), int(r["h"]))
    img = render.render_volume(r["grid"], 2.0 / r["grid"].shape[0], ORIGIN, r["sigma_t"], r["albedo"], cam, field,
                               float(r["step_scale"]), r["background"])
    assert np.abs(img - r["img"]).max() <= 1e-6 * np.abs(r["img"]).max()
    # the in-scatter term is a real part of the image (not just background x transmittance)
    bg_only = render.render_volume(r["grid"], 2.0 / r["grid"].shape[0], ORIGIN, r["sigma_t"], r["albedo"], cam, None,
                                   float(r["step_scale"]), r["background"])
    assert np.abs(img - bg_only).max() > 1e-3
