"""The reference's known-answer / property tests that the oracle suite (tests/test_oracle.py) pins
on the CPU, run here on the GPU path itself:

  trilinear exact on affine fields, 0 outside, exact at centres      tests/test_volume_grid.cpp:36-65
  pyramid level count, 8-child mean, top = global mean, bounds        tests/test_volume_grid.cpp:95-137
  conv3 identity exact / box kernel                                  tests/test_feature_pipeline.cpp:76-102
  placement translate + scale, highlight rotation equivariance       tests/test_templates.cpp:164-213
  zeroed output head -> y = 0 and F = 0 (FP32 and tensor-core paths) tests/test_predictor.cpp:161-180
"""
import os

import numpy as np
import pytest

from conftest import DATA, ORIGIN

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2401_14051_b200")
from paper_2401_14051_b200 import scenes  # noqa: E402


def test_trilinear_affine_fields_exact():
    n, vs = 16, 0.125
    rng = np.random.default_rng(1)
    a, b = 0.3, rng.uniform(-0.5, 0.5, 3)
    c = -1.0 + (np.arange(n) + 0.5) * vs  # voxel centres along each axis (the box is [-1, 1]^3)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    field = (a + b[0] * x + b[1] * y + b[2] * z).astype(np.float32)
    g = sf.DensityGrid.from_array(field, vs, ORIGIN)
    # inside the hull of the centres: no clamped corner, trilinear reproduces the affine field
    lo, hi = ORIGIN + 0.5 * vs, ORIGIN + (n - 0.5) * vs
    pts = rng.uniform(lo, hi, (4096, 3))
    want = a + pts @ b
    assert np.abs(g.sample_trilinear(pts) - want).max() <= 1e-5
    # exactly the stored value at every centre
    centres = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    assert np.array_equal(g.sample_trilinear(centres), field.ravel().astype(np.float64))
    # 0 outside the closed box
    out = np.array([[ORIGIN[0] - 1e-3, 0.0, 0.0], [0.0, ORIGIN[1] + n * vs + 1e-3, 0.0], [5.0, 5.0, 5.0]])
    assert np.all(g.sample_trilinear(out) == 0.0)


def test_pyramid_child_mean_and_global_mean():
    n = 32
    vol = scenes.procedural_cloud(n, 3)
    g = sf.DensityGrid.from_array(vol, 2.0 / n, ORIGIN)
    pyr = sf.DensityPyramid(g)
    assert pyr.level_count() == int(np.log2(n)) + 1
    prev = vol.astype(np.float64)
    for i in range(1, pyr.level_count()):
        lv = pyr.level(i)
        v = lv.values()
        m = prev.shape[0] // 2
        child_mean = prev.reshape(m, 2, m, 2, m, 2).mean(axis=(1, 3, 5))
        assert np.abs(v - child_mean).max() <= 1e-6
        assert np.allclose(lv.bounds(), g.bounds())
        prev = v.astype(np.float64)
    top = pyr.level(pyr.level_count() - 1).values()
    assert top.shape == (1, 1, 1)
    assert abs(float(top.ravel()[0]) - vol.astype(np.float64).mean()) <= 1e-5


def test_conv3_identity_and_box():
    n = 16
    rng = np.random.default_rng(2)
    vol = rng.uniform(0.0, 1.0, (n, n, n)).astype(np.float32)
    g = sf.DensityGrid.from_array(vol, 2.0 / n, ORIGIN)
    ident = np.zeros(27, np.float32)
    ident[13] = 1.0
    assert np.array_equal(sf.conv3_replicate(g, ident).values(), vol)
    box = np.full(27, 1.0 / 27.0, np.float32)
    got = sf.conv3_replicate(g, box).values()
    pad = np.pad(vol.astype(np.float64), 1, mode="edge")
    want = sum(pad[dz:dz + n, dy:dy + n, dx:dx + n] for dz in range(3) for dy in range(3) for dx in range(3)) / 27.0
    assert np.abs(got - want).max() <= 1e-6
    const = sf.DensityGrid.from_array(np.full((n, n, n), 0.37, np.float32), 2.0 / n, ORIGIN)
    assert np.abs(sf.conv3_replicate(const, box).values() - 0.37).max() <= 1e-6


def _rotation(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def test_placement_translate_scale_and_rotation_equivariance():
    dt = sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl"))
    ht = sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl"))
    rng = np.random.default_rng(3)
    m = 64
    p = rng.uniform(-0.8, 0.8, (m, 3))
    w = rng.normal(size=(m, 3))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    entry = p + rng.uniform(0.2, 0.6, (m, 1)) * np.array([0.2, 1.0, -0.1])
    # diffuse: a pure translation of the scaled template
    base, _ = sf.place_template(dt, np.zeros((1, 3)), w[:1], np.zeros((1, 3)) + 1.0, 1.0)
    for s in (1.0, 0.25):
        pts, _ = sf.place_template(dt, p, w, entry, s)
        assert np.abs(pts - (p[:, None, :] + s * base)).max() <= 1e-12
    # highlight: rotating p, omega and the entry rotates the placed points (about the origin)
    R = _rotation(rng)
    pts, caps = sf.place_template(ht, p, w, entry, 1.0)
    ptsR, capsR = sf.place_template(ht, p @ R.T, w @ R.T, entry @ R.T, 1.0)
    assert np.abs(ptsR - pts @ R.T).max() <= 1e-9
    assert np.abs(capsR - caps).max() <= 1e-12


def test_zeroed_head_gives_zero_output():
    vol = scenes.procedural_cloud(64, 2)
    g = sf.DensityGrid.from_array(vol, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
    sc = sf.Scene(g, tv, sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
                  sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7),
                  sf.PhaseTable(64, 128, 32, 16))
    cfg = sf.BackboneConfig(seed=0)
    params = sf.make_backbone(cfg).params()
    params[-(3 * 64 + 3):] = 0.0  # the 64 -> 3 output layer (walk_params' last tensors)
    net = sf.make_backbone(cfg, params)
    rows = scenes.draw_centers(vol, 1000, 4, scenes.LIGHT)
    med = sf.MediumParams((0.7,), (0.99,) * 3)
    for prec in (sf.FP32, sf.BF16, sf.FP16):
        y = np.empty((len(rows), 3), np.float32)
        F = sf.query(sc, net, med, rows, prec, y_out=y)
        assert np.all(y == 0.0) and np.all(F == 0.0), prec
