"""The production path (fused sample/sort + tcgen05 backbone, bf16 and fp16 operands) against the FP32 exact path
across the configuration space the reference supports: phase models (isotropic, HG, 2- and
3-lobe HG), literal attention, template scale, per-query lights (the diffuse light side is not
the precomputed one), ragged batch sizes and queries on the box boundary. Tolerance: the
stated bf16 bound of tests/test_gpu_parity.py in its scale-aware form: bf16 rounding through the
network grows with the output, so |dy| <= 0.03 max(1, |y|) and, through decode's Jacobian,
|dF| <= 0.03 max(1, |y|) (|F| + eta^gamma) (literal attention drives y to ~6 on these scenes);
fp16 operands (10-bit mantissa) the same with 0.01."""
import os

import numpy as np
import pytest

from conftest import DATA, ORIGIN

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2401_14051_b200")
from paper_2401_14051_b200 import scenes  # noqa: E402


@pytest.fixture(scope="module")
def base():
    vol = scenes.procedural_cloud(64, 2)
    g = sf.DensityGrid.from_array(vol, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
    tm = (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
          sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))
    return vol, g, tv, tm, sf.PhaseTable(64, 128, 32, 16)


def _check(scene, net, med, rows, albedo):
    """Both 16-bit operand types: bf16 within 0.03 (scale-aware), fp16 within 0.01."""
    n = len(rows)
    y32 = np.empty((n, 3), np.float32)
    F32 = sf.query(scene, net, med, rows, sf.FP32, y_out=y32)
    scale = np.maximum(1.0, np.abs(y32))
    eg = np.power(np.asarray(albedo), 4.0)
    out = None
    for prec, bound in ((sf.BF16, 0.03), (sf.FP16, 0.01)):
        y16 = np.empty((n, 3), np.float32)
        F16 = sf.query(scene, net, med, rows, prec, y_out=y16)
        assert np.all(np.isfinite(F16))
        dy = np.abs(y16 - y32)
        assert np.all(dy <= bound * scale), (prec, (dy / scale).max())
        assert np.all(np.abs(F16 - F32) <= bound * scale * (np.abs(F32) + eg))
        out = dy if out is None else out
    return out


MODELS = {
    "iso": (sf.PhaseModel.isotropic(), (0.0,)),
    "hg": (sf.PhaseModel.hg(0.7), (0.7,)),
    "hg2": (sf.PhaseModel.multi_hg([(0.7, 0.6), (0.3, -0.2)]), (0.6, -0.2)),
    "hg3": (sf.PhaseModel.multi_hg([(0.5, 0.8), (0.3, 0.1), (0.2, -0.5)]), (0.8, 0.1, -0.5)),
}


@pytest.mark.parametrize("model", list(MODELS))
def test_phase_models(base, model):
    vol, g, tv, tm, table = base
    m, gs = MODELS[model]
    scene = sf.Scene(g, tv, tm[0], tm[1], m, table)
    rows = scenes.draw_centers(vol, 1000, 3, scenes.LIGHT)
    _check(scene, sf.make_backbone(sf.BackboneConfig(seed=0)), sf.MediumParams(gs, (0.95,) * 3), rows, (0.95,) * 3)


def test_literal_attention_and_template_scale(base):
    vol, g, tv, tm, table = base
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), table, template_scale=2.5)
    rows = scenes.draw_centers(vol, 777, 5, scenes.LIGHT)
    net = sf.make_backbone(sf.BackboneConfig(seed=7, literal_attention=True))
    _check(scene, net, sf.MediumParams((0.5,), (0.9, 0.8, 0.7)), rows, (0.9, 0.8, 0.7))


def test_per_query_lights_and_directions(base):
    """Rows whose light differs from row 0's take the computed diffuse light side."""
    vol, g, tv, tm, table = base
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.7), table)
    rows = scenes.draw_centers(vol, 600, 9, scenes.LIGHT)
    rng = np.random.default_rng(0)
    other = rng.normal(size=(300, 3))
    rows[300:, 6:] = other / np.linalg.norm(other, axis=1, keepdims=True)
    rows[5, 3:6] = rows[5, 6:9]  # omega parallel to the light: highlight frame fallback
    rows[6, 3:6] = -rows[6, 6:9]
    _check(scene, sf.make_backbone(sf.BackboneConfig(seed=0)), sf.MediumParams((0.7,), (0.99,) * 3), rows,
           (0.99,) * 3)


@pytest.mark.parametrize("n", [1, 7, 127, 128, 129, 1000, 4097])
def test_ragged_batches(base, n):
    vol, g, tv, tm, table = base
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.7), table)
    rows = scenes.draw_centers(vol, n, 13 + n, scenes.LIGHT)
    _check(scene, sf.make_backbone(sf.BackboneConfig(seed=0)), sf.MediumParams((0.7,), (0.99,) * 3), rows,
           (0.99,) * 3)


def test_boundary_and_outside_points(base):
    """Shading points on the box faces and just outside (density 0 there, tvol 1)."""
    vol, g, tv, tm, table = base
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.7), table)
    rows = scenes.draw_centers(vol, 256, 17, scenes.LIGHT)
    rows[:32, 0] = 1.0
    rows[32:64, 1] = -1.0
    rows[64:96, 2] = 1.0 + 1e-3
    rows[96:128, :3] *= 0.999999
    _check(scene, sf.make_backbone(sf.BackboneConfig(seed=0)), sf.MediumParams((0.7,), (0.99,) * 3), rows,
           (0.99,) * 3)


def test_bf16_predict_nondefault_counts(small):
    """The tensor-core backbone on a non-default layer configuration (K padding, 2-slot
    highlight stack) against the FP32 backbone on the same features."""
    from conftest import rel_err  # noqa: F401
    cfg = sf.BackboneConfig(diffuse_counts=(3, 5, 9, 17, 33, 62, 40, 19), highlight_counts=(31, 20, 13, 8), seed=3)
    net = sf.make_backbone(cfg)
    rng = np.random.default_rng(1)
    n = 300
    nd, nh = sum(cfg.diffuse_counts), sum(cfg.highlight_counts)
    feats = rng.uniform(0, 1, (n, 3 * (nd + nh))).astype(np.float32)
    cfg8 = np.zeros((n, 8))
    cfg8[:, 0] = 1
    cfg8[:, 1] = 0.6
    cfg8[:, 4:7] = 0.97
    cfg8[:, 7] = rng.uniform(0, np.pi, n)
    y32, F32 = sf.predict(net, feats, cfg8, sf.FP32)
    y16, F16 = sf.predict(net, feats, cfg8, sf.BF16)
    assert np.all(np.abs(y16 - y32) <= 0.03 * np.maximum(1.0, np.abs(y32)))
    yh, Fh = sf.predict(net, feats, cfg8, sf.FP16)
    assert np.all(np.abs(yh - y32) <= 0.01 * np.maximum(1.0, np.abs(y32)))
