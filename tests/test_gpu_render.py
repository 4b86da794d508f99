"""Image entry point: bake_field + render_volume, i.e. render_neural
(src/predictor.cpp:585-614), against the reference's own image (tests/golden/render.npz)
and the oracle's baked field."""
import os

import numpy as np
import pytest

from conftest import DATA, GOLD, ORIGIN

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2401_14051_b200")


@pytest.fixture(scope="module")
def r():
    return dict(np.load(os.path.join(GOLD, "render.npz")))


@pytest.fixture(scope="module")
def setup(r):
    g = sf.DensityGrid.from_array(r["grid"], 2.0 / r["grid"].shape[0], ORIGIN)
    cam = sf.Camera(tuple(r["cam"]), tuple(r["look"]), tuple(r["up"]), float(r["vfov"]), int(r["w"]), int(r["h"]))
    tm = (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
          sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))
    table = sf.PhaseTable(*[int(x) for x in r["table"]])
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((float(r["g"]),), tuple(r["albedo"]))
    return g, cam, tm, table, net, med


def _render(r, setup, precision):
    g, cam, tm, table, net, med = setup
    opts = sf.RenderOptions(float(r["step_scale"]), tuple(r["background"]))
    cfg = sf.FeatureConfig(lambda_=float(r["lam"]), step_scale=float(r["step_scale"]))
    return sf.render_neural(g, r["light"], cam, net, table, tm[0], tm[1], sf.PhaseModel.hg(float(r["g"])), med,
                            sigma_t=tuple(r["sigma_t"]), material_class="gas", cfg=cfg, opts=opts,
                            precision=precision)


def test_render_neural_fp32_vs_reference(r, setup):
    img = _render(r, setup, sf.FP32)
    ref = r["img"]
    assert img.shape == ref.shape
    assert np.all(np.abs(img - ref) <= 1e-3 * np.abs(ref) + 1e-6 * np.abs(ref).max())


def test_bake_field_vs_oracle_and_render_exact(r, setup, oracle, templates):
    """bake_field F at every occupied voxel vs the oracle (F rel 1e-3), and render_volume fed
    the oracle's own field reproduces the reference image to FP64 march noise."""
    from test_oracle import oracle_baked_field
    g, cam, tm, table, net, med = setup
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), r["light"])
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(float(r["g"])), table)
    field = sf.bake_field(scene, net, med, tuple(r["cam"]), sf.FP32)
    want = oracle_baked_field(oracle, templates, r)
    occ = r["grid"] > 0
    assert np.all(field[:, ~occ] == 0)
    f, w = field[:, occ], want[:, occ]
    assert np.all(np.abs(f - w) <= 1e-3 * np.abs(w) + 1e-6 * np.abs(w).max())
    img = sf.render_volume(g, tuple(r["sigma_t"]), tuple(r["albedo"]), cam, want,
                           sf.RenderOptions(float(r["step_scale"]), tuple(r["background"])), "gas")
    assert np.abs(img - r["img"]).max() <= 1e-6 * np.abs(r["img"]).max()


def test_render_neural_bf16(r, setup):
    """Tensor-core path. The stated per-voxel bound |dF| <= 0.03 (|F| + eta^gamma)
    (test_gpu_parity.py) integrates along each ray to |dL| <= 0.03 (S + eta^gamma W), with
    S = sum T sigma_s F h (the in-scatter part of the pixel) and W = sum T sigma_s h (the
    same march with F = 1)."""
    g, cam, *_ = setup
    img32 = _render(r, setup, sf.FP32)
    img16 = _render(r, setup, sf.BF16)
    opts = sf.RenderOptions(float(r["step_scale"]), tuple(r["background"]))
    bg = sf.render_volume(g, tuple(r["sigma_t"]), tuple(r["albedo"]), cam, None, opts, "gas")
    ones = np.ones((3,) + r["grid"].shape, np.float32)
    W = sf.render_volume(g, tuple(r["sigma_t"]), tuple(r["albedo"]), cam, ones, opts, "gas") - bg
    S = np.abs(img32 - bg)
    eg = np.asarray(r["albedo"]) ** 4
    assert np.all(np.abs(img16 - img32) <= 0.03 * (S + eg * W) + 1e-6)
    assert S.max() > 1e-3


def test_render_errors(setup):
    import torch
    g, cam, *_ = setup
    with pytest.raises(sf.ScatterfieldError):
        sf.render_volume(g, (1, 1, 1), (0.4, 0.4, 0.4), sf.Camera((0, 0, -3), vfov=190.0))
    with pytest.raises(sf.ScatterfieldError):  # gas albedo must be <= 0.5
        sf.render_volume(g, (1, 1, 1), (0.9, 0.9, 0.9), sf.Camera((0, 0, -3)), material_class="gas")
    out = torch.empty((8, 8, 3), dtype=torch.float32, device="cuda")  # device output, empty medium
    empty = sf.DensityGrid.from_array(np.zeros((8, 8, 8), np.float32), 0.25, ORIGIN)
    sf.render_volume(empty, (1, 1, 1), (0.9, 0.9, 0.9), sf.Camera((0, 0, -3), width=8, height=8),
                     opts=sf.RenderOptions(background=(0.1, 0.2, 0.3)), material_class="solid_liquid", out=out)
    assert np.allclose(out.cpu().numpy(), np.broadcast_to([0.1, 0.2, 0.3], (8, 8, 3)))


# ---- artifact formats on the device ------------------------------
def test_io_device_round_trips(tmp_path):
    from paper_2401_14051_b200 import io
    src = os.path.join(GOLD, "io")
    net = io.load_backbone(os.path.join(src, "tiny.vnet"))
    _, params = io.read_network(os.path.join(src, "tiny.vnet"))
    assert np.array_equal(net.params(), params)
    io.save_backbone(net, str(tmp_path / "t.vnet"))
    assert (tmp_path / "t.vnet").read_bytes() == open(os.path.join(src, "tiny.vnet"), "rb").read()
    g = io.load_density(os.path.join(src, "small.vgrid"))
    io.save_density(g, str(tmp_path / "t.vgrid"))
    assert (tmp_path / "t.vgrid").read_bytes() == open(os.path.join(src, "small.vgrid"), "rb").read()


def test_precompute_tables_vs_reference_vfeat(tmp_path):
    """precompute_tables on the GPU from the reference's .vgrid reproduces the reference's
    .vfeat: features at the feature bar (1e-5 relative, floor 1e-6 max), the rest exact."""
    from conftest import LIGHT
    from paper_2401_14051_b200 import io
    src = os.path.join(GOLD, "io")
    want = io.load_feature_table(os.path.join(src, "small.vfeat"))
    g = io.load_density(os.path.join(src, "small.vgrid"))
    pyr = sf.DensityPyramid(g)
    tv = sf.build_transmittance_volume(pyr, LIGHT)
    tm = (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
          sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))
    got = io.precompute_tables(want.centers, tm[0], tm[1], g, tv, sf.PhaseModel.hg(0.7), sf.PhaseTable(9, 17, 5, 8),
                               sf.CombinerWeights.identity(pyr.level_count()), sf.FeatureConfig(template_scale=1.5))
    assert np.array_equal(got.centers, want.centers) and np.array_equal(got.kernels, want.kernels)
    assert np.array_equal(got.scales, want.scales) and (got.lambda_, got.template_scale) == (0.6, 1.5)
    assert np.abs(got.phase_table.view(np.int32).astype(np.int64) - want.phase_table.view(np.int32)).max() <= 1
    f, w = got.features(), want.features()
    assert np.all(np.abs(f - w) <= 1e-5 * np.abs(w) + 1e-6 * np.abs(w).max())
    io.save_feature_table(got, str(tmp_path / "t.vfeat"))
    assert io.load_feature_table(str(tmp_path / "t.vfeat")).features().shape == w.shape
