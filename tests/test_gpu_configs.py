"""Configurations C3 (multi-light), C4 (per-query medium) and C5 (animated light) against the
oracle on seeded, scaled-down instances of the BASELINE.json workloads:
the same generators, smaller grids and query counts so the oracle finishes in seconds.
FP32 end to end at the C1 bar (F within 1e-3 relative, floor 1e-6 max |F|); BF16 against
the FP32 path at the stated tensor-core tolerance (test_gpu_parity.py)."""
import os

import numpy as np
import pytest

from conftest import DATA, ORIGIN, rel_err

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2401_14051_b200")
from paper_2401_14051_b200 import configs, scenes  # noqa: E402

TABLE = (9, 17, 5, 8)  # small phase table: the oracle builds the same one on the CPU


@pytest.fixture(scope="module")
def tm():
    return (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
            sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))


@pytest.fixture(scope="module")
def otab(oracle):
    return oracle.phase_table(*TABLE)


def _oracle_F(oracle, templates, otab, vol, tvol, rows, g, albedo, vs=None):
    from oracle.oracle import BackboneCfg, PhaseModel
    vs = vs or 2.0 / vol.shape[0]
    sc = oracle.make_scene(vol, tvol, vs, ORIGIN, templates[0], templates[1], PhaseModel.hg(g), otab)
    feats = oracle.features(sc, rows)
    cfg = BackboneCfg(seed=0)
    _, F = oracle.predict(cfg, oracle.backbone_init(cfg), feats, scenes.config_rows(rows, [g], albedo))
    return F


def _close(F, ref):
    return rel_err(F, ref, 1e-6 * np.abs(ref).max()).max()


def test_c3_multi_light_vs_oracle(oracle, templates, otab, tm):
    vol = scenes.smoke_plume(32, 5)
    assert 0.65 <= np.mean(vol == 0) <= 0.75  # ~70% empty voxels (C3)
    lights, inten = scenes.c3_lights()
    lights, inten = lights[:3], inten[:3]
    rows = scenes.draw_centers(vol, 96, 9, lights[0])
    g = sf.DensityGrid.from_array(vol, 2.0 / 32, ORIGIN)
    pyr = sf.DensityPyramid(g)
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((0.5,), (0.95,) * 3)
    F, per = configs.multi_light_query(g, pyr, lights, inten, rows, tm[0], tm[1], sf.PhaseModel.hg(0.5),
                                       sf.PhaseTable(*TABLE), med, net, sf.FP32)
    ref = np.zeros_like(F)
    for light, i, Fl in zip(lights, inten, per):
        tv = oracle.build_tvol(vol, 2.0 / 32, ORIGIN, np.asarray(light))
        Fo = _oracle_F(oracle, templates, otab, vol, tv, configs.with_light(rows, light), 0.5, [0.95] * 3)
        assert _close(Fl, Fo) <= 1e-3
        ref += i * Fo
    assert _close(F, ref) <= 1e-3


def test_c4_per_query_medium_vs_oracle(oracle, templates, otab, tm):
    from conftest import LIGHT
    dens, alb, gg = scenes.mixed_medium(32, 4)
    rows = scenes.draw_centers(dens, 48, 3, LIGHT)
    media = scenes.sample_media(alb, gg, rows)
    assert media[:, 0].min() >= 0.3 and media[:, 0].max() <= 0.9
    assert media[:, 1].min() >= 0.9 and media[:, 1].max() <= 0.999
    g = sf.DensityGrid.from_array(dens, 2.0 / 32, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), LIGHT)
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), sf.PhaseTable(*TABLE))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    F = sf.query_media(scene, net, rows, media, sf.FP32)
    otv = oracle.build_tvol(dens, 2.0 / 32, ORIGIN, np.asarray(LIGHT))
    ref = np.concatenate([_oracle_F(oracle, templates, otab, dens, otv, rows[i:i + 1], media[i, 0], media[i, 1:])
                          for i in range(len(rows))])
    assert _close(F, ref) <= 1e-3
    # uniform media rows == the scene-wide medium path (scene model hg(0.6)) bit for bit
    med = sf.MediumParams((0.6,), (0.97,) * 3)
    uni = np.tile([0.6, 0.97, 0.97, 0.97], (len(rows), 1))
    scene6 = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.6), sf.PhaseTable(*TABLE))
    assert np.array_equal(sf.query_media(scene, net, rows, uni, sf.FP32), sf.query(scene6, net, med, rows, sf.FP32))


def test_c4_bf16_vs_fp32(tm):
    from conftest import LIGHT
    dens, alb, gg = scenes.mixed_medium(64, 6)
    rows = scenes.draw_centers(dens, 4096, 8, LIGHT)
    media = scenes.sample_media(alb, gg, rows)
    g = sf.DensityGrid.from_array(dens, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), LIGHT)
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), sf.PhaseTable(64, 128, 32, 16))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    y32 = np.empty((len(rows), 3), np.float32)
    y16 = np.empty((len(rows), 3), np.float32)
    F32 = sf.query_media(scene, net, rows, media, sf.FP32, y_out=y32)
    F16 = sf.query_media(scene, net, rows, media, sf.BF16, y_out=y16)
    assert np.abs(y16 - y32).max() <= 0.03
    eg = media[:, 1:] ** 4
    assert np.all(np.abs(F16 - F32) <= 0.03 * (np.abs(F32) + eg))


@pytest.mark.parametrize("table", [(64, 128, 32, 16), (9, 17, 5, 8), (4, 6, 3, 8)])
def test_c4_fp16_table_quads(tm, table):
    """The production mixed-media sampler reads the phase table through 16-byte quad records
    (two rows of {P(g, a, h), P(g, a, h + 1), P(g + 1, a, h), P(g + 1, a, h + 1)}); small and odd
    table shapes (and g at the ends of the range) against the FP32 path at the fp16 bound."""
    from conftest import LIGHT
    dens, alb, gg = scenes.mixed_medium(64, 9)
    rows = scenes.draw_centers(dens, 3000, 5, LIGHT)
    media = scenes.sample_media(alb, gg, rows)
    media[:64, 0] = -0.98  # g cells at both ends of the table's g axis
    media[64:128, 0] = 0.98
    g = sf.DensityGrid.from_array(dens, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), LIGHT)
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), sf.PhaseTable(*table))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    y32 = np.empty((len(rows), 3), np.float32)
    y16 = np.empty((len(rows), 3), np.float32)
    F32 = sf.query_media(scene, net, rows, media, sf.FP32, y_out=y32)
    F16 = sf.query_media(scene, net, rows, media, sf.FP16, y_out=y16)
    assert np.all(np.isfinite(F16))
    scale = np.maximum(1.0, np.abs(y32))
    assert (np.abs(y16 - y32) / scale).max() <= 0.01
    eg = media[:, 1:] ** 4
    assert np.all(np.abs(F16 - F32) <= 0.01 * scale * (np.abs(F32) + eg))


@pytest.mark.parametrize("precision", ["fp16", "bf16"])
def test_chunking_invariance_small_chunks(tm, monkeypatch, precision):
    """F does not depend on how the batch is split into sampler / backbone chunks (the reference's
    contract that results do not depend on how work is split, inc/parallel.h:16-17): 5,000 queries
    as one chunk, as 8-tile chunks (a ragged last chunk) and as 1-tile chunks, fixed-medium and
    per-query-media paths, host and device buffers."""
    import torch
    from conftest import LIGHT
    prec = sf.FP16 if precision == "fp16" else sf.BF16
    dens, alb, gg = scenes.mixed_medium(64, 6)
    rows = scenes.draw_centers(dens, 5000, 11, LIGHT)
    media = scenes.sample_media(alb, gg, rows)
    g = sf.DensityGrid.from_array(dens, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), LIGHT, fast=True)
    scene = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.5), sf.PhaseTable(*TABLE))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((0.5,), (0.97,) * 3)
    one = sf.query(scene, net, med, rows, prec)
    one_m = sf.query_media(scene, net, rows, media, prec)
    for cap in ("8", "1"):
        monkeypatch.setenv("SF_CHUNK_CAP", cap)
        assert np.array_equal(sf.query(scene, net, med, rows, prec), one)
        assert np.array_equal(sf.query_media(scene, net, rows, media, prec), one_m)
        Fd = torch.empty((len(rows), 3), dtype=torch.float64, device="cuda")
        sf.query(scene, net, med, torch.from_numpy(rows).cuda(), prec, F_out=Fd)
        assert np.array_equal(Fd.cpu().numpy(), one)
    monkeypatch.delenv("SF_CHUNK_CAP")


def test_c5_animated_frames_vs_oracle(oracle, templates, otab, tm):
    vol = scenes.noise_volume(16, 5)
    rows = scenes.draw_centers(vol, 64, 2, scenes.LIGHT)
    g = sf.DensityGrid.from_array(vol, 2.0 / 16, ORIGIN)
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((0.7,), (0.99,) * 3)
    frames = [0, 5, 11, 24]
    Fs = configs.animated_sequence(g, 32, rows, tm[0], tm[1], sf.PhaseModel.hg(0.7), sf.PhaseTable(*TABLE), med,
                                   net, sf.FP32, frames=frames)
    for f, F in zip(frames, Fs):
        light = scenes.rotating_light(f, 32)
        tv = oracle.build_tvol(vol, 2.0 / 16, ORIGIN, np.asarray(light))
        ref = _oracle_F(oracle, templates, otab, vol, tv, configs.with_light(rows, light), 0.7, [0.99] * 3)
        assert _close(F, ref) <= 1e-3
