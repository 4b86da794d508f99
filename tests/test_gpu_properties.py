"""The reference's own known-answer / property tests, run on the GPU path:

  graded transmittance closed form on a homogeneous field, 2e-3   tests/test_feature_pipeline.cpp:31-59
  graded transmittance grows with level on a constant field       tests/test_feature_pipeline.cpp:61-74
  identity combiner = mean of the upsampled levels, 1e-5          tests/test_feature_pipeline.cpp:104-130
  combiner linear in the per-level scales, 1e-5                   tests/test_feature_pipeline.cpp:132-148
  transmittance volume is vacuum (1) outside the grid             tests/test_feature_pipeline.cpp:150-158
  isotropic phase: diffuse phase features independent of omega    tests/test_feature_pipeline.cpp:298-319

plus the C ABI's determinism contract ("results must not depend on thread
count"): every query row is computed independently, so F is bit-identical whatever batch it
travels in, whether its buffers are on the device, in pinned (torch or sf.pinned_empty) or in
pageable host memory (the host path streams large batches in two windows; pinned F is written
in place by the backbone), on both precisions."""
import os

import numpy as np
import pytest

from conftest import DATA, ORIGIN

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2401_14051_b200")
from paper_2401_14051_b200 import scenes  # noqa: E402


def homogeneous(n, rho):
    return sf.DensityGrid.from_array(np.full((n, n, n), rho, np.float32), 2.0 / n, ORIGIN)


def centres(g):
    nx, ny, nz = g.dims
    vs, o = g.voxel_size(), np.asarray(g.origin())
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([o[0] + (x + 0.5) * vs, o[1] + (y + 0.5) * vs, o[2] + (z + 0.5) * vs], -1)


def test_graded_closed_form_homogeneous():
    """T_i(c) = exp(-lambda^(i+1) rho d), d = distance from c to the light-side exit."""
    rho, lam = 1.3, 0.6
    pyr = sf.DensityPyramid(homogeneous(16, rho))
    for level in range(3):
        lg = pyr.level(level)
        f = sf.graded_transmittance(pyr, level, (0.0, -1.0, 0.0), lam, 0.25 * lg.voxel_size())
        assert f.values.dims == lg.dims and f.level == level
        d = 1.0 - centres(lg)[..., 1]
        want = np.exp(-lam ** (level + 1) * rho * d)
        assert np.all(np.abs(f.values.values() - want) <= 2e-3 * want)


def test_graded_grows_with_level():
    pyr = sf.DensityPyramid(homogeneous(8, 2.0))
    light = np.array([0.3, -1.0, 0.2]) / np.linalg.norm([0.3, -1.0, 0.2])
    prev = -1.0
    for level in range(pyr.level_count()):
        f = sf.graded_transmittance(pyr, level, light, 0.6, 0.25 * pyr.level(level).voxel_size())
        v = float(f.values.sample_trilinear(np.zeros((1, 3)))[0])
        assert v > prev
        prev = v


def _fields(pyr, light):
    return [sf.graded_transmittance(pyr, i, light, 0.6, 0.25 * pyr.level(i).voxel_size())
            for i in range(pyr.level_count())]


def test_identity_combiner_is_level_mean():
    g = sf.DensityGrid.from_array(scenes.procedural_cloud(16, 7), 2.0 / 16, ORIGIN)
    pyr = sf.DensityPyramid(g)
    fields = _fields(pyr, (0.0, -1.0, 0.0))
    tv = sf.combine_transmittance(fields, sf.CombinerWeights.identity(pyr.level_count()))
    c = centres(g).reshape(-1, 3)
    mean = np.mean([f.values.sample_trilinear(c) for f in fields], axis=0)
    got = tv.values.values().reshape(-1)
    assert np.all(np.abs(got - mean) <= 1e-5 * np.abs(mean))


def test_combiner_linear_in_scales():
    pyr = sf.DensityPyramid(homogeneous(8, 1.0))
    fields = _fields(pyr, (0.0, -1.0, 0.0))
    w1 = sf.CombinerWeights.identity(pyr.level_count())
    w2 = sf.CombinerWeights(w1.kernels.copy(), (w1.scales * np.float32(3.0)).astype(np.float32))
    t1 = sf.combine_transmittance(fields, w1).values.values()
    t2 = sf.combine_transmittance(fields, w2).values.values()
    assert np.all(np.abs(t2 - 3.0 * t1) <= 1e-5 * np.abs(3.0 * t1))


@pytest.mark.parametrize("fast", [False, True])
def test_vacuum_outside_and_empty_medium(fast):
    pyr = sf.DensityPyramid(homogeneous(8, 1.0))
    tv = sf.build_transmittance_volume(pyr, (0.0, -1.0, 0.0), fast=fast)
    s = tv.sample(np.array([[5.0, 0.0, 0.0], [0.0, 0.0, 0.0]]))
    assert s[0] == 1.0 and s[1] < 1.0
    empty = sf.build_transmittance_volume(sf.DensityPyramid(homogeneous(8, 0.0)), (0.0, -1.0, 0.0), fast=fast)
    assert np.all(np.abs(empty.values.values() - 1.0) <= 1e-6)


def test_fast_build_homogeneous_close_to_exact():
    pyr = sf.DensityPyramid(homogeneous(32, 1.7))
    light = np.array([0.2, -1.0, 0.1]) / np.linalg.norm([0.2, -1.0, 0.1])
    a = sf.build_transmittance_volume(pyr, light).values.values()
    b = sf.build_transmittance_volume(pyr, light, fast=True).values.values()
    assert np.abs(a - b).max() <= 2e-5


def test_isotropic_phase_independent_of_omega():
    g = homogeneous(8, 1.0)
    pyr = sf.DensityPyramid(g)
    tv = sf.build_transmittance_volume(pyr, (0.0, -1.0, 0.0))
    dt = sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl"))
    rows = np.array([[0, 0, 0, 0, 0, 1, 0, -1, 0], [0, 0, 0, 1, 0, 0, 0, -1, 0]], np.float64)
    f = sf.sample_features(rows, dt, g, tv, sf.PhaseModel.isotropic(), sf.PhaseTable(3, 9, 9, 8))
    assert np.all(np.abs(f[0, 2] - f[1, 2]) <= 1e-6 * np.abs(f[1, 2]))
    assert np.array_equal(f[0, :2], f[1, :2])


# ---- determinism contract -----------------------------------------------------------
@pytest.fixture(scope="module")
def det():
    vol = scenes.procedural_cloud(64, 4)
    g = sf.DensityGrid.from_array(vol, 2.0 / 64, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
    scene = sf.Scene(g, tv, sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
                     sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.7),
                     sf.PhaseTable(64, 128, 32, 16))
    rows = scenes.draw_centers(vol, 30000, 21, scenes.LIGHT)  # 235 tiles: host rows arrive in 2 windows
    return scene, sf.make_backbone(sf.BackboneConfig(seed=0)), sf.MediumParams((0.7,), (0.99,) * 3), rows


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_rows_independent_of_batch_and_buffers(det, precision):
    import torch
    scene, net, med, rows = det
    prec = sf.BF16 if precision == "bf16" else sf.FP32
    ref = sf.query(scene, net, med, rows, prec)  # pageable host in / out
    dev = torch.empty((len(rows), 3), dtype=torch.float64, device="cuda")
    sf.query(scene, net, med, torch.from_numpy(rows).cuda(), prec, F_out=dev)
    assert np.array_equal(dev.cpu().numpy(), ref)
    pin_in = torch.from_numpy(rows).pin_memory()
    pin_out = torch.empty((len(rows), 3), dtype=torch.float64).pin_memory()
    sf.query(scene, net, med, pin_in.numpy(), prec, F_out=pin_out.numpy())
    assert np.array_equal(pin_out.numpy(), ref)
    hp_in, hp_out = sf.pinned_empty(rows.shape), sf.pinned_empty((len(rows), 3))  # sf_host_alloc buffers
    hp_in[:] = rows
    sf.query(scene, net, med, hp_in, prec, F_out=hp_out)
    assert np.array_equal(hp_out, ref)
    odd = sf.pinned_empty((len(rows) * 3 + 1,))[1:].reshape(-1, 3)  # 8-byte aligned F: no in-place path
    sf.query(scene, net, med, hp_in, prec, F_out=odd)
    assert np.array_equal(odd, ref)
    for a, b in ((0, 1), (1234, 5678), (14207, 30000), (100, 229)):  # sub-batches, ragged tiles
        assert np.array_equal(sf.query(scene, net, med, rows[a:b], prec), ref[a:b]), (a, b)
    perm = np.random.default_rng(5).permutation(len(rows))
    assert np.array_equal(sf.query(scene, net, med, rows[perm], prec), ref[perm])


@pytest.mark.parametrize("precision", ["fp16", "bf16", "fp32"])
def test_empty_batch(det, precision):
    """No queries: an empty F and no error on every precision (the reference's predict_field over
    an empty table returns an empty vector, src/predictor.cpp:531-543), and the next call is
    unaffected."""
    scene, net, med, rows = det
    prec = {"fp16": sf.FP16, "bf16": sf.BF16, "fp32": sf.FP32}[precision]
    F = sf.query(scene, net, med, np.empty((0, 9)), prec)
    assert F.shape == (0, 3)
    one = sf.query(scene, net, med, rows[:1], prec)
    assert one.shape == (1, 3) and np.array_equal(one, sf.query(scene, net, med, rows[:3], prec)[:1])


def test_two_lights_across_windows(det):
    """Rows lit by two lights, the second starting inside the host path's second window:
    every window compares its rows' lights with the batch's row 0 (whose light the diffuse
    constants hold), so the host-window path equals the single-window device path bit for bit
    and the FP32 path within the bf16 bound."""
    import torch
    scene, net, med, rows = det
    rows = rows.copy()
    other = np.array([0.6, -0.7, 0.3]) / np.linalg.norm([0.6, -0.7, 0.3])
    rows[20000:, 6:9] = other
    F_host = sf.query(scene, net, med, rows, sf.BF16)
    F_dev = torch.empty((len(rows), 3), dtype=torch.float64, device="cuda")
    sf.query(scene, net, med, torch.from_numpy(rows).cuda(), sf.BF16, F_out=F_dev)
    assert np.array_equal(F_dev.cpu().numpy(), F_host)
    y16 = np.empty((len(rows), 3), np.float32)
    y32 = np.empty((len(rows), 3), np.float32)
    sf.query(scene, net, med, rows[19000:21000], sf.BF16, y_out=y16[:2000])
    sf.query(scene, net, med, rows[19000:21000], sf.FP32, y_out=y32[:2000])
    assert np.all(np.abs(y16[:2000] - y32[:2000]) <= 0.03 * np.maximum(1.0, np.abs(y32[:2000])))


def test_morton_chunks_host_vs_device(monkeypatch):
    """A volume beyond L2 (256^3: queries processed in Morton order, results scattered back to
    the caller's rows) and a batch of two chunks (SF_CHUNK_CAP = 4096 tiles): F and y are
    bit-identical with device buffers, pageable and pinned host buffers, and with the same
    batch processed as one chunk (the default cap)."""
    import torch
    monkeypatch.setenv("SF_CHUNK_CAP", "4096")
    vol = scenes.noise_volume(256, 5)
    g = sf.DensityGrid.from_array(vol, 2.0 / 256, ORIGIN)
    tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT, fast=True)
    tm = (sf.load_template(os.path.join(DATA, "diffuse_seed7.vtmpl")),
          sf.load_template(os.path.join(DATA, "highlight_seed8.vtmpl")))
    sc = sf.Scene(g, tv, tm[0], tm[1], sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
    net = sf.make_backbone(sf.BackboneConfig(seed=0))
    med = sf.MediumParams((0.7,), (0.99,) * 3)
    n = 600_000  # > one 4096-tile (524,288-query) chunk
    rows = scenes.draw_centers(vol, n, 3, scenes.LIGHT)
    Fd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    yd = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    sf.query(sc, net, med, torch.from_numpy(rows).cuda(), sf.FP16, F_out=Fd, y_out=yd)
    torch.cuda.synchronize()
    yh = np.empty((n, 3), np.float32)
    Fh = sf.query(sc, net, med, rows, sf.FP16, y_out=yh)
    assert np.array_equal(Fh, Fd.cpu().numpy())
    assert np.array_equal(yh, yd.cpu().numpy())
    Fp = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    sf.query(sc, net, med, torch.from_numpy(rows).pin_memory(), sf.FP16, F_out=Fp)
    assert np.array_equal(Fp.numpy(), Fh)
    monkeypatch.delenv("SF_CHUNK_CAP")  # one chunk
    F1 = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    sf.query(sc, net, med, torch.from_numpy(rows).cuda(), sf.FP16, F_out=F1)
    assert np.array_equal(F1.cpu().numpy(), Fh)
    assert np.array_equal(sf.query(sc, net, med, rows, sf.FP16), Fh)
