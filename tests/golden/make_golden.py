"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Runs only in the build container (needs oracle/_ref/libsf_ref.so, i.e. the
reference core compiled from /root/reference by `make -C oracle ref`). The
outputs are committed; tests (CPU and GPU) read them without /root/reference.

  python tests/golden/make_golden.py

Fixtures
  templates : paper_2401_14051_b200/data/{diffuse_seed7,highlight_seed8}.vtmpl
              (generate_*_template as in tests/acceptance.cpp:607-609) — also the
              product's default templates.
  small.npz : 16^3 cloud (seed 3): pyramid, graded fields, identity + random
              combiner tvols, conv3, phase table (17,33,9,8), lookups, 48 centers,
              features (HG 0.7 and 2-lobe HG), y/F for backbone seed 0 and a tiny
              literal-attention config.
  c1.npz    : config 1 (64^3 cloud seed 0, HG g=0.7, albedo 0.99): tvol, 192
              centers, features with the full (64,128,32,16) table, y and F.
  phase_table_full.npz : PhaseTable(64,128,32,16) values.
  render.npz: render_neural (src/predictor.cpp:585-614) of the small 16^3 cloud: gas
              medium (sigma_t 14/12/10, albedo 0.45/0.40/0.35), HG 0.7, table (17,33,9,8),
              backbone seed 0, camera (0.3,0.2,-3.5) -> origin, vfov 40, 24x16, background
              (0.05,0.1,0.2). `python tests/golden/make_golden.py render` regenerates only it.
  render_rc.npz: the same render with a seeded random combiner in the FeatureTable (kernels,
              scales, image).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import BackboneCfg, PhaseModel, Reference, load_vtmpl  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2401_14051_b200", "data")
LIGHT = np.array([0.2, -1.0, 0.1])
LIGHT = LIGHT / np.sqrt(LIGHT @ LIGHT)
ORIGIN = np.array([-1.0, -1.0, -1.0])


def cfg_rows(R, centers, g, albedo):
    from paper_2401_14051_b200.scenes import config_rows
    return config_rows(centers, g, albedo)


RENDER = dict(sigma_t=(14.0, 12.0, 10.0), albedo=(0.45, 0.40, 0.35), g=0.7, table=(17, 33, 9, 8),
              cam=(0.3, 0.2, -3.5), look=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), vfov=40.0, w=24, h=16,
              background=(0.05, 0.1, 0.2), step_scale=0.5, lam=0.6)


def render_fixture(R):
    n, vs = 16, 2.0 / 16
    g = R.generate_medium(2, n, 3)
    r = RENDER
    tvol = R.build_tvol(g, vs, ORIGIN, LIGHT)
    ctx = R.make_ctx(g, tvol, vs, ORIGIN, os.path.join(DATA, "diffuse_seed7.vtmpl"),
                     os.path.join(DATA, "highlight_seed8.vtmpl"), PhaseModel.hg(r["g"]), R.phase_table(*r["table"]))
    b = R.backbone(BackboneCfg(seed=0))
    img = R.render_neural(ctx, b, r["sigma_t"], r["albedo"], 1, LIGHT, r["cam"], r["look"], r["up"], r["vfov"],
                          r["w"], r["h"], r["lam"], r["step_scale"], r["background"])
    np.savez_compressed(os.path.join(GOLD, "render.npz"), grid=g, img=img, light=LIGHT,
                        **{k: np.asarray(v, np.float64) for k, v in r.items()})
    # the same scene with a seeded random FeatureTable combiner (the 3D-CNN weights render_neural
    # takes from the table, src/predictor.cpp:593-599): kernels U(-0.2, 0.2) + 1 at the centre tap
    L = 5
    rng = np.random.default_rng(11)
    kern = rng.uniform(-0.2, 0.2, (L, 27)).astype(np.float32)
    kern[:, 13] += 1.0
    scales = np.full(L, 1.0 / L, np.float32)
    img_rc = R.render_neural(ctx, b, r["sigma_t"], r["albedo"], 1, LIGHT, r["cam"], r["look"], r["up"], r["vfov"],
                             r["w"], r["h"], r["lam"], r["step_scale"], r["background"], kern, scales)
    np.savez_compressed(os.path.join(GOLD, "render_rc.npz"), img=img_rc, kernels=kern, scales=scales)


def io_fixtures(R):
    """Reference-written artifacts (tests/golden/io/): small.vgrid (16^3 cloud seed 3, origin
    (-1,-1,-1), vs 1/8), small.vfeat (precompute_tables of 4 centers on it, HG 0.7, table
    (9,17,5,8), identity combiner, lambda 0.6, template scale 1.5), tiny.vnet (backbone
    counts (2,3)/(2,), widths 4/8/8, seed 5) and lit.vnet (same with literal attention)."""
    out = os.path.join(GOLD, "io")
    os.makedirs(out, exist_ok=True)
    n, vs = 16, 2.0 / 16
    g = R.generate_medium(2, n, 3)
    R.save_density(g, vs, ORIGIN, os.path.join(out, "small.vgrid"))
    tv = R.build_tvol(g, vs, ORIGIN, LIGHT)
    ctx = R.make_ctx(g, tv, vs, ORIGIN, os.path.join(DATA, "diffuse_seed7.vtmpl"),
                     os.path.join(DATA, "highlight_seed8.vtmpl"), PhaseModel.hg(0.7), R.phase_table(9, 17, 5, 8),
                     template_scale=1.5)
    centers = R.draw_centers(g, vs, ORIGIN, 4, 5, LIGHT)
    R.save_feature_table(ctx, centers, 5, 0.6, os.path.join(out, "small.vfeat"))
    for name, lit in (("tiny", False), ("lit", True)):
        b = R.backbone(BackboneCfg(diffuse_counts=(2, 3), highlight_counts=(2,), width=4, merge_width=8,
                                   head_width=8, seed=5, literal_attention=lit))
        R.save_backbone(b, os.path.join(out, f"{name}.vnet"))


def main():
    R = Reference()
    if sys.argv[1:] == ["render"]:
        render_fixture(R)
        return
    if sys.argv[1:] == ["io"]:
        io_fixtures(R)
        return
    os.makedirs(DATA, exist_ok=True)
    dpath = os.path.join(DATA, "diffuse_seed7.vtmpl")
    hpath = os.path.join(DATA, "highlight_seed8.vtmpl")
    R.gen_template("diffuse", 7, dpath)
    R.gen_template("highlight", 8, hpath, gen_distance=1.0, cone_half_angle=5.0 * np.pi / 180.0)
    dt, ht = load_vtmpl(dpath), load_vtmpl(hpath)
    nd, nh = int(dt.counts.sum()), int(ht.counts.sum())

    # ---------------- small scene
    n = 16
    vs = 2.0 / n
    g = R.generate_medium(2, n, 3)
    levels = R.pyramid(g, vs, ORIGIN)
    graded = [R.graded(g, vs, ORIGIN, i, LIGHT, 0.6, 0.5 * vs * 2 ** i) for i in range(len(levels))]
    tvol_id = R.build_tvol(g, vs, ORIGIN, LIGHT)
    rng = np.random.default_rng(1234)
    L = len(levels)
    kern = rng.uniform(-0.2, 0.2, (L, 27)).astype(np.float32)
    kern[:, 13] += 1.0
    scales = np.full(L, np.float32(1.0 / L), np.float32)
    tvol_rand = R.build_tvol(g, vs, ORIGIN, LIGHT, kernels=kern, scales=scales)
    conv_in = graded[0]
    conv_out = R.conv3(conv_in, kern[0])
    table_s = R.phase_table(17, 33, 9, 8)
    lk = rng.uniform(0, 1, (256, 3)) * [1.98, np.pi, np.pi] - [0.99, 0, 0]
    lk[:8] = [[-0.99, 0, 0], [0.99, np.pi, np.pi], [0.5, 0, np.pi], [-1.5, -0.2, 4.0],
              [1.2, 3.5, -1.0], [0.0, np.pi / 2, 0.0], [0.3, 1.0, 1e-9], [0.98999, 3.14159, 3.14159]]
    lk_out = R.lookup_hg(table_s, lk[:, 0], lk[:, 1], lk[:, 2])
    centers = R.draw_centers(g, vs, ORIGIN, 48, 5, LIGHT)
    # edge rows: p outside the box, on a face, and a far-away template scale is separate
    centers[0, :3] = [1.5, 0.2, -0.3]
    centers[1, :3] = [0.25, 1.0, 0.1]
    centers[2, 3:6] = LIGHT  # omega parallel to the light -> highlight frame fallback
    m_hg = PhaseModel.hg(0.7)
    m_2 = PhaseModel.multi_hg([(0.7, 0.6), (0.3, -0.2)])
    m_iso = PhaseModel.isotropic()
    feats = {}
    for name, m in (("hg", m_hg), ("multi", m_2), ("iso", m_iso)):
        ctx = R.make_ctx(g, tvol_rand, vs, ORIGIN, dpath, hpath, m, table_s)
        feats[name] = R.features(ctx, centers, nd, nh)
    ctx = R.make_ctx(g, tvol_rand, vs, ORIGIN, dpath, hpath, m_hg, table_s, template_scale=3.0)
    feats_scaled = R.features(ctx, centers, nd, nh)

    bb = BackboneCfg(seed=0)
    b = R.backbone(bb)
    params0 = R.backbone_params(b)
    cfg8 = cfg_rows(R, centers, [0.7], [0.99, 0.99, 0.99])
    y_hg, F_hg = R.predict(b, feats["hg"], cfg8)
    cfg8_m = cfg_rows(R, centers, [0.6, -0.2], [0.9, 0.85, 0.8])
    y_m, F_m = R.predict(b, feats["multi"], cfg8_m)
    tiny = BackboneCfg(diffuse_counts=(6, 8, 12, 16, 24, 32, 48, 48), highlight_counts=(32, 16, 16, 8),
                       width=32, merge_width=64, head_width=64, seed=21, literal_attention=True)
    bt = R.backbone(tiny)
    y_lit, F_lit = R.predict(bt, feats["hg"], cfg8)

    np.savez_compressed(
        os.path.join(GOLD, "small.npz"),
        grid=g, levels=np.concatenate([l.reshape(-1) for l in levels]), graded=np.concatenate(
            [x.reshape(-1) for x in graded]), tvol_id=tvol_id, tvol_rand=tvol_rand, kern=kern, scales=scales,
        conv_out=conv_out, table=table_s, lookup_in=lk, lookup_out=lk_out, centers=centers,
        feats_hg=feats["hg"], feats_multi=feats["multi"], feats_iso=feats["iso"], feats_scaled=feats_scaled,
        params0_sum=np.float64(params0.astype(np.float64).sum()), params0_head=params0[:4096],
        params0_tail=params0[-4096:], cfg8=cfg8, y_hg=y_hg, F_hg=F_hg, cfg8_m=cfg8_m, y_m=y_m, F_m=F_m,
        y_lit=y_lit, F_lit=F_lit)

    # ---------------- config 1 (64^3 cloud seed 0, HG 0.7, albedo 0.99)
    n = 64
    vs = 2.0 / n
    g = R.generate_medium(2, n, 0)
    tvol = R.build_tvol(g, vs, ORIGIN, LIGHT)
    table = R.phase_table(64, 128, 32, 16)
    centers = R.draw_centers(g, vs, ORIGIN, 192, 5, LIGHT)
    ctx = R.make_ctx(g, tvol, vs, ORIGIN, dpath, hpath, m_hg, table)
    f1 = R.features(ctx, centers, nd, nh)
    cfg8 = cfg_rows(R, centers, [0.7], [0.99, 0.99, 0.99])
    y1, F1 = R.predict(b, f1, cfg8)
    np.savez_compressed(os.path.join(GOLD, "c1.npz"), tvol=tvol, centers=centers, feats=f1, cfg8=cfg8, y=y1,
                        F=F1)
    np.savez_compressed(os.path.join(GOLD, "phase_table_full.npz"), table=table)
    render_fixture(R)
    io_fixtures(R)
    for f in sorted(os.listdir(GOLD)):
        print(f, os.path.getsize(os.path.join(GOLD, f)))


if __name__ == "__main__":
    main()
