// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product).
//
// A thin C-ABI driver over the UNMODIFIED reference core library
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libsf_ref.so). It exists so that tests/, tests/golden/make_golden.py
// and bench.py's reference / cpu_baseline arm can call the reference's own
// hot-path functions with plain arrays:
//
//   generate_medium          proj/core/src/scene_gen.cpp:74-109
//   DensityPyramid           proj/core/src/volume_grid.cpp:91-126
//   graded_transmittance     proj/core/src/feature_pipeline.cpp:37-68
//   conv3_replicate          proj/core/src/feature_pipeline.cpp:70-92
//   build_transmittance_volume proj/core/src/feature_pipeline.cpp:200-211
//   PhaseTable / lookup_hg   proj/core/src/phase.cpp:159-219
//   generate_*_template      proj/core/src/templates.cpp:118-205 (+ save_template :258-284)
//   sample_features          proj/core/src/feature_pipeline.cpp:139-172
//   make_backbone / predict_y / decode_prediction  proj/core/src/predictor.cpp:308-409
//   draw_centers             proj/core/src/feature_pipeline.cpp:174-198
//
// Feature block layout used across the repo (one query):
//   diffuse  {density[nd], transmittance[nd], phase[nd]}
//   highlight{density[nh], transmittance[nh], phase[nh]}
// Config layout (one query, 8 doubles): n_g, g0, g1, g2, albedo.x, .y, .z, alpha.

#include <array>
#include <chrono>
#include <memory>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "scatterfield/error.h"
#include "scatterfield/feature_pipeline.h"
#include "scatterfield/parallel.h"
#include "scatterfield/phase.h"
#include "scatterfield/predictor.h"
#include "scatterfield/camera.h"
#include "scatterfield/rte.h"
#include "scatterfield/scene_gen.h"
#include "scatterfield/templates.h"
#include "scatterfield/volume_grid.h"

namespace sf = scatterfield;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const sf::Error& e) {
        g_err = e.what();
        return int(e.code()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

sf::DensityGrid make_grid(const float* vals, int nx, int ny, int nz, double vs,
                          const double* origin) {
    sf::DensityGrid g(nx, ny, nz, vs, sf::Vec3{origin[0], origin[1], origin[2]});
    std::memcpy(g.values().data(), vals, sizeof(float) * size_t(nx) * ny * nz);
    return g;
}

sf::Vec3 v3(const double* p) { return sf::Vec3{p[0], p[1], p[2]}; }

sf::CombinerWeights make_combiner(const float* kernels, const float* scales, int L) {
    if (!kernels) return sf::CombinerWeights::identity(L);
    sf::CombinerWeights w;
    w.kernels.resize(size_t(L));
    w.scales.resize(size_t(L));
    for (int l = 0; l < L; ++l) {
        for (int t = 0; t < 27; ++t) w.kernels[size_t(l)][size_t(t)] = kernels[l * 27 + t];
        w.scales[size_t(l)] = scales[l];
    }
    return w;
}

sf::PhaseModel make_model(int kind, int n_lobes, const double* weights, const double* gs) {
    if (kind == 0) return sf::PhaseModel::isotropic();
    if (kind == 1) return sf::PhaseModel::hg(gs[0]);
    std::vector<sf::PhaseLobe> lobes(static_cast<size_t>(n_lobes));
    for (int k = 0; k < n_lobes; ++k) lobes[size_t(k)] = {weights[k], gs[k]};
    return sf::PhaseModel::multi_hg(lobes);
}

sf::ConfigParams make_cfg(const double* c) {
    sf::ConfigParams cp;
    int ng = int(c[0]);
    for (int i = 0; i < ng; ++i) cp.g_params.push_back(c[1 + i]);
    cp.albedo = sf::Vec3{c[4], c[5], c[6]};
    cp.alpha = c[7];
    return cp;
}

sf::SampleFeatureBlock block_from(const float* f, int n) {
    sf::SampleFeatureBlock b;
    b.density.assign(f, f + n);
    b.transmittance.assign(f + n, f + 2 * n);
    b.phase.assign(f + 2 * n, f + 3 * n);
    return b;
}

void block_to(const sf::SampleFeatureBlock& b, float* f) {
    size_t n = b.density.size();
    std::memcpy(f, b.density.data(), n * 4);
    std::memcpy(f + n, b.transmittance.data(), n * 4);
    std::memcpy(f + 2 * n, b.phase.data(), n * 4);
}

struct Ctx {
    sf::DensityGrid density;
    sf::TransmittanceFeatureVolume tvol;
    sf::SamplingTemplate dt, ht;
    sf::PhaseModel model;
    sf::PhaseTable table;
    double template_scale = 1.0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { sf::set_thread_cap(n); }
int ref_get_threads() { return sf::thread_cap(); }

int ref_generate_medium(int kind, int dims, uint64_t seed, float* out) {
    return guard([&] {
        sf::DensityGrid g = sf::generate_medium(sf::MediumKind(kind), dims, seed);
        std::memcpy(out, g.values().data(), g.values().size() * 4);
    });
}

// Writes every pyramid level back to back; *n_levels receives the count.
int ref_pyramid(const float* vals, int nx, int ny, int nz, double vs, const double* origin,
                float* out, int* n_levels) {
    return guard([&] {
        sf::DensityPyramid pyr(make_grid(vals, nx, ny, nz, vs, origin));
        size_t off = 0;
        for (int i = 0; i < pyr.level_count(); ++i) {
            const auto& v = pyr.level(i).values();
            std::memcpy(out + off, v.data(), v.size() * 4);
            off += v.size();
        }
        *n_levels = pyr.level_count();
    });
}

int ref_graded(const float* vals, int nx, int ny, int nz, double vs, const double* origin,
               int level, const double* light, double lambda, double step, float* out) {
    return guard([&] {
        sf::DensityPyramid pyr(make_grid(vals, nx, ny, nz, vs, origin));
        sf::GradedTransmittanceField f =
            sf::graded_transmittance(pyr, level, v3(light), lambda, step);
        std::memcpy(out, f.values.values().data(), f.values.values().size() * 4);
    });
}

int ref_conv3(const float* in, int nx, int ny, int nz, const float* k27, float* out) {
    return guard([&] {
        double o[3] = {0, 0, 0};
        std::array<float, 27> k;
        for (int t = 0; t < 27; ++t) k[size_t(t)] = k27[t];
        sf::DensityGrid r = sf::conv3_replicate(make_grid(in, nx, ny, nz, 1.0, o), k);
        std::memcpy(out, r.values().data(), r.values().size() * 4);
    });
}

// kernels == NULL selects the identity combiner (proj/core/src/feature_pipeline.cpp:29-35).
int ref_build_tvol(const float* vals, int nx, int ny, int nz, double vs, const double* origin,
                   const double* light, double lambda, double step_scale,
                   const float* kernels, const float* scales, float* out) {
    return guard([&] {
        sf::DensityPyramid pyr(make_grid(vals, nx, ny, nz, vs, origin));
        sf::FeatureConfig cfg;
        cfg.lambda = lambda;
        cfg.step_scale = step_scale;
        sf::TransmittanceFeatureVolume t = sf::build_transmittance_volume(
            pyr, v3(light), make_combiner(kernels, scales, pyr.level_count()), cfg);
        std::memcpy(out, t.values.values().data(), t.values.values().size() * 4);
    });
}

int ref_phase_table(int g_res, int a_res, int h_res, int nodes, float* out) {
    return guard([&] {
        sf::PhaseTable t(g_res, a_res, h_res, nodes);
        std::memcpy(out, t.values().data(), t.values().size() * 4);
    });
}

int ref_lookup_hg(const float* table, int g_res, int a_res, int h_res, int64_t n,
                  const double* g, const double* angle, const double* half, double* out) {
    return guard([&] {
        std::vector<float> v(table, table + size_t(g_res) * a_res * h_res);
        sf::PhaseTable t = sf::PhaseTable::from_values(g_res, a_res, h_res, std::move(v));
        for (int64_t i = 0; i < n; ++i) out[i] = t.lookup_hg(g[i], angle[i], half[i]);
    });
}

// kind 0 = diffuse (default counts), 1 = highlight (default counts).
int ref_gen_template(int kind, uint64_t seed, double gen_distance, double cone_half_angle,
                     const char* path) {
    return guard([&] {
        sf::SamplingTemplate t =
            kind == 0 ? sf::generate_diffuse_template(sf::diffuse_default_counts(), seed)
                      : sf::generate_highlight_template(sf::highlight_default_counts(),
                                                        gen_distance, cone_half_angle, seed);
        sf::save_template(t, path);
    });
}

int ref_draw_centers(const float* vals, int nx, int ny, int nz, double vs, const double* origin,
                     int count, uint64_t seed, const double* light, double* out9) {
    return guard([&] {
        std::vector<sf::CenterSpec> c =
            sf::draw_centers(make_grid(vals, nx, ny, nz, vs, origin), count, seed, v3(light));
        for (size_t i = 0; i < c.size(); ++i) {
            double* o = out9 + 9 * i;
            o[0] = c[i].p.x; o[1] = c[i].p.y; o[2] = c[i].p.z;
            o[3] = c[i].omega.x; o[4] = c[i].omega.y; o[5] = c[i].omega.z;
            o[6] = c[i].light.x; o[7] = c[i].light.y; o[8] = c[i].light.z;
        }
    });
}

void* ref_ctx_new(const float* vals, int nx, int ny, int nz, double vs, const double* origin,
                  const float* tvol_vals, const char* diffuse_path, const char* highlight_path,
                  int phase_kind, int n_lobes, const double* lobe_w, const double* lobe_g,
                  const float* table_vals, int g_res, int a_res, int h_res,
                  double template_scale) {
    Ctx* c = nullptr;
    int rc = guard([&] {
        auto ctx = std::make_unique<Ctx>();
        ctx->density = make_grid(vals, nx, ny, nz, vs, origin);
        ctx->tvol.values = make_grid(tvol_vals, nx, ny, nz, vs, origin);
        ctx->dt = sf::load_template(diffuse_path);
        ctx->ht = sf::load_template(highlight_path);
        ctx->model = make_model(phase_kind, n_lobes, lobe_w, lobe_g);
        std::vector<float> tv(table_vals, table_vals + size_t(g_res) * a_res * h_res);
        ctx->table = sf::PhaseTable::from_values(g_res, a_res, h_res, std::move(tv));
        ctx->template_scale = template_scale;
        c = ctx.release();
    });
    return rc == 0 ? c : nullptr;
}

void ref_ctx_free(void* c) { delete static_cast<Ctx*>(c); }

int ref_ctx_counts(void* cp, int* nd, int* nh) {
    Ctx* c = static_cast<Ctx*>(cp);
    *nd = c->dt.total_points();
    *nh = c->ht.total_points();
    return 0;
}

int ref_ctx_features(void* cp, int64_t q, const double* centers9, float* out) {
    Ctx* c = static_cast<Ctx*>(cp);
    return guard([&] {
        int nd = c->dt.total_points(), nh = c->ht.total_points();
        size_t stride = size_t(3) * (nd + nh);
        sf::parallel_for(q, [&](int64_t i) {
            const double* s = centers9 + 9 * i;
            sf::SampleFeatureBlock d = sf::sample_features(
                v3(s), v3(s + 3), v3(s + 6), c->dt, c->density, c->tvol, c->model, c->table,
                c->template_scale);
            sf::SampleFeatureBlock h = sf::sample_features(
                v3(s), v3(s + 3), v3(s + 6), c->ht, c->density, c->tvol, c->model, c->table,
                c->template_scale);
            block_to(d, out + stride * size_t(i));
            block_to(h, out + stride * size_t(i) + size_t(3) * nd);
        });
    });
}

void* ref_backbone_new(uint64_t seed, int literal, const int* dcounts, int n_d,
                       const int* hcounts, int n_h, int width, int merge_width,
                       int head_width, double gamma) {
    sf::Backbone<float>* out = nullptr;
    int rc = guard([&] {
        sf::BackboneConfig cfg;
        cfg.diffuse_counts.assign(dcounts, dcounts + n_d);
        cfg.highlight_counts.assign(hcounts, hcounts + n_h);
        cfg.width = width;
        cfg.merge_width = merge_width;
        cfg.head_width = head_width;
        cfg.gamma = gamma;
        cfg.seed = seed;
        cfg.literal_attention = literal != 0;
        out = new sf::Backbone<float>(sf::make_backbone<float>(cfg));
    });
    return rc == 0 ? out : nullptr;
}

void ref_backbone_free(void* b) { delete static_cast<sf::Backbone<float>*>(b); }

int64_t ref_backbone_param_count(void* bp) {
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    int64_t n = 0;
    for (const auto& p : b->params.params) n += int64_t(p.value.size());
    return n;
}

int ref_backbone_get_params(void* bp, float* out) {
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    size_t off = 0;
    for (const auto& p : b->params.params) {
        std::memcpy(out + off, p.value.v.data(), p.value.size() * 4);
        off += p.value.size();
    }
    return 0;
}

int ref_backbone_set_params(void* bp, const float* in) {
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    size_t off = 0;
    for (auto& p : b->params.params) {
        std::memcpy(p.value.v.data(), in + off, p.value.size() * 4);
        off += p.value.size();
    }
    return 0;
}

int ref_backbone_save(void* bp, const char* path) {
    return guard([&] { sf::save_backbone(*static_cast<sf::Backbone<float>*>(bp), path); });
}

// y and F are [q][3] doubles; features use the block layout above.
int ref_predict(void* bp, int64_t q, const float* feats, const double* cfg8, double* y_out,
                double* F_out) {
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    return guard([&] {
        int nd = 0, nh = 0;
        for (int c : b->config.diffuse_counts) nd += c;
        for (int c : b->config.highlight_counts) nh += c;
        size_t stride = size_t(3) * (nd + nh);
        sf::parallel_for(q, [&](int64_t i) {
            const float* f = feats + stride * size_t(i);
            sf::SampleFeatureBlock d = block_from(f, nd);
            sf::SampleFeatureBlock h = block_from(f + 3 * nd, nh);
            sf::ConfigParams cp = make_cfg(cfg8 + 8 * i);
            sf::Vec3 y = sf::predict_y(*b, d, h, cp);
            sf::Vec3 F = sf::decode_prediction(y, cp.albedo, b->config.gamma);
            double* yo = y_out + 3 * i;
            double* fo = F_out + 3 * i;
            yo[0] = y.x; yo[1] = y.y; yo[2] = y.z;
            fo[0] = F.x; fo[1] = F.y; fo[2] = F.z;
        });
    });
}

// The reference's per-query hot loop (features for both templates, predict_y,
// decode_prediction) over q queries with the current thread cap; returns the
// wall seconds via *seconds. This is what bench.py times as the CPU baseline.
int ref_time_queries(void* cp, void* bp, int64_t q, const double* centers9,
                     const double* cfg8, double* F_out, double* seconds) {
    Ctx* c = static_cast<Ctx*>(cp);
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    return guard([&] {
        auto t0 = std::chrono::steady_clock::now();
        sf::parallel_for(q, [&](int64_t i) {
            const double* s = centers9 + 9 * i;
            sf::SampleFeatureBlock d = sf::sample_features(
                v3(s), v3(s + 3), v3(s + 6), c->dt, c->density, c->tvol, c->model, c->table,
                c->template_scale);
            sf::SampleFeatureBlock h = sf::sample_features(
                v3(s), v3(s + 3), v3(s + 6), c->ht, c->density, c->tvol, c->model, c->table,
                c->template_scale);
            sf::ConfigParams cfg = make_cfg(cfg8 + 8 * i);
            sf::Vec3 y = sf::predict_y(*b, d, h, cfg);
            sf::Vec3 F = sf::decode_prediction(y, cfg.albedo, b->config.gamma);
            double* fo = F_out + 3 * i;
            fo[0] = F.x; fo[1] = F.y; fo[2] = F.z;
        });
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// render_neural (src/predictor.cpp:585-614) on the context's density, phase model and
// phase table with the FeatureTable's combiner (kernels [L][27] + scales [L], or NULL for the
// identity combiner precompute_tables makes): build the tvol, bake F at every occupied voxel
// centre, march render_volume (src/rte.cpp:407-447). out_img [h][w][3].
int ref_render_neural(void* cp, void* bp, const double* sigma_t3, const double* albedo3, int material_class,
                      const double* light3, const double* cam_pos, const double* look_at, const double* up,
                      double vfov, int w, int h, double lambda, double step_scale, const double* background,
                      const float* kernels, const float* scales, float* out_img) {
    Ctx* c = static_cast<Ctx*>(cp);
    auto* b = static_cast<sf::Backbone<float>*>(bp);
    return guard([&] {
        sf::Medium medium;
        medium.grid = c->density;
        medium.props.sigma_t_scale = v3(sigma_t3);
        medium.props.albedo = v3(albedo3);
        medium.props.material_class = static_cast<sf::MaterialClass>(material_class);
        medium.phase = c->model;
        sf::DistantLight light;
        light.direction = v3(light3);
        light.intensity = sf::Vec3{1.0, 1.0, 1.0};
        sf::Camera cam(v3(cam_pos), v3(look_at), v3(up), vfov, w, h);
        sf::FeatureTable table;
        table.phase_table = c->table;
        sf::DensityPyramid pyr(c->density);
        table.combiner = sf::CombinerWeights::identity(int(pyr.level_count()));
        if (kernels && scales)
            for (int l = 0; l < int(pyr.level_count()); ++l) {
                for (int k = 0; k < 27; ++k) table.combiner.kernels[size_t(l)][size_t(k)] = kernels[27 * l + k];
                table.combiner.scales[size_t(l)] = scales[l];
            }
        table.lambda = lambda;
        table.template_scale = c->template_scale;
        sf::FeatureConfig fcfg;
        fcfg.step_scale = step_scale;
        sf::RenderOptions ro;
        ro.step_scale = step_scale;
        ro.background = v3(background);
        sf::ImageF img = sf::render_neural(medium, light, cam, *b, table, c->dt, c->ht, fcfg, ro);
        std::memcpy(out_img, img.rgb.data(), img.rgb.size() * sizeof(float));
    });
}

// save_density (src/volume_grid.cpp:224-238) of the given grid.
int ref_save_density(const float* vals, int nx, int ny, int nz, double vs, const double* origin, const char* path) {
    return guard([&] { sf::save_density(make_grid(vals, nx, ny, nz, vs, origin), path); });
}

// load_density (src/volume_grid.cpp:175-222): dims/vs/origin into info[7], values into out (may be null).
int ref_load_density(const char* path, double* info, float* out) {
    return guard([&] {
        sf::DensityGrid g = sf::load_density(path);
        info[0] = g.nx(); info[1] = g.ny(); info[2] = g.nz(); info[3] = g.voxel_size();
        info[4] = g.origin().x; info[5] = g.origin().y; info[6] = g.origin().z;
        if (out) std::memcpy(out, g.values().data(), g.values().size() * sizeof(float));
    });
}

// precompute_tables' per-center blocks (sample_features x2 on the context) for the given
// centers, then save_feature_table (src/feature_pipeline.cpp:268-294) with the context's
// phase table, the identity combiner of `levels` levels, lambda and template_scale.
int ref_save_feature_table(void* cp, int64_t q, const double* centers9, int levels, double lambda,
                           const char* path) {
    Ctx* c = static_cast<Ctx*>(cp);
    return guard([&] {
        sf::FeatureTable t;
        for (int64_t i = 0; i < q; ++i) {
            const double* s = centers9 + 9 * i;
            t.diffuse.push_back(sf::sample_features(v3(s), v3(s + 3), v3(s + 6), c->dt, c->density, c->tvol,
                                                    c->model, c->table, c->template_scale));
            t.highlight.push_back(sf::sample_features(v3(s), v3(s + 3), v3(s + 6), c->ht, c->density, c->tvol,
                                                      c->model, c->table, c->template_scale));
        }
        t.phase_table = c->table;
        t.combiner = sf::CombinerWeights::identity(levels);
        t.lambda = lambda;
        t.template_scale = c->template_scale;
        sf::save_feature_table(t, path);
    });
}

}  // extern "C"
