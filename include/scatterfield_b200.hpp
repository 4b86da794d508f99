// include/scatterfield_b200.hpp — C++ shim over the C ABI with the reference's
// C++ signatures (proj/core/include/scatterfield/*.h), so a reference caller can
// switch `#include "scatterfield/feature_pipeline.h"` & co. to this header and
// `scatterfield::` to `scatterfield_b200::`. Failures throw scatterfield_b200::Error
// carrying the reference Errc (inc/error.h:11-32). Header-only; link libsf_b200.so.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "scatterfield_b200.h"

namespace scatterfield_b200 {

enum class Errc {
    io,
    malformed_header,
    bad_dims,
    bad_value,
    truncated,
    invalid_argument,
    shape_mismatch,
    provenance_mismatch,
    numeric,
    cuda
};

class Error : public std::runtime_error {
  public:
    Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
    Errc code() const { return code_; }

  private:
    Errc code_;
};

inline void check(int rc) {
    if (rc == SF_OK) return;
    Errc e = rc == SF_ERR_CUDA ? Errc::cuda : Errc(rc - 1);
    throw Error(e, sf_last_error());
}

struct Vec3 {
    double x = 0, y = 0, z = 0;
};

// ---- DensityGrid (inc/volume_grid.h:17-58) ---------------------------------------
class DensityGrid {
  public:
    DensityGrid(int nx, int ny, int nz, double voxel_size, const Vec3& origin,
                const float* values = nullptr) {
        double o[3] = {origin.x, origin.y, origin.z};
        sf_grid* g = nullptr;
        check(sf_grid_create(nx, ny, nz, voxel_size, o, values, &g));
        h_.reset(g, sf_grid_destroy);
    }
    explicit DensityGrid(const sf_grid* borrowed, std::shared_ptr<void> owner)
        : borrowed_(borrowed), owner_(std::move(owner)) {}
    static DensityGrid adopt(sf_grid* g) {
        DensityGrid d;
        d.h_.reset(g, sf_grid_destroy);
        return d;
    }
    const sf_grid* handle() const { return h_ ? h_.get() : borrowed_; }
    int nx() const { return info()[0]; }
    int ny() const { return info()[1]; }
    int nz() const { return info()[2]; }
    std::vector<float> values() const {
        auto d = info();
        std::vector<float> v(size_t(d[0]) * d[1] * d[2]);
        check(sf_grid_download(handle(), v.data(), nullptr));
        return v;
    }
    double sample_trilinear(const Vec3& p) const {
        double pts[3] = {p.x, p.y, p.z}, out = 0.0;
        check(sf_grid_sample_trilinear(handle(), 1, pts, &out, nullptr));
        return out;
    }

  private:
    DensityGrid() = default;
    std::array<int, 3> info() const {
        std::array<int, 3> d{};
        check(sf_grid_info(handle(), d.data(), nullptr, nullptr));
        return d;
    }
    std::shared_ptr<sf_grid> h_;
    const sf_grid* borrowed_ = nullptr;
    std::shared_ptr<void> owner_;
};

// ---- DensityPyramid (inc/volume_grid.h:62-72) -------------------------------------
class DensityPyramid {
  public:
    explicit DensityPyramid(const DensityGrid& finest) {
        sf_pyramid* p = nullptr;
        check(sf_pyramid_build(finest.handle(), &p, nullptr));
        h_.reset(p, sf_pyramid_destroy);
    }
    int level_count() const { return sf_pyramid_level_count(h_.get()); }
    DensityGrid level(int i) const {
        const sf_grid* g = sf_pyramid_level(h_.get(), i);
        if (!g) throw Error(Errc::invalid_argument, "pyramid: level out of range");
        return DensityGrid(g, h_);
    }
    const sf_pyramid* handle() const { return h_.get(); }

  private:
    std::shared_ptr<sf_pyramid> h_;
};

inline DensityPyramid build_pyramid(const DensityGrid& g) { return DensityPyramid(g); }

// ---- feature pipeline (inc/feature_pipeline.h) -------------------------------------
struct CombinerWeights {
    std::vector<std::array<float, 27>> kernels;
    std::vector<float> scales;
    static CombinerWeights identity(int level_count) {
        CombinerWeights w;
        w.kernels.assign(size_t(level_count), {});
        w.scales.assign(size_t(level_count), float(1.0 / level_count));
        for (auto& k : w.kernels) k[13] = 1.0f;
        return w;
    }
    int level_count() const { return int(kernels.size()); }
};

struct FeatureConfig {
    double lambda = 0.6;
    double step_scale = 0.5;
    double template_scale = 1.0;
    int phase_g_res = 64;
    int phase_angle_res = 128;
    int phase_aperture_res = 32;
    int phase_quad_nodes = 16;
};

class TransmittanceFeatureVolume {
  public:
    explicit TransmittanceFeatureVolume(sf_tvol* t) : h_(t, sf_tvol_destroy) {}
    DensityGrid values() const { return DensityGrid(sf_tvol_values(h_.get()), h_); }
    const sf_tvol* handle() const { return h_.get(); }

  private:
    std::shared_ptr<sf_tvol> h_;
};

inline DensityGrid graded_transmittance(const DensityPyramid& p, int level, const Vec3& light,
                                        double lambda, double step) {
    double l[3] = {light.x, light.y, light.z};
    sf_grid* g = nullptr;
    check(sf_graded_transmittance(p.handle(), level, l, lambda, step, &g, nullptr));
    return DensityGrid::adopt(g);
}

inline DensityGrid conv3_replicate(const DensityGrid& in, const std::array<float, 27>& kernel) {
    sf_grid* g = nullptr;
    check(sf_conv3_replicate(in.handle(), kernel.data(), &g, nullptr));
    return DensityGrid::adopt(g);
}

inline TransmittanceFeatureVolume build_transmittance_volume(const DensityPyramid& p,
                                                             const Vec3& light,
                                                             const CombinerWeights& w,
                                                             const FeatureConfig& cfg) {
    std::vector<float> k, s(w.scales);
    for (const auto& kk : w.kernels) k.insert(k.end(), kk.begin(), kk.end());
    double l[3] = {light.x, light.y, light.z};
    sf_tvol* t = nullptr;
    check(sf_build_transmittance_volume(p.handle(), l, k.data(), s.data(), cfg.lambda,
                                        cfg.step_scale, &t, nullptr));
    return TransmittanceFeatureVolume(t);
}

// ---- phase (inc/phase.h) -------------------------------------------------------------
struct PhaseLobe {
    double weight = 1.0;
    double g = 0.0;
};

struct PhaseModel {
    int kind = SF_PHASE_ISOTROPIC;
    std::vector<PhaseLobe> lobes{{1.0, 0.0}};
    static PhaseModel isotropic() { return PhaseModel{}; }
    static PhaseModel hg(double g) { return PhaseModel{SF_PHASE_HG, {{1.0, g}}}; }
    static PhaseModel multi_hg(const std::vector<PhaseLobe>& l) { return PhaseModel{SF_PHASE_MULTI_HG, l}; }
    sf_phase_model to_c() const {
        sf_phase_model m{};
        m.kind = kind;
        m.n_lobes = int(lobes.size());
        for (size_t i = 0; i < lobes.size() && i < 3; ++i) {
            m.weight[i] = lobes[i].weight;
            m.g[i] = lobes[i].g;
        }
        return m;
    }
};

class PhaseTable {
  public:
    PhaseTable(int g_res, int angle_res, int aperture_res, int quad_nodes = 16) {
        sf_phase_table* t = nullptr;
        check(sf_phase_table_build(g_res, angle_res, aperture_res, quad_nodes, &t, nullptr));
        h_.reset(t, sf_phase_table_destroy);
    }
    double lookup_hg(double g, double angle, double half_angle) const {
        double out = 0.0;
        check(sf_phase_table_lookup_hg(h_.get(), 1, &g, &angle, &half_angle, &out, nullptr));
        return out;
    }
    const sf_phase_table* handle() const { return h_.get(); }

  private:
    std::shared_ptr<sf_phase_table> h_;
};

// ---- templates (inc/templates.h) -------------------------------------------------------
struct TemplateLayer {
    int index = 0;
    double radius = 0.0;
    double cap_radius = 0.0;
    std::vector<Vec3> points;
};

struct SamplingTemplate {
    int kind = SF_TEMPLATE_DIFFUSE;
    uint64_t seed = 0;
    std::vector<TemplateLayer> layers;
    double gen_distance = 0.0;
    double cone_half_angle = 0.0;
    int total_points() const {
        int n = 0;
        for (const auto& l : layers) n += int(l.points.size());
        return n;
    }
    std::shared_ptr<sf_template> device() const {
        std::vector<int> counts;
        std::vector<double> pts, caps;
        for (const auto& l : layers) {
            counts.push_back(int(l.points.size()));
            caps.push_back(l.cap_radius);
            for (const auto& p : l.points) pts.insert(pts.end(), {p.x, p.y, p.z});
        }
        sf_template* t = nullptr;
        check(sf_template_create(kind, int(counts.size()), counts.data(), pts.data(), caps.data(),
                                 gen_distance, cone_half_angle, &t));
        return std::shared_ptr<sf_template>(t, sf_template_destroy);
    }
};

// SampleFeatureBlock (inc/feature_pipeline.h:50-55)
struct SampleFeatureBlock {
    Vec3 p, omega, light;
    std::vector<float> density, transmittance, phase;
};

inline SampleFeatureBlock sample_features(const Vec3& p, const Vec3& omega, const Vec3& light,
                                          const SamplingTemplate& tmpl, const DensityGrid& density,
                                          const TransmittanceFeatureVolume& tvol,
                                          const PhaseModel& model, const PhaseTable& table,
                                          double template_scale) {
    auto t = tmpl.device();
    sf_phase_model m = model.to_c();
    double q[9] = {p.x, p.y, p.z, omega.x, omega.y, omega.z, light.x, light.y, light.z};
    int n = tmpl.total_points();
    std::vector<float> out(size_t(3) * n);
    check(sf_sample_features(density.handle(), tvol.handle(), t.get(), &m, table.handle(),
                             template_scale, 1, q, out.data(), nullptr));
    SampleFeatureBlock b{p, omega, light, {}, {}, {}};
    b.density.assign(out.begin(), out.begin() + n);
    b.transmittance.assign(out.begin() + n, out.begin() + 2 * n);
    b.phase.assign(out.begin() + 2 * n, out.end());
    return b;
}

// ---- predictor (inc/predictor.h) ---------------------------------------------------------
struct ConfigParams {
    std::vector<double> g_params;
    Vec3 albedo{0.5, 0.5, 0.5};
    double alpha = 0.0;
};

struct BackboneConfig {
    std::vector<int> diffuse_counts{6, 8, 12, 16, 24, 32, 48, 48};
    std::vector<int> highlight_counts{32, 16, 16, 8};
    int width = 32, merge_width = 64, head_width = 64;
    double gamma = 4.0;
    uint64_t seed = 1;
    bool literal_attention = false;
    sf_backbone_config to_c() const {
        sf_backbone_config c{};
        c.n_diffuse_layers = int(diffuse_counts.size());
        c.n_highlight_layers = int(highlight_counts.size());
        for (size_t i = 0; i < diffuse_counts.size() && i < 16; ++i) c.diffuse_counts[i] = diffuse_counts[i];
        for (size_t i = 0; i < highlight_counts.size() && i < 16; ++i)
            c.highlight_counts[i] = highlight_counts[i];
        c.width = width;
        c.merge_width = merge_width;
        c.head_width = head_width;
        c.gamma = gamma;
        c.seed = seed;
        c.literal_attention = literal_attention;
        return c;
    }
};

class Backbone {
  public:
    explicit Backbone(const BackboneConfig& cfg, const float* params = nullptr) : config(cfg) {
        sf_backbone_config c = cfg.to_c();
        sf_backbone* b = nullptr;
        check(sf_backbone_create(&c, params, &b));
        h_.reset(b, sf_backbone_destroy);
    }
    BackboneConfig config;
    const sf_backbone* handle() const { return h_.get(); }

  private:
    std::shared_ptr<sf_backbone> h_;
};

inline Backbone make_backbone(const BackboneConfig& cfg) { return Backbone(cfg); }

inline Vec3 predict_y(const Backbone& net, const SampleFeatureBlock& d, const SampleFeatureBlock& h,
                      const ConfigParams& cfg, int precision = SF_PRECISION_FP32) {
    std::vector<float> row;
    for (const auto* v : {&d.density, &d.transmittance, &d.phase, &h.density, &h.transmittance, &h.phase})
        row.insert(row.end(), v->begin(), v->end());
    double c8[8] = {double(cfg.g_params.size()), 0, 0, 0, cfg.albedo.x, cfg.albedo.y, cfg.albedo.z, cfg.alpha};
    for (size_t i = 0; i < cfg.g_params.size() && i < 3; ++i) c8[1 + i] = cfg.g_params[i];
    float y[3];
    check(sf_predict(net.handle(), 1, row.data(), c8, precision, y, nullptr, nullptr));
    return {y[0], y[1], y[2]};
}

inline Vec3 decode_prediction(const Vec3& y, const Vec3& albedo, double gamma) {
    for (double a : {albedo.x, albedo.y, albedo.z})
        if (!(a > 0.0 && a < 1.0)) throw Error(Errc::bad_value, "albedo components must lie in (0,1)");
    return {std::pow(albedo.x, gamma) * std::expm1(y.x), std::pow(albedo.y, gamma) * std::expm1(y.y),
            std::pow(albedo.z, gamma) * std::expm1(y.z)};
}

// ---- the fused per-shading-point query (render_neural's bake loop) ------------------------
// Bound inputs of the query; the handles must outlive it (the reference's render_neural holds
// the same objects while baking, src/predictor.cpp:585-614).
class Scene {
  public:
    Scene(const DensityGrid& density, const TransmittanceFeatureVolume& tvol, const SamplingTemplate& diffuse,
          const SamplingTemplate& highlight, const PhaseModel& model, const PhaseTable& table,
          double template_scale = 1.0)
        : dt_(diffuse.device()), ht_(highlight.device()), density_(density), tvol_(tvol), table_(table) {
        sf_phase_model m = model.to_c();
        sf_scene* s = nullptr;
        check(sf_scene_create(density.handle(), tvol.handle(), dt_.get(), ht_.get(), &m, table.handle(),
                              template_scale, &s));
        h_.reset(s, sf_scene_destroy);
    }
    const sf_scene* handle() const { return h_.get(); }

  private:
    std::shared_ptr<sf_template> dt_, ht_;
    DensityGrid density_;
    TransmittanceFeatureVolume tvol_;
    PhaseTable table_;
    std::shared_ptr<sf_scene> h_;
};

// Per query (p, omega, l): sample_features x2 -> make_config -> predict_y -> decode_prediction.
// rows: 9 doubles per query; returns F (3 doubles per query).
inline std::vector<double> query(const Scene& scene, const Backbone& net, const ConfigParams& medium,
                                 const std::vector<double>& rows, int precision = SF_PRECISION_FP32) {
    sf_medium_params m{};
    m.n_g = int(medium.g_params.size());
    for (size_t i = 0; i < medium.g_params.size() && i < 3; ++i) m.g[i] = medium.g_params[i];
    m.albedo[0] = medium.albedo.x;
    m.albedo[1] = medium.albedo.y;
    m.albedo[2] = medium.albedo.z;
    std::vector<double> F(rows.size() / 9 * 3);
    check(sf_query(scene.handle(), net.handle(), &m, int64_t(rows.size() / 9), rows.data(), precision, F.data(),
                   nullptr, nullptr));
    return F;
}

// Rows [z0, z1) of build_transmittance_volume's values (the per-light build sharded by z-slab).
inline std::vector<float> build_transmittance_slab(const DensityPyramid& p, const Vec3& light,
                                                   const CombinerWeights& w, const FeatureConfig& cfg, int z0,
                                                   int z1, int nx, int ny) {
    std::vector<float> k, s(w.scales), out(size_t(nx) * ny * size_t(z1 > z0 ? z1 - z0 : 0));
    for (const auto& kk : w.kernels) k.insert(k.end(), kk.begin(), kk.end());
    double l[3] = {light.x, light.y, light.z};
    check(sf_build_transmittance_slab(p.handle(), l, k.data(), s.data(), cfg.lambda, cfg.step_scale, 0, z0, z1,
                                      out.data(), nullptr));
    return out;
}

// ---- image entry point (inc/camera.h, inc/rte.h, inc/image.h) ----------------------------
struct Camera {
    Vec3 position, look_at{0, 0, 0}, up{0, 1, 0};
    double vfov_degrees = 40.0;
    int width = 64, height = 64;
};

struct RenderOptions {
    double step_scale = 0.5;
    Vec3 background{0.0, 0.0, 0.0};
};

struct ImageF {
    int width = 0, height = 0;
    std::vector<float> rgb;  // width * height * 3, row-major
};

enum class MaterialClass { Air, Gas, SolidLiquid, Skin };

// render_neural (src/predictor.cpp:585-614): tvol for `light`, bake F on the density lattice
// (sf_bake_field), march the image (sf_render_volume).
inline ImageF render_neural(const DensityGrid& grid, const DensityPyramid& pyr, const Vec3& light,
                            const Camera& cam, const Backbone& net, const PhaseTable& table,
                            const SamplingTemplate& dt, const SamplingTemplate& ht, const PhaseModel& model,
                            const Vec3& sigma_t, const ConfigParams& medium, MaterialClass mc,
                            const FeatureConfig& fcfg = {}, const RenderOptions& ro = {},
                            int precision = SF_PRECISION_FP32) {
    TransmittanceFeatureVolume tvol =
        build_transmittance_volume(pyr, light, CombinerWeights::identity(pyr.level_count()), fcfg);
    Scene scene(grid, tvol, dt, ht, model, table, fcfg.template_scale);
    sf_medium_params m{};
    m.n_g = int(medium.g_params.size());
    for (size_t i = 0; i < medium.g_params.size() && i < 3; ++i) m.g[i] = medium.g_params[i];
    m.albedo[0] = medium.albedo.x;
    m.albedo[1] = medium.albedo.y;
    m.albedo[2] = medium.albedo.z;
    int dims[3];
    double vs, o[3];
    check(sf_grid_info(grid.handle(), dims, &vs, o));
    std::vector<float> field(size_t(3) * dims[0] * dims[1] * dims[2]);
    double cp[3] = {cam.position.x, cam.position.y, cam.position.z};
    check(sf_bake_field(scene.handle(), net.handle(), &m, cp, precision, field.data(), nullptr));
    ImageF img{cam.width, cam.height, std::vector<float>(size_t(cam.width) * cam.height * 3)};
    double st[3] = {sigma_t.x, sigma_t.y, sigma_t.z}, al[3] = {medium.albedo.x, medium.albedo.y, medium.albedo.z};
    double la[3] = {cam.look_at.x, cam.look_at.y, cam.look_at.z}, up[3] = {cam.up.x, cam.up.y, cam.up.z};
    double bg[3] = {ro.background.x, ro.background.y, ro.background.z};
    check(sf_render_volume(grid.handle(), st, al, int(mc), cp, la, up, cam.vfov_degrees, cam.width, cam.height,
                           field.data(), ro.step_scale, bg, img.rgb.data(), nullptr));
    return img;
}

}  // namespace scatterfield_b200
