// include/scatterfield_b200.hpp — C++ shim over the C ABI with the reference's
// C++ signatures (proj/core/include/scatterfield/*.h), so a reference caller can
// switch `#include "scatterfield/feature_pipeline.h"` & co. to this header and
// `scatterfield::` to `scatterfield_b200::`. Failures throw scatterfield_b200::Error
// carrying the reference Errc (inc/error.h:11-32). Header-only; link libsf_b200.so.
#pragma once

#include <array>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
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
    // PhaseModel::validate (src/phase.cpp): lobes present, weights >= 0 summing to 1, g in (-1, 1)
    void validate() const {
        if (lobes.empty()) throw Error(Errc::bad_value, "phase: model has no lobes");
        double sum = 0.0;
        for (const PhaseLobe& l : lobes) {
            if (!(l.weight >= 0.0)) throw Error(Errc::bad_value, "phase: lobe weight must be nonnegative");
            if (!(l.g > -1.0 && l.g < 1.0)) throw Error(Errc::bad_value, "phase: asymmetry must lie in (-1, 1)");
            sum += l.weight;
        }
        if (std::fabs(sum - 1.0) > 1e-9) throw Error(Errc::bad_value, "phase: lobe weights must sum to 1");
    }
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
    PhaseTable() = default;  // empty (as the reference's default-constructed table)
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

enum class MaterialClass { Air, Gas, SolidLiquid, Skin };

// ---- media and lights (inc/volume_grid.h:74-89, inc/rte.h:23-41) --------------------------
struct MediumProperties {
    Vec3 sigma_t_scale{1.0, 1.0, 1.0};  // mu_t, 1/length per channel
    Vec3 albedo{0.5, 0.5, 0.5};         // eta per channel, each in (0,1)
    MaterialClass material_class = MaterialClass::Gas;
    // MediumProperties::validate (src/volume_grid.cpp:132-154)
    void validate() const {
        for (double a : {albedo.x, albedo.y, albedo.z})
            if (!(a > 0.0 && a < 1.0)) throw Error(Errc::bad_value, "medium: albedo components must lie in (0,1)");
        const bool low = material_class == MaterialClass::Air || material_class == MaterialClass::Gas;
        const double lo = low ? 0.0 : 0.5, hi = low ? 0.5 : 1.0;
        for (double a : {albedo.x, albedo.y, albedo.z})
            if (a < lo || a > hi) throw Error(Errc::bad_value, "medium: albedo outside the material class range");
        for (double t : {sigma_t_scale.x, sigma_t_scale.y, sigma_t_scale.z})
            if (!(t > 0.0) || !std::isfinite(t)) throw Error(Errc::bad_value, "medium: sigma_t scale must be positive");
    }
};

struct Medium {
    DensityGrid grid;
    MediumProperties props;
    PhaseModel phase;
};

struct DistantLight {
    Vec3 direction;                    // unit travel direction of the light
    Vec3 intensity{1.0, 1.0, 1.0};     // per-channel radiance scale, >= 0
    // DistantLight::validate (src/rte.cpp:111-116)
    void validate() const {
        const double len = std::sqrt(direction.x * direction.x + direction.y * direction.y +
                                     direction.z * direction.z);
        if (std::fabs(len - 1.0) > 1e-9) throw Error(Errc::bad_value, "light: direction must be unit length");
        if (intensity.x < 0.0 || intensity.y < 0.0 || intensity.z < 0.0)
            throw Error(Errc::bad_value, "light: intensity must be nonnegative");
    }
};

// CenterSpec and FeatureTable (inc/feature_pipeline.h:57-70)
struct CenterSpec {
    Vec3 p, omega, light;
};

struct FeatureTable {
    std::vector<SampleFeatureBlock> diffuse;
    std::vector<SampleFeatureBlock> highlight;
    PhaseTable phase_table;
    CombinerWeights combiner;
    double lambda = 0.6;
    double template_scale = 1.0;
};

inline int expected_g_count(MaterialClass c) {  // src/predictor.cpp:29-37
    return c == MaterialClass::SolidLiquid ? 2 : (c == MaterialClass::Skin ? 3 : 1);
}

inline double angle_between(const Vec3& a, const Vec3& b) {  // inc/math.h:53-56
    const double d = a.x * b.x + a.y * b.y + a.z * b.z;
    const double c = d / std::sqrt((a.x * a.x + a.y * a.y + a.z * a.z) * (b.x * b.x + b.y * b.y + b.z * b.z));
    return std::acos(std::fmin(1.0, std::fmax(-1.0, c)));
}

// ConfigParams::validate (src/predictor.cpp:247-259)
inline void validate_config(const ConfigParams& c, MaterialClass cls) {
    if (int(c.g_params.size()) != expected_g_count(cls))
        throw Error(Errc::shape_mismatch, "asymmetry parameter count does not match material class");
    for (double g : c.g_params)
        if (!(g > -1.0 && g < 1.0)) throw Error(Errc::bad_value, "asymmetry parameter outside (-1,1)");
    for (double a : {c.albedo.x, c.albedo.y, c.albedo.z})
        if (!(a > 0.0 && a < 1.0)) throw Error(Errc::bad_value, "config albedo outside (0,1)");
    if (!(c.alpha >= 0.0 && c.alpha <= 3.14159265358979323846 + 1e-9))
        throw Error(Errc::bad_value, "alpha must be an angle in [0, pi]");
}

// make_config (inc/predictor.h:30-31, src/predictor.cpp:261-274)
inline ConfigParams make_config(const MediumProperties& props, const PhaseModel& phase, const Vec3& omega,
                                const Vec3& light_dir) {
    phase.validate();
    ConfigParams cfg;
    if (phase.kind == SF_PHASE_ISOTROPIC)
        cfg.g_params.assign(size_t(expected_g_count(props.material_class)), 0.0);
    else
        for (const PhaseLobe& l : phase.lobes) cfg.g_params.push_back(l.g);
    cfg.albedo = props.albedo;
    cfg.alpha = angle_between(omega, light_dir);
    validate_config(cfg, props.material_class);
    return cfg;
}

namespace detail {
inline sf_medium_params medium_params(const ConfigParams& c) {
    sf_medium_params m{};
    m.n_g = int(c.g_params.size());
    for (size_t i = 0; i < c.g_params.size() && i < 3; ++i) m.g[i] = c.g_params[i];
    m.albedo[0] = c.albedo.x;
    m.albedo[1] = c.albedo.y;
    m.albedo[2] = c.albedo.z;
    return m;
}
inline std::vector<float> flat_kernels(const CombinerWeights& w) {
    std::vector<float> k;
    for (const auto& kk : w.kernels) k.insert(k.end(), kk.begin(), kk.end());
    return k;
}
}  // namespace detail

// precompute_tables (inc/feature_pipeline.h:127-132, src/feature_pipeline.cpp:213-246): the
// identity combiner, the transmittance volume of centers[0]'s light, the phase table, and one
// feature block per center per template kind (batched on the GPU).
inline FeatureTable precompute_tables(const DensityGrid& density, const DensityPyramid& pyramid,
                                      const SamplingTemplate& diffuse_tmpl, const SamplingTemplate& highlight_tmpl,
                                      const std::vector<CenterSpec>& centers, const PhaseModel& model,
                                      const FeatureConfig& cfg) {
    if (centers.empty()) throw Error(Errc::invalid_argument, "precompute_tables: no centers");
    bool any = false;
    for (float v : density.values())
        if (v > 0.0f) {
            any = true;
            break;
        }
    if (!any) throw Error(Errc::bad_value, "precompute_tables: empty medium");
    FeatureTable table;
    table.lambda = cfg.lambda;
    table.template_scale = cfg.template_scale;
    table.combiner = CombinerWeights::identity(pyramid.level_count());
    TransmittanceFeatureVolume tvol = build_transmittance_volume(pyramid, centers[0].light, table.combiner, cfg);
    table.phase_table = PhaseTable(cfg.phase_g_res, cfg.phase_angle_res, cfg.phase_aperture_res, cfg.phase_quad_nodes);
    std::vector<double> rows;
    rows.reserve(centers.size() * 9);
    for (const CenterSpec& c : centers)
        rows.insert(rows.end(), {c.p.x, c.p.y, c.p.z, c.omega.x, c.omega.y, c.omega.z, c.light.x, c.light.y,
                                 c.light.z});
    const sf_phase_model m = model.to_c();
    for (int kind = 0; kind < 2; ++kind) {
        const SamplingTemplate& t = kind == 0 ? diffuse_tmpl : highlight_tmpl;
        auto dev = t.device();
        const int n = t.total_points();
        std::vector<float> out(centers.size() * size_t(3) * n);
        check(sf_sample_features(density.handle(), tvol.handle(), dev.get(), &m, table.phase_table.handle(),
                                 cfg.template_scale, int64_t(centers.size()), rows.data(), out.data(), nullptr));
        auto& blocks = kind == 0 ? table.diffuse : table.highlight;
        blocks.resize(centers.size());
        for (size_t i = 0; i < centers.size(); ++i) {
            const float* o = out.data() + i * size_t(3) * n;
            blocks[i] = SampleFeatureBlock{centers[i].p, centers[i].omega, centers[i].light,
                                           std::vector<float>(o, o + n), std::vector<float>(o + n, o + 2 * n),
                                           std::vector<float>(o + 2 * n, o + 3 * n)};
        }
    }
    return table;
}

// predict_field (inc/predictor.h:138-139, src/predictor.cpp:531-543): make_config + predict_y +
// decode_prediction for every center of the table, batched (sf_predict).
inline std::vector<Vec3> predict_field(const Backbone& net, const FeatureTable& table, const MediumProperties& props,
                                       const PhaseModel& phase, int precision = SF_PRECISION_FP32) {
    if (table.diffuse.size() != table.highlight.size())
        throw Error(Errc::shape_mismatch, "feature table kinds disagree on center count");
    const size_t n = table.diffuse.size();
    std::vector<float> feats;
    std::vector<double> cfg8;
    for (size_t i = 0; i < n; ++i) {
        const SampleFeatureBlock& d = table.diffuse[i];
        const SampleFeatureBlock& h = table.highlight[i];
        for (const auto* v : {&d.density, &d.transmittance, &d.phase, &h.density, &h.transmittance, &h.phase})
            feats.insert(feats.end(), v->begin(), v->end());
        const ConfigParams c = make_config(props, phase, d.omega, d.light);
        double row[8] = {double(c.g_params.size()), 0, 0, 0, c.albedo.x, c.albedo.y, c.albedo.z, c.alpha};
        for (size_t k = 0; k < c.g_params.size() && k < 3; ++k) row[1 + k] = c.g_params[k];
        cfg8.insert(cfg8.end(), row, row + 8);
    }
    std::vector<double> F(3 * n);
    if (n) check(sf_predict(net.handle(), int64_t(n), feats.data(), cfg8.data(), precision, nullptr, F.data(), nullptr));
    std::vector<Vec3> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = {F[3 * i], F[3 * i + 1], F[3 * i + 2]};
    return out;
}

// ---- image entry point (inc/camera.h, inc/rte.h, inc/image.h) ----------------------------
struct Camera {
    Vec3 position, look_at{0, 0, 0}, up{0, 1, 0};
    double vfov_degrees = 40.0;
    int width = 64, height = 64;
    Camera() = default;
    // Camera(position, look_at, up, vfov_degrees, width, height) (inc/camera.h:19-20)
    Camera(const Vec3& pos, const Vec3& at, const Vec3& u, double vfov, int w, int h)
        : position(pos), look_at(at), up(u), vfov_degrees(vfov), width(w), height(h) {}
};

struct RenderOptions {
    double step_scale = 0.5;
    Vec3 background{0.0, 0.0, 0.0};
};

struct ImageF {
    int width = 0, height = 0;
    std::vector<float> rgb;  // width * height * 3, row-major
};

// render_neural (inc/predictor.h:145-149, src/predictor.cpp:585-614) with the reference's
// signature: lambda, template scale, combiner and phase table come from the FeatureTable; the
// transmittance feature volume is built for light.direction on the GPU, F is baked at every
// occupied voxel centre (sf_bake_field: the fused query, omega toward the voxel from the
// camera) and the image marched with render_volume's midpoint rule (sf_render_volume).
inline ImageF render_neural(const Medium& medium, const DistantLight& light, const Camera& camera,
                            const Backbone& net, const FeatureTable& table, const SamplingTemplate& diffuse_tmpl,
                            const SamplingTemplate& highlight_tmpl, const FeatureConfig& fcfg,
                            const RenderOptions& ropts = {}, int precision = SF_PRECISION_FP32) {
    medium.props.validate();
    medium.phase.validate();
    light.validate();
    if (!table.phase_table.handle()) throw Error(Errc::invalid_argument, "render_neural: feature table has no phase table");
    FeatureConfig cfg = fcfg;
    cfg.lambda = table.lambda;
    cfg.template_scale = table.template_scale;
    DensityPyramid pyramid(medium.grid);
    if (table.combiner.level_count() != pyramid.level_count())
        throw Error(Errc::shape_mismatch, "combine_transmittance: weight/level mismatch");
    TransmittanceFeatureVolume tvol = build_transmittance_volume(pyramid, light.direction, table.combiner, cfg);
    Scene scene(medium.grid, tvol, diffuse_tmpl, highlight_tmpl, medium.phase, table.phase_table, cfg.template_scale);
    // make_config per voxel differs only in alpha (validated for every voxel by the reference;
    // alpha = angle_between is always in [0, pi]): the medium part is validated once here
    const ConfigParams med = make_config(medium.props, medium.phase, light.direction, light.direction);
    const sf_medium_params m = detail::medium_params(med);
    int dims[3];
    double vs, o[3];
    check(sf_grid_info(medium.grid.handle(), dims, &vs, o));
    std::vector<float> field(size_t(3) * dims[0] * dims[1] * dims[2]);
    double cp[3] = {camera.position.x, camera.position.y, camera.position.z};
    check(sf_bake_field(scene.handle(), net.handle(), &m, cp, precision, field.data(), nullptr));
    ImageF img{camera.width, camera.height, std::vector<float>(size_t(camera.width) * camera.height * 3)};
    const MediumProperties& pr = medium.props;
    double st[3] = {pr.sigma_t_scale.x, pr.sigma_t_scale.y, pr.sigma_t_scale.z};
    double al[3] = {pr.albedo.x, pr.albedo.y, pr.albedo.z};
    double la[3] = {camera.look_at.x, camera.look_at.y, camera.look_at.z};
    double up[3] = {camera.up.x, camera.up.y, camera.up.z};
    double bg[3] = {ropts.background.x, ropts.background.y, ropts.background.z};
    check(sf_render_volume(medium.grid.handle(), st, al, int(pr.material_class), cp, la, up, camera.vfov_degrees,
                           camera.width, camera.height, field.data(), ropts.step_scale, bg, img.rgb.data(), nullptr));
    return img;
}

// ---- artifact readers a reference caller uses next to render_neural -------------------------
// load_density (.vgrid, inc/volume_grid.h:94-98, src/volume_grid.cpp:175-222)
inline DensityGrid load_density(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(Errc::io, "load_density: cannot open '" + path + "'");
    char magic[4] = {};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "VGRD", 4) != 0)
        throw Error(Errc::malformed_header, "load_density: bad magic in '" + path + "'");
    uint32_t version = 0, dims[3] = {0, 0, 0};
    float vs = 0.0f, org[3] = {0, 0, 0};
    in.read(reinterpret_cast<char*>(&version), 4);
    if (!in || version != 1) throw Error(Errc::malformed_header, "load_density: unsupported version");
    in.read(reinterpret_cast<char*>(dims), 12);
    in.read(reinterpret_cast<char*>(&vs), 4);
    in.read(reinterpret_cast<char*>(org), 12);
    if (!in) throw Error(Errc::malformed_header, "load_density: truncated header");
    for (uint32_t d : dims)
        if (d == 0 || d > (1u << 16) || (d & (d - 1))) throw Error(Errc::bad_dims, "load_density: dims must be powers of two");
    if (!(vs > 0.0f) || !std::isfinite(vs)) throw Error(Errc::bad_value, "load_density: voxel_size must be positive");
    std::vector<float> v(size_t(dims[0]) * dims[1] * dims[2]);
    in.read(reinterpret_cast<char*>(v.data()), std::streamsize(v.size() * sizeof(float)));
    if (size_t(in.gcount()) != v.size() * sizeof(float))
        throw Error(Errc::truncated, "load_density: truncated payload in '" + path + "'");
    for (float x : v) {
        if (!std::isfinite(x)) throw Error(Errc::bad_value, "load_density: non-finite density");
        if (x < 0.0f) throw Error(Errc::bad_value, "load_density: negative density");
    }
    return DensityGrid(int(dims[0]), int(dims[1]), int(dims[2]), vs, {org[0], org[1], org[2]}, v.data());
}

namespace detail {
// The JSON subset of .vtmpl files (objects, arrays, numbers, strings, literals).
struct Json {
    enum Kind { Null, Num, Str, Arr, Obj, Bool } kind = Null;
    double num = 0.0;
    std::string str;
    std::vector<Json> arr;
    std::map<std::string, Json> obj;
    const Json& at(const std::string& k) const {
        auto it = obj.find(k);
        if (kind != Obj || it == obj.end()) throw Error(Errc::malformed_header, "load_template: missing key '" + k + "'");
        return it->second;
    }
    double number() const {
        if (kind != Num) throw Error(Errc::malformed_header, "load_template: number expected");
        return num;
    }
};
struct JsonParser {
    const std::string& s;
    size_t i = 0;
    [[noreturn]] void bad() { throw Error(Errc::malformed_header, "load_template: JSON syntax error"); }
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    Json value() {
        ws();
        if (i >= s.size()) bad();
        Json j;
        const char c = s[i];
        if (c == '{') {
            j.kind = Json::Obj;
            ++i;
            ws();
            if (i < s.size() && s[i] == '}') return ++i, j;
            for (;;) {
                ws();
                Json k = value();
                if (k.kind != Json::Str) bad();
                ws();
                if (i >= s.size() || s[i++] != ':') bad();
                j.obj[k.str] = value();
                ws();
                if (i < s.size() && s[i] == ',') { ++i; continue; }
                if (i < s.size() && s[i] == '}') { ++i; break; }
                bad();
            }
        } else if (c == '[') {
            j.kind = Json::Arr;
            ++i;
            ws();
            if (i < s.size() && s[i] == ']') return ++i, j;
            for (;;) {
                j.arr.push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') { ++i; continue; }
                if (i < s.size() && s[i] == ']') { ++i; break; }
                bad();
            }
        } else if (c == '"') {
            j.kind = Json::Str;
            ++i;
            while (i < s.size() && s[i] != '"') j.str += s[i++];
            if (i >= s.size()) bad();
            ++i;
        } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 5, "false") == 0 || s.compare(i, 4, "null") == 0) {
            j.kind = s[i] == 'n' ? Json::Null : Json::Bool;
            j.num = s[i] == 't' ? 1.0 : 0.0;
            i += s[i] == 'f' ? 5 : 4;
        } else {
            const char* b = s.c_str() + i;
            char* e = nullptr;
            j.kind = Json::Num;
            j.num = std::strtod(b, &e);  // round-trips the %.17g numbers save_template writes
            if (e == b) bad();
            i += size_t(e - b);
        }
        return j;
    }
};
}  // namespace detail

// load_template (.vtmpl JSON, inc/templates.h, src/templates.cpp:286-328)
inline SamplingTemplate load_template(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error(Errc::io, "load_template: cannot open '" + path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    detail::JsonParser p{text};
    const detail::Json j = p.value();
    SamplingTemplate t;
    const std::string kind = j.at("kind").str;
    if (kind == "diffuse")
        t.kind = SF_TEMPLATE_DIFFUSE;
    else if (kind == "highlight")
        t.kind = SF_TEMPLATE_HIGHLIGHT;
    else
        throw Error(Errc::bad_value, "load_template: unknown kind '" + kind + "'");
    t.seed = uint64_t(j.at("seed").number());
    if (t.kind == SF_TEMPLATE_HIGHLIGHT) {
        t.gen_distance = j.at("gen_distance").number();
        t.cone_half_angle = j.at("cone_half_angle").number();
    }
    for (const detail::Json& jl : j.at("layers").arr) {
        TemplateLayer layer;
        layer.index = int(jl.at("index").number());
        layer.radius = jl.at("radius").number();
        layer.cap_radius = jl.at("cap_radius").number();
        for (const detail::Json& pt : jl.at("points").arr) {
            if (pt.arr.size() != 3) throw Error(Errc::malformed_header, "load_template: point must have 3 components");
            layer.points.push_back({pt.arr[0].number(), pt.arr[1].number(), pt.arr[2].number()});
        }
        if (double(layer.points.size()) != jl.at("count").number())
            throw Error(Errc::truncated, "load_template: point count mismatch");
        t.layers.push_back(std::move(layer));
    }
    return t;
}

}  // namespace scatterfield_b200
