// Drop-in program for the C++ shim (include/scatterfield_b200.hpp): the reference's C++ call
// sequence as proj/tools/main.cpp's neural render and precompute commands make it
// (load_density, load_template, precompute_tables, predict_field, render_neural with the
// FeatureTable's combiner / lambda / template scale), against the B200 ABI.
//
// usage: shim_smoke FIXTURE_DIR
//   FIXTURE_DIR holds, written by tests/test_gpu_parity.py::test_cpp_shim_runs from
//   tests/golden/render.npz and render_rc.npz (the reference's own images):
//   grid.vgrid, diffuse.vtmpl, highlight.vtmpl, expect_id.f32 (render_neural with the identity
//   combiner), expect_rc.f32 + rc_kernels.f32 + rc_scales.f32 (a random combiner).
// Exit 0 when every check holds; prints one line per check.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "scatterfield_b200.hpp"

namespace sf = scatterfield_b200;

static std::vector<float> read_f32(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw sf::Error(sf::Errc::io, "cannot open " + path);
    const std::streamsize n = in.tellg();
    std::vector<float> v(size_t(n) / sizeof(float));
    in.seekg(0);
    in.read(reinterpret_cast<char*>(v.data()), n);
    return v;
}

// |img - ref| <= 1e-3 |ref| + 1e-6 max|ref| (tests/test_gpu_render.py's bound)
static bool image_close(const sf::ImageF& img, const std::vector<float>& ref, double* worst) {
    if (img.rgb.size() != ref.size()) return false;
    double mx = 0.0;
    for (float r : ref) mx = std::fmax(mx, std::fabs(r));
    bool ok = true;
    *worst = 0.0;
    for (size_t i = 0; i < ref.size(); ++i) {
        const double d = std::fabs(double(img.rgb[i]) - ref[i]);
        *worst = std::fmax(*worst, d / (std::fabs(ref[i]) + 1e-30));
        if (d > 1e-3 * std::fabs(ref[i]) + 1e-6 * mx) ok = false;
    }
    return ok;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::printf("usage: shim_smoke FIXTURE_DIR\n");
        return 64;
    }
    const std::string dir = argv[1];
    int fails = 0;
    auto report = [&](const char* what, bool ok) {
        std::printf("%-58s %s\n", what, ok ? "ok" : "FAIL");
        fails += ok ? 0 : 1;
    };
    try {
        // ---- the reference render scene (tests/golden/make_golden.py RENDER)
        sf::Medium medium{sf::load_density(dir + "/grid.vgrid"), {}, sf::PhaseModel::hg(0.7)};
        medium.props.sigma_t_scale = {14.0, 12.0, 10.0};
        medium.props.albedo = {0.45, 0.40, 0.35};
        medium.props.material_class = sf::MaterialClass::Gas;
        const double ln = std::sqrt(0.2 * 0.2 + 1.0 + 0.1 * 0.1);
        sf::DistantLight light{{0.2 / ln, -1.0 / ln, 0.1 / ln}, {1.0, 1.0, 1.0}};
        sf::Camera cam({0.3, 0.2, -3.5}, {0.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, 40.0, 24, 16);
        const sf::SamplingTemplate dt = sf::load_template(dir + "/diffuse.vtmpl");
        const sf::SamplingTemplate ht = sf::load_template(dir + "/highlight.vtmpl");
        report("load_template: 194 diffuse + 72 highlight points", dt.total_points() == 194 && ht.total_points() == 72);
        sf::BackboneConfig bc;
        bc.seed = 0;
        sf::Backbone net(bc);
        sf::DensityPyramid pyr(medium.grid);
        sf::FeatureConfig fcfg;  // lambda 0.6, step 0.5, template scale 1
        fcfg.phase_g_res = 17;
        fcfg.phase_angle_res = 33;
        fcfg.phase_aperture_res = 9;
        fcfg.phase_quad_nodes = 8;
        sf::RenderOptions ro{0.5, {0.05, 0.1, 0.2}};

        // precompute_tables on a few centres, then predict_field == the fused query on the same rows
        std::vector<sf::CenterSpec> centers;
        for (int i = 0; i < 64; ++i) {
            const double a = 0.37 * i, b = 0.11 * i;
            const sf::Vec3 w{std::cos(a) * std::sin(b + 0.3), std::sin(a) * std::sin(b + 0.3), std::cos(b + 0.3)};
            centers.push_back({{-0.3 + 0.01 * i, 0.2 - 0.005 * i, 0.05 * std::sin(a)}, w, light.direction});
        }
        sf::FeatureTable table = sf::precompute_tables(medium.grid, pyr, dt, ht, centers, medium.phase, fcfg);
        report("precompute_tables: one block per centre and kind",
               table.diffuse.size() == 64 && table.highlight.size() == 64 && table.diffuse[0].density.size() == 194);
        std::vector<sf::Vec3> F = sf::predict_field(net, table, medium.props, medium.phase);
        sf::TransmittanceFeatureVolume tvol =
            sf::build_transmittance_volume(pyr, light.direction, table.combiner, fcfg);
        sf::Scene scene(medium.grid, tvol, dt, ht, medium.phase, table.phase_table, fcfg.template_scale);
        std::vector<double> rows;
        for (const auto& c : centers)
            rows.insert(rows.end(), {c.p.x, c.p.y, c.p.z, c.omega.x, c.omega.y, c.omega.z, c.light.x, c.light.y,
                                     c.light.z});
        const sf::ConfigParams med = sf::make_config(medium.props, medium.phase, centers[0].omega, light.direction);
        std::vector<double> Fq = sf::query(scene, net, med, rows);
        bool same = true;
        for (size_t i = 0; i < centers.size(); ++i)
            same = same && F[i].x == Fq[3 * i] && F[i].y == Fq[3 * i + 1] && F[i].z == Fq[3 * i + 2];
        report("predict_field == fused query (bit-identical)", same);

        // render_neural with the reference signature, identity combiner (precompute_tables')
        double worst = 0.0;
        sf::ImageF img = sf::render_neural(medium, light, cam, net, table, dt, ht, fcfg, ro);
        const bool id_ok = image_close(img, read_f32(dir + "/expect_id.f32"), &worst);
        std::printf("  identity combiner: max relative deviation %.3e\n", worst);
        report("render_neural == reference image (1e-3)", id_ok);

        // the same call with a random 3D-CNN combiner in the table (reference image made with it)
        const std::vector<float> k = read_f32(dir + "/rc_kernels.f32"), s = read_f32(dir + "/rc_scales.f32");
        sf::FeatureTable rc = table;
        for (size_t l = 0; l < rc.combiner.kernels.size(); ++l) {
            for (int t = 0; t < 27; ++t) rc.combiner.kernels[l][size_t(t)] = k[27 * l + size_t(t)];
            rc.combiner.scales[l] = s[l];
        }
        sf::ImageF img_rc = sf::render_neural(medium, light, cam, net, rc, dt, ht, fcfg, ro);
        const bool rc_ok = image_close(img_rc, read_f32(dir + "/expect_rc.f32"), &worst);
        std::printf("  random combiner: max relative deviation %.3e\n", worst);
        report("render_neural honours table.combiner (1e-3)", rc_ok);
        bool differs = false;
        for (size_t i = 0; i < img.rgb.size(); ++i) differs = differs || img.rgb[i] != img_rc.rgb[i];
        report("the combiner changes the image", differs);

        // reference error behaviour
        auto throws = [&](auto&& fn, sf::Errc code) {
            try {
                fn();
            } catch (const sf::Error& e) {
                return e.code() == code;
            }
            return false;
        };
        sf::DistantLight bad = light;
        bad.direction = {0.0, -2.0, 0.0};
        report("non-unit light direction -> bad_value",
               throws([&] { sf::render_neural(medium, bad, cam, net, table, dt, ht, fcfg, ro); }, sf::Errc::bad_value));
        sf::MediumProperties dense = medium.props;
        dense.albedo = {0.99, 0.99, 0.99};  // outside the gas class range
        report("make_config: albedo outside the class range -> bad_value",
               throws([&] { dense.validate(); }, sf::Errc::bad_value));
        report("precompute_tables: no centres -> invalid_argument",
               throws([&] { sf::precompute_tables(medium.grid, pyr, dt, ht, {}, medium.phase, fcfg); },
                      sf::Errc::invalid_argument));
        report("load_template: missing file -> io",
               throws([&] { sf::load_template(dir + "/missing.vtmpl"); }, sf::Errc::io));

        // sharded build: two slabs == the full build's rows
        const int n = medium.grid.nx();
        std::vector<float> full = tvol.values().values();
        std::vector<float> a = sf::build_transmittance_slab(pyr, light.direction, table.combiner, fcfg, 0, 7, n, n);
        std::vector<float> c = sf::build_transmittance_slab(pyr, light.direction, table.combiner, fcfg, 7, n, n, n);
        a.insert(a.end(), c.begin(), c.end());
        report("build_transmittance_slab: slabs == full build", a == full);
    } catch (const sf::Error& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
    return fails == 0 ? 0 : 2;
}
