// Drop-in smoke program for the C++ shim (include/scatterfield_b200.hpp): the
// reference's C++ call sequence (render_neural's per-light build + one
// sample_features + predict_y, src/predictor.cpp:585-609) against the B200 ABI.
// tests/test_abi_host.py syntax-checks it on CPU; tests/test_gpu_parity.py
// builds and runs it on the GPU.
#include <cstdio>
#include <vector>

#include "scatterfield_b200.hpp"

namespace sf = scatterfield_b200;

int main() {
    const int n = 16;
    std::vector<float> v(size_t(n) * n * n, 0.0f);
    for (int z = 4; z < 12; ++z)
        for (int y = 4; y < 12; ++y)
            for (int x = 4; x < 12; ++x) v[(size_t(z) * n + y) * n + x] = 1.0f;
    try {
        sf::DensityGrid grid(n, n, n, 2.0 / n, {-1, -1, -1}, v.data());
        sf::DensityPyramid pyr(grid);
        sf::Vec3 light{0.0, -1.0, 0.0};
        sf::TransmittanceFeatureVolume tvol = sf::build_transmittance_volume(
            pyr, light, sf::CombinerWeights::identity(pyr.level_count()), sf::FeatureConfig{});
        sf::PhaseTable table(17, 33, 9, 8);
        sf::SamplingTemplate dt;
        dt.kind = SF_TEMPLATE_DIFFUSE;
        dt.layers.push_back({0, 0.1, 0.05, {{0, 0, 0}, {0.05, 0, 0}}});
        sf::SampleFeatureBlock b = sf::sample_features({0, 0, 0}, {0, 0, 1}, light, dt, grid, tvol,
                                                       sf::PhaseModel::hg(0.7), table, 1.0);
        std::printf("density %.6f trans %.6f phase %.6f levels %d\n", b.density[0], b.transmittance[0],
                    b.phase[0], pyr.level_count());
        if (!(b.density[0] == 1.0f && b.phase[0] == 1.0f && pyr.level_count() == 5)) return 2;
        // sharded build: two slabs == the full build's rows
        sf::FeatureConfig fc;
        auto w = sf::CombinerWeights::identity(pyr.level_count());
        std::vector<float> full = tvol.values().values();
        std::vector<float> a = sf::build_transmittance_slab(pyr, light, w, fc, 0, 7, n, n);
        std::vector<float> c = sf::build_transmittance_slab(pyr, light, w, fc, 7, n, n, n);
        a.insert(a.end(), c.begin(), c.end());
        if (a != full) return 3;
        // render_neural with the reference's default backbone on an empty-ish camera view:
        // pixels missing the box show the background exactly
        sf::Camera cam{{0.0, 0.0, -4.0}, {0, 0, 0}, {0, 1, 0}, 40.0, 16, 12};
        sf::RenderOptions ro{0.5, {0.1, 0.2, 0.3}};
        sf::SamplingTemplate d8, h8;  // default-size templates are loaded by the Python tests
        d8.kind = SF_TEMPLATE_DIFFUSE;
        d8.layers.push_back({0, 0.0, 0.05, {{0, 0, 0}}});
        h8.kind = SF_TEMPLATE_HIGHLIGHT;
        h8.gen_distance = 1.0;
        h8.cone_half_angle = 0.087;
        h8.layers.push_back({0, 0.1, 0.05, {{0, 0, 0.5}}});
        sf::BackboneConfig bc;
        bc.diffuse_counts = {1};
        bc.highlight_counts = {1};
        sf::Backbone net(bc);
        sf::ConfigParams med{{0.7}, {0.4, 0.4, 0.4}, 0.0};
        sf::ImageF img = sf::render_neural(grid, pyr, light, cam, net, table, d8, h8, sf::PhaseModel::hg(0.7),
                                           {4, 4, 4}, med, sf::MaterialClass::Gas, fc, ro);
        std::printf("render %dx%d corner %.3f %.3f %.3f\n", img.width, img.height, img.rgb[0], img.rgb[1], img.rgb[2]);
        return (img.rgb.size() == 16 * 12 * 3 && img.rgb[0] == 0.1f && img.rgb[2] == 0.3f) ? 0 : 4;
    } catch (const sf::Error& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
}
