// sf_exact.cuh — the exact (FP64, reference-order) per-point feature of sample_features
// (src/feature_pipeline.cpp:139-172), shared by the parity kernel k_sample_features (sf_query.cu)
// and the production sampler's exact fallback for degenerate highlight placements (sf_fused.cu).
#pragma once

#include "sf_internal.h"

namespace sfb {

// {density, transmittance} at s (sample_trilinear + TransmittanceFeatureVolume::sample,
// src/volume_grid.cpp:40-62, inc/feature_pipeline.h:44-46).
__device__ __forceinline__ void sample_dt(const SceneDev& sc, const double* s, double& rho,
                                          double& tr) {
    const GridDev& g = sc.grid;
    if (!in_box(g, s[0], s[1], s[2])) {
        rho = 0.0;
        tr = 1.0;
        return;
    }
    if (sc.dt == nullptr) {
        rho = trilinear(g, s[0], s[1], s[2]);
        GridDev t = g;
        t.v = sc.tvol;
        tr = trilinear(t, s[0], s[1], s[2]);
        return;
    }
    Cell c = cell_of(g, s[0], s[1], s[2]);
    const size_t sy = size_t(g.nx), sz = size_t(g.nx) * g.ny;
    const float2* v = sc.dt;
    float2 a000 = __ldg(v + c.z0 * sz + c.y0 * sy + c.x0), a100 = __ldg(v + c.z0 * sz + c.y0 * sy + c.x1);
    float2 a010 = __ldg(v + c.z0 * sz + c.y1 * sy + c.x0), a110 = __ldg(v + c.z0 * sz + c.y1 * sy + c.x1);
    float2 a001 = __ldg(v + c.z1 * sz + c.y0 * sy + c.x0), a101 = __ldg(v + c.z1 * sz + c.y0 * sy + c.x1);
    float2 a011 = __ldg(v + c.z1 * sz + c.y1 * sy + c.x0), a111 = __ldg(v + c.z1 * sz + c.y1 * sy + c.x1);
    double c00 = lerp1(a000.x, a100.x, c.tx), c10 = lerp1(a010.x, a110.x, c.tx);
    double c01 = lerp1(a001.x, a101.x, c.tx), c11 = lerp1(a011.x, a111.x, c.tx);
    rho = lerp1(lerp1(c00, c10, c.ty), lerp1(c01, c11, c.ty), c.tz);
    c00 = lerp1(a000.y, a100.y, c.tx);
    c10 = lerp1(a010.y, a110.y, c.tx);
    c01 = lerp1(a001.y, a101.y, c.tx);
    c11 = lerp1(a011.y, a111.y, c.tx);
    tr = lerp1(lerp1(c00, c10, c.ty), lerp1(c01, c11, c.ty), c.tz);
}

// Placement of template point i for query (p, omega, light): place_template +
// placed_cap_radii (src/templates.cpp:207-256), entry from light_entry_point.
// Returns false when the highlight entry coincides with p (the reference throws).
__device__ __forceinline__ bool place_point(const SceneDev& sc, const TemplateDev& td, int i,
                                            const double* p, const double* omega,
                                            const double* light, double* s, double& cap) {
    const double* q = td.pts + 3 * i;
    if (td.kind == 0) {
        s[0] = p[0] + q[0] * sc.template_scale;
        s[1] = p[1] + q[1] * sc.template_scale;
        s[2] = p[2] + q[2] * sc.template_scale;
        cap = td.caps[i] * sc.template_scale;
        return true;
    }
    const double lo[3] = {sc.grid.ox, sc.grid.oy, sc.grid.oz};
    const double hi[3] = {sc.grid.hx, sc.grid.hy, sc.grid.hz};
    double entry[3];
    light_entry(lo, hi, p, light, entry);
    double span[3] = {p[0] - entry[0], p[1] - entry[1], p[2] - entry[2]};
    double len = sqrt(dot3(span, span));
    if (len <= 0.0) return false;
    double il = 1.0 / len;
    double axis[3] = {span[0] * il, span[1] * il, span[2] * il};
    double od = dot3(omega, axis);
    double t[3] = {omega[0] - axis[0] * od, omega[1] - axis[1] * od, omega[2] - axis[2] * od};
    double tl = sqrt(dot3(t, t));
    double b[3];
    if (tl > 1e-9) {
        double it = 1.0 / tl;
        t[0] = t[0] * it;
        t[1] = t[1] * it;
        t[2] = t[2] * it;
        b[0] = axis[1] * t[2] - axis[2] * t[1];
        b[1] = axis[2] * t[0] - axis[0] * t[2];
        b[2] = axis[0] * t[1] - axis[1] * t[0];
    } else {
        orthonormal_basis(axis, t, b);
    }
    double scale = len / td.gen_distance;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double v = t[c] * q[0] + b[c] * q[1];
        v = v + axis[c] * q[2];
        s[c] = entry[c] + v * scale;
    }
    cap = td.caps[i] * scale;
    return true;
}

// Features of template point i for query row c = (p, omega, light) (9 doubles):
// sample_features' per-point body (src/feature_pipeline.cpp:151-170), FP64, the reference's
// operations in its order, stored as floats. media: NULL, or the query's {g, albedo rgb} (one HG
// lobe at g, config C4). Returns false when the highlight entry coincides with p.
__device__ __forceinline__ bool exact_point_features(const SceneDev& sc, const TemplateDev& td, int i,
                                                     const double* c, const double* media, float& rho_o,
                                                     float& tr_o, float& f_o) {
    const double p[3] = {c[0], c[1], c[2]}, omega[3] = {c[3], c[4], c[5]}, light[3] = {c[6], c[7], c[8]};
    double s[3], cap;
    if (!place_point(sc, td, i, p, omega, light, s, cap)) return false;
    double rho, tr;
    sample_dt(sc, s, rho, tr);
    const double d[3] = {s[0] - p[0], s[1] - p[1], s[2] - p[2]};
    const double dist = sqrt(dot3(d, d));
    double f;
    if (dist <= 0.0) {
        f = 1.0;  // diffuse centre: both caps are the full sphere
    } else {
        const double half = cap >= dist ? kPi : asin(cap / dist);
        const double il = 1.0 / dist;
        const double axis[3] = {d[0] * il, d[1] * il, d[2] * il};
        PhaseDev ph = sc.phase;
        if (media) {  // per-query single-lobe HG (C4: per-voxel g sampled at p by the harness)
            ph.kind = 1;
            ph.n_lobes = 1;
            ph.w[0] = 1.0;
            ph.g[0] = media[0];
        }
        f = phase_lookup(ph, omega, axis, half) * phase_lookup(ph, light, axis, half);
    }
    rho_o = float(rho);
    tr_o = float(tr);
    f_o = float(f);
    return true;
}

}  // namespace sfb
