// sf_device.cuh — device-side numeric primitives of the hot path.
//
// Every function restates one reference primitive with the same operation order
// so FP64 results are bit-identical to the CPU reference (the library is built
// with --fmad=false; IEEE div/sqrt are correctly rounded on both sides). Citations
// are relative to /root/reference/proj/core.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/scatterfield_b200.h"

namespace sfb {

constexpr double kPi = 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);

// DensityGrid geometry in device form (inc/volume_grid.h:17-58). hi = origin +
// n*vs computed on the host exactly as DensityGrid::bounds (src/volume_grid.cpp:35-38).
struct GridDev {
    const float* v;
    int nx, ny, nz;
    double vs;
    double ox, oy, oz;
    double hx, hy, hz;
    double ivs;  // 1/vs when vs is a power of two (x/vs == x*ivs exactly), else 0
    // strides of the padded xy-quad record layout (k_xpair), in 32-byte records: per y row / per
    // z brick slab
    uint32_t rec_sx, rec_sz;
};

struct PhaseDev {
    int kind;  // 0 iso, 1 HG, 2 multi-HG
    int n_lobes;
    double w[3];
    double g[3];
    const float* table;
    int gr, ar, hr;
    const float4* quad;  // sf_phase_table::d_quad (mixed-media production sampler), or null
};

#if defined(__CUDACC__)

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

// clamp(v, lo, hi) = std::min(hi, std::max(lo, v)) (inc/math.h:51)
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    double m = (lo < v) ? v : lo;
    return (m < hi) ? m : hi;
}

__device__ __forceinline__ bool in_box(const GridDev& g, double px, double py, double pz) {
    return px >= g.ox && px <= g.hx && py >= g.oy && py <= g.hy && pz >= g.oz && pz <= g.hz;
}

// Continuous voxel coordinate, cell and weights (src/volume_grid.cpp:45-56).
struct Cell {
    int x0, y0, z0, x1, y1, z1;
    double tx, ty, tz;
};

__device__ __forceinline__ Cell cell_of(const GridDev& g, double px, double py, double pz) {
    double fx, fy, fz;
    if (g.ivs != 0.0) {  // exact: scaling by a power of two
        fx = (px - g.ox) * g.ivs - 0.5;
        fy = (py - g.oy) * g.ivs - 0.5;
        fz = (pz - g.oz) * g.ivs - 0.5;
    } else {
        fx = (px - g.ox) / g.vs - 0.5;
        fy = (py - g.oy) / g.vs - 0.5;
        fz = (pz - g.oz) / g.vs - 0.5;
    }
    Cell c;
    c.x0 = int(floor(fx));
    c.y0 = int(floor(fy));
    c.z0 = int(floor(fz));
    c.tx = fx - c.x0;
    c.ty = fy - c.y0;
    c.tz = fz - c.z0;
    c.x1 = clampi(c.x0 + 1, 0, g.nx - 1);
    c.y1 = clampi(c.y0 + 1, 0, g.ny - 1);
    c.z1 = clampi(c.z0 + 1, 0, g.nz - 1);
    c.x0 = clampi(c.x0, 0, g.nx - 1);
    c.y0 = clampi(c.y0, 0, g.ny - 1);
    c.z0 = clampi(c.z0, 0, g.nz - 1);
    return c;
}

__device__ __forceinline__ double lerp1(double a, double b, double t) { return a + t * (b - a); }

// DensityGrid::sample_trilinear (src/volume_grid.cpp:40-62): 0 outside the closed box.
__device__ __forceinline__ double trilinear(const GridDev& g, double px, double py, double pz) {
    if (!in_box(g, px, py, pz)) return 0.0;
    Cell c = cell_of(g, px, py, pz);
    const float* v = g.v;
    const size_t sy = size_t(g.nx), sz = size_t(g.nx) * g.ny;
    double c00 = lerp1(v[c.z0 * sz + c.y0 * sy + c.x0], v[c.z0 * sz + c.y0 * sy + c.x1], c.tx);
    double c10 = lerp1(v[c.z0 * sz + c.y1 * sy + c.x0], v[c.z0 * sz + c.y1 * sy + c.x1], c.tx);
    double c01 = lerp1(v[c.z1 * sz + c.y0 * sy + c.x0], v[c.z1 * sz + c.y0 * sy + c.x1], c.tx);
    double c11 = lerp1(v[c.z1 * sz + c.y1 * sy + c.x0], v[c.z1 * sz + c.y1 * sy + c.x1], c.tx);
    return lerp1(lerp1(c00, c10, c.ty), lerp1(c01, c11, c.ty), c.tz);
}

// Slab test (inc/math.h:85-107).
__device__ __forceinline__ bool intersect_box(const double lo[3], const double hi[3],
                                              const double o[3], const double d[3], double& t0o,
                                              double& t1o) {
    double t0 = -1e300, t1 = 1e300;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (d[i] == 0.0) {
            if (o[i] < lo[i] || o[i] > hi[i]) return false;
            continue;
        }
        double inv = 1.0 / d[i];
        double ta = (lo[i] - o[i]) * inv;
        double tb = (hi[i] - o[i]) * inv;
        if (ta > tb) {
            double s = ta;
            ta = tb;
            tb = s;
        }
        t0 = (t0 < ta) ? ta : t0;
        t1 = (tb < t1) ? tb : t1;
        if (t0 > t1) return false;
    }
    t0o = t0;
    t1o = t1;
    return true;
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// angle_between (inc/math.h:53-56)
__device__ __forceinline__ double angle_between(const double* a, const double* b) {
    double c = dot3(a, b) / sqrt(dot3(a, a) * dot3(b, b));
    return acos(clampd(c, -1.0, 1.0));
}

// light_entry_point (src/feature_pipeline.cpp:130-137)
__device__ __forceinline__ void light_entry(const double lo[3], const double hi[3],
                                            const double p[3], const double light[3],
                                            double entry[3]) {
    double len = sqrt(dot3(light, light));
    double ld[3] = {light[0] / len, light[1] / len, light[2] / len};
    double ts[3] = {-ld[0], -ld[1], -ld[2]};
    double t0, t1;
    if (!intersect_box(lo, hi, p, ts, t0, t1)) {
        entry[0] = p[0] - ld[0] * 1e-9;
        entry[1] = p[1] - ld[1] * 1e-9;
        entry[2] = p[2] - ld[2] * 1e-9;
        return;
    }
    double t = (t1 < 1e-9) ? 1e-9 : t1;
    entry[0] = p[0] + ts[0] * t;
    entry[1] = p[1] + ts[1] * t;
    entry[2] = p[2] + ts[2] * t;
}

// orthonormal_basis (inc/math.h:59-65)
__device__ __forceinline__ void orthonormal_basis(const double* n, double* t, double* b) {
    double sign = copysign(1.0, n[2]);
    double a = -1.0 / (sign + n[2]);
    double c = n[0] * n[1] * a;
    t[0] = 1.0 + sign * n[0] * n[0] * a;
    t[1] = sign * c;
    t[2] = -sign * n[0];
    b[0] = c;
    b[1] = sign + n[1] * n[1] * a;
    b[2] = -n[1];
}

// PhaseTable::lookup_hg (src/phase.cpp:191-219): FP64 trilinear over the float table.
__device__ __forceinline__ void table_coord(double v, double lo, double hi, int res, int& i0,
                                           double& t) {
    double u = (clampd(v, lo, hi) - lo) / (hi - lo) * (res - 1);
    int i = int(u);
    i0 = i < res - 2 ? i : res - 2;
    t = u - i0;
}

__device__ __forceinline__ double lookup_hg(const float* __restrict__ T, int gr, int ar, int hr,
                                            double g, double angle, double half) {
    int gi, ai, hi;
    double gt, at, ht;
    table_coord(g, -0.99, 0.99, gr, gi, gt);
    table_coord(angle, 0.0, kPi, ar, ai, at);
    table_coord(half, 0.0, kPi, hr, hi, ht);
    double v = 0.0;
#pragma unroll
    for (int dg = 0; dg < 2; ++dg) {
        double wg = dg ? gt : 1.0 - gt;
#pragma unroll
        for (int da = 0; da < 2; ++da) {
            double wa = da ? at : 1.0 - at;
            const float* row = T + (size_t(gi + dg) * ar + (ai + da)) * hr + hi;
            v += wg * wa * (1.0 - ht) * double(__ldg(row));
            v += wg * wa * ht * double(__ldg(row + 1));
        }
    }
    return v;
}

// PhaseTable::lookup (src/phase.cpp:221-230) for a cap with unit `axis`.
__device__ __forceinline__ double phase_lookup(const PhaseDev& pm, const double* fixed_dir,
                                               const double* axis, double half) {
    double angle = angle_between(fixed_dir, axis);
    if (pm.kind == 0) return lookup_hg(pm.table, pm.gr, pm.ar, pm.hr, 0.0, angle, half);
    double v = 0.0;
    for (int k = 0; k < pm.n_lobes; ++k)
        v += pm.w[k] * lookup_hg(pm.table, pm.gr, pm.ar, pm.hr, pm.g[k], angle, half);
    return v;
}

// make_config row {n_g, g0, g1, g2, albedo rgb, alpha = angle_between(omega, l)}
// (src/predictor.cpp:261-274): scene-wide medium, or per-query {g, albedo rgb} (one HG lobe).
__device__ __forceinline__ void write_cfg8(const sf_medium_params& m, const double* media, const double* c,
                                           double* o) {
    if (media) {
        o[0] = 1.0;
        o[1] = media[0];
        o[2] = 0.0;
        o[3] = 0.0;
        o[4] = media[1];
        o[5] = media[2];
        o[6] = media[3];
    } else {
        o[0] = m.n_g;
        o[1] = m.n_g > 0 ? m.g[0] : 0.0;
        o[2] = m.n_g > 1 ? m.g[1] : 0.0;
        o[3] = m.n_g > 2 ? m.g[2] : 0.0;
        o[4] = m.albedo[0];
        o[5] = m.albedo[1];
        o[6] = m.albedo[2];
    }
    o[7] = angle_between(c + 3, c + 6);
}

#endif  // __CUDACC__

#if defined(__CUDACC__)
// Exclusive scan of one int per thread across the block (warp shuffles + one shared-memory pass
// over the warp totals; blockDim.x a multiple of 32, <= 1024); `total` = the block's sum.
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_sums, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int ws = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ws, off);
            if (lane >= off) ws += y;
        }
        if (lane < nw) warp_sums[lane] = ws;  // inclusive over warps
    }
    __syncthreads();
    total = warp_sums[nw - 1];
    return x - v + (w > 0 ? warp_sums[w - 1] : 0);
}
#endif

}  // namespace sfb
