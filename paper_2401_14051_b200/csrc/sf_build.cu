// sf_build.cu — per-light build kernels: density mip pyramid (K1), graded
// transmittance march (K2), the 3x3x3 combiner "3D-CNN" (K3), the phase-table
// build (K4), plus the small batched primitives exposed for parity tests.
//
// Layout in HBM: every grid is a dense x-fastest float32 array (the reference's
// DensityGrid order, inc/volume_grid.h:28-33), so the level-0 volumes of a 512^3
// scene are 512 MiB each and every coarser level adds 1/8 of the previous.
// All kernels are SIMT: none of these operations has a channel or reduction
// dimension that a tensor-core GEMM could use (the combiner is one 1-in/1-out
// 27-tap stencil per level).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "sf_internal.h"

namespace sfb {

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(size_t n, int block = kBlock) {
    size_t g = (n + block - 1) / block;
    return unsigned(g > 0x7fffffff ? 0x7fffffff : (g == 0 ? 1 : g));
}

// K1: DensityPyramid level k -> k+1 (src/volume_grid.cpp:91-126). FP64 sum of the
// eight clamped children in dz,dy,dx order, divided by the count, stored float.
__global__ void k_pyramid_down(const float* __restrict__ src, int sx, int sy, int sz,
                               float* __restrict__ dst, int dx, int dy, int dz) {
    size_t n = size_t(dx) * dy * dz;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < n;
         idx += size_t(gridDim.x) * blockDim.x) {
        int x = int(idx % dx);
        int y = int((idx / dx) % dy);
        int z = int(idx / (size_t(dx) * dy));
        double sum = 0.0;
        int count = 0;
#pragma unroll
        for (int cz = 0; cz < 2; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                for (int cx = 0; cx < 2; ++cx) {
                    int ix = min(2 * x + cx, sx - 1);
                    int iy = min(2 * y + cy, sy - 1);
                    int iz = min(2 * z + cz, sz - 1);
                    sum += src[(size_t(iz) * sy + iy) * sx + ix];
                    ++count;
                }
        dst[idx] = float(sum / count);
    }
}

// Per-level x-pair copy of a density level in FP64: {double(v(x)), double(v(min(x+1, nx-1)))}.
// The march below then reads the 8 corners of a trilinear cell as 4 16-byte loads with the
// float->double conversions done once per voxel instead of once per sample.
__global__ void k_xpair_f64(const float* __restrict__ v, int nx, int ny, int nz, double2* __restrict__ out) {
    const int n = nx * ny * nz;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int x = i % nx;
        out[i] = make_double2(double(v[i]), double(v[x + 1 < nx ? i + 1 : i]));
    }
}

// DensityGrid::sample_trilinear (src/volume_grid.cpp:40-62) on the x-pair copy: the same FP64
// operations in the same order as sf_device.cuh trilinear(). At x0 = -1 the reference lerps
// v(0) with itself; the pair at 0 is {v(0), v(1)}, so tx = 0 gives v(0) + 0 * (v(1) - v(0)) =
// v(0) exactly. At x0 = nx-1 the pair is {v(nx-1), v(nx-1)} as in the reference.
// The march calls it only at points strictly inside the closed box (a ray from a voxel centre to
// the box exit, the last sample h/2 before the exit), where the reference's outside test is
// always false, so the test is left out.
__device__ __forceinline__ double trilinear_xp(const GridDev& g, const double2* __restrict__ xp, double px,
                                               double py, double pz) {
    double fx, fy, fz;
    if (g.ivs != 0.0) {
        fx = (px - g.ox) * g.ivs - 0.5;
        fy = (py - g.oy) * g.ivs - 0.5;
        fz = (pz - g.oz) * g.ivs - 0.5;
    } else {
        fx = (px - g.ox) / g.vs - 0.5;
        fy = (py - g.oy) / g.vs - 0.5;
        fz = (pz - g.oz) / g.vs - 0.5;
    }
    const double flx = floor(fx), fly = floor(fy), flz = floor(fz);
    const int x0 = int(flx), y0 = int(fly), z0 = int(flz);
    double tx = fx - flx;
    const double ty = fy - fly, tz = fz - flz;
    if (x0 < 0) tx = 0.0;
    const int xc = x0 < 0 ? 0 : x0;
    const int ya = clampi(y0, 0, g.ny - 1), yb = clampi(y0 + 1, 0, g.ny - 1);
    const int za = clampi(z0, 0, g.nz - 1), zb = clampi(z0 + 1, 0, g.nz - 1);
    const double2* row = xp + ((za * g.ny + ya) * g.nx + xc);
    const int dy = (yb - ya) * g.nx, dz = (zb - za) * g.nx * g.ny;
    const double2 r00 = __ldg(row), r10 = __ldg(row + dy);
    const double2 r01 = __ldg(row + dz), r11 = __ldg(row + dz + dy);
    const double c00 = lerp1(r00.x, r00.y, tx), c10 = lerp1(r10.x, r10.y, tx);
    const double c01 = lerp1(r01.x, r01.y, tx), c11 = lerp1(r11.x, r11.y, tx);
    return lerp1(lerp1(c00, c10, ty), lerp1(c01, c11, ty), tz);
}

// Optical depth of the ray from voxel (x, y, z)'s centre toward the light (graded_transmittance,
// src/feature_pipeline.cpp:57-66, with DensityGrid::optical_depth, src/volume_grid.cpp:64-78):
// intersect_box, q = p + ts * t1, len, n = max(1, ceil(len / step)), h = len / n, dir = d * (1 / len),
// midpoint samples. FP64 throughout, the reference's operations in its order.
__device__ __forceinline__ double graded_tau_f64(const GridDev& g, const double2* __restrict__ xp, int x, int y,
                                                 int z, const double ts[3], double step) {
    const double lo[3] = {g.ox, g.oy, g.oz};
    const double hi[3] = {g.hx, g.hy, g.hz};
    double p[3] = {g.ox + (x + 0.5) * g.vs, g.oy + (y + 0.5) * g.vs, g.oz + (z + 0.5) * g.vs};
    double t0, t1, tau = 0.0;
    if (intersect_box(lo, hi, p, ts, t0, t1) && t1 > 0.0) {
        double q[3] = {p[0] + ts[0] * t1, p[1] + ts[1] * t1, p[2] + ts[2] * t1};
        double d[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
        double len = sqrt(dot3(d, d));
        if (len != 0.0) {
            int ns = int(ceil(len / step));
            ns = ns < 1 ? 1 : ns;
            double h = len / ns;
            double il = 1.0 / len;
            double dir[3] = {d[0] * il, d[1] * il, d[2] * il};
            double sum = 0.0;
            for (int i = 0; i < ns; ++i) {
                double s = (i + 0.5) * h;
                sum += trilinear_xp(g, xp, p[0] + dir[0] * s, p[1] + dir[1] * s, p[2] + dir[2] * s);
            }
            tau = sum * h;
        }
    }
    return tau;
}

// K2: graded transmittance of one level (src/feature_pipeline.cpp:37-68) with the
// midpoint-rule optical depth (src/volume_grid.cpp:64-78), for voxel rows z in [zlo, zhi)
// (a z-slab when the build is sharded over GPUs). One thread per voxel; neighbouring
// threads march neighbouring parallel rays, so a warp's gathers stay within a few lines.
// FP64 throughout, as the reference. (k_graded_taps below is the fast form of the same march.)
__global__ void k_graded(GridDev g, const double2* __restrict__ xp, double tsx, double tsy, double tsz,
                         double coeff, double step, int zlo, int zhi, float* __restrict__ out) {
    const int plane = g.nx * g.ny;
    const int i0 = zlo * plane, i1 = zhi * plane;
    const double ts[3] = {tsx, tsy, tsz};
    for (int idx = i0 + blockIdx.x * blockDim.x + threadIdx.x; idx < i1; idx += gridDim.x * blockDim.x) {
        const int x = idx % g.nx;
        const int y = (idx / g.nx) % g.ny;
        const int z = idx / plane;
        out[idx] = float(exp(-coeff * graded_tau_f64(g, xp, x, y, z, ts, step)));
    }
}

// Production (bf16 query path) variant of K2: the same per-voxel ray setup in FP64
// (intersect_box, len, ns, h, dir exactly as above), then the march in FP32 on float x-pair
// records {v(x), v(min(x+1, nx-1))} with fused multiply-adds and a compensated (Kahan) sum.
// The optical depth differs from the FP64 reference by ~1e-6 relative (tests state 2e-5 on
// T), far below the bf16 rounding of the features it feeds; 2-3x the FP64 march's rate.
__global__ void k_xpair_f32(const float* __restrict__ v, int nx, int ny, int nz, float2* __restrict__ out) {
    const int n = nx * ny * nz;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int x = i % nx;
        out[i] = make_float2(v[i], v[x + 1 < nx ? i + 1 : i]);
    }
}

__device__ __forceinline__ double graded_tau_f32(const GridDev& g, const float2* __restrict__ xp, int x, int y,
                                                 int z, const double ts[3], double step) {
    const int plane = g.nx * g.ny;
    const double lo[3] = {g.ox, g.oy, g.oz};
    const double hi[3] = {g.hx, g.hy, g.hz};
    double p[3] = {g.ox + (x + 0.5) * g.vs, g.oy + (y + 0.5) * g.vs, g.oz + (z + 0.5) * g.vs};
    double t0, t1, tau = 0.0;
    if (intersect_box(lo, hi, p, ts, t0, t1) && t1 > 0.0) {
        double q[3] = {p[0] + ts[0] * t1, p[1] + ts[1] * t1, p[2] + ts[2] * t1};
        double d[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
        double len = sqrt(dot3(d, d));
        if (len != 0.0) {
            int ns = int(ceil(len / step));
            ns = ns < 1 ? 1 : ns;
            const double h = len / ns;
            const double il = 1.0 / len;
            // voxel-space ray: f(s) = f0 + df * s, f0 = the voxel centre's own coordinates
            const float f0[3] = {float(x), float(y), float(z)};
            const float df[3] = {float(d[0] * il * (1.0 / g.vs)), float(d[1] * il * (1.0 / g.vs)),
                                 float(d[2] * il * (1.0 / g.vs))};
            const float hf = float(h);
            float sum = 0.0f, comp = 0.0f;
            // Samples whose cell and its +1 neighbour are in range on every axis need no clamps:
            // [ia, ib) from the ray's interior interval, with a 1e-3 voxel margin, so the fast
            // loop does exactly what the clamped one would (the sum order is unchanged).
            float slo = 0.0f, shi = float(len) * float(1.0 / g.vs) * 2.0f + 4.0f;
            const int nn[3] = {g.nx, g.ny, g.nz};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float lo_f = 1e-3f, hi_f = float(nn[a] - 1) - 1e-3f;  // floor(f) in [0, n - 2]
                if (df[a] > 0.0f) {
                    slo = fmaxf(slo, (lo_f - f0[a]) / df[a]);
                    shi = fminf(shi, (hi_f - f0[a]) / df[a]);
                } else if (df[a] < 0.0f) {
                    slo = fmaxf(slo, (hi_f - f0[a]) / df[a]);
                    shi = fminf(shi, (lo_f - f0[a]) / df[a]);
                } else if (!(f0[a] >= lo_f && f0[a] <= hi_f)) {
                    shi = -1.0f;  // this axis never interior
                }
            }
            int ia = ns, ib = ns;
            if (shi > slo) {
                ia = max(0, int(ceilf(slo / hf - 0.5f)) + 1);
                ib = min(ns, int(floorf(shi / hf - 0.5f)));  // exclusive bound: one sample of margin
                if (ib < ia) ia = ib = ns;
            }
            auto add = [&](float v) {
                const float yk = v - comp;  // Kahan
                const float tk = sum + yk;
                comp = (tk - sum) - yk;
                sum = tk;
            };
            auto clamped = [&](int i) {
                const float sf = (float(i) + 0.5f) * hf;
                const float fx = fmaf(df[0], sf, f0[0]), fy = fmaf(df[1], sf, f0[1]), fz = fmaf(df[2], sf, f0[2]);
                // No box test: every sample lies strictly inside the closed box (the ray runs from
                // a voxel centre to the box exit and the last sample is h/2 before the exit), so
                // sample_trilinear's outside branch (0) never applies; the clamps below still do.
                const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
                const int x0 = int(flx), y0 = int(fly), z0 = int(flz);
                float tx = fx - flx;
                const float ty = fy - fly, tz = fz - flz;
                if (x0 < 0) tx = 0.0f;
                const int xc = x0 < 0 ? 0 : x0;
                const int ya = max(y0, 0), yb = min(y0 + 1, g.ny - 1), za = max(z0, 0), zb = min(z0 + 1, g.nz - 1);
                const float2* row = xp + ((za * g.ny + ya) * g.nx + xc);
                const int dy = (yb - ya) * g.nx, dz = (zb - za) * plane;
                const float2 r00 = __ldg(row), r10 = __ldg(row + dy);
                const float2 r01 = __ldg(row + dz), r11 = __ldg(row + dz + dy);
                const float c00 = fmaf(tx, r00.y - r00.x, r00.x), c10 = fmaf(tx, r10.y - r10.x, r10.x);
                const float c01 = fmaf(tx, r01.y - r01.x, r01.x), c11 = fmaf(tx, r11.y - r11.x, r11.x);
                const float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
                add(fmaf(tz, e1 - e0, e0));
            };
            for (int i = 0; i < ia; ++i) clamped(i);
            for (int i = ia; i < ib; ++i) {  // interior: 0 <= cell, cell + 1 <= n - 1 on every axis
                const float sf = (float(i) + 0.5f) * hf;
                const float fx = fmaf(df[0], sf, f0[0]), fy = fmaf(df[1], sf, f0[1]), fz = fmaf(df[2], sf, f0[2]);
                const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
                const float tx = fx - flx, ty = fy - fly, tz = fz - flz;
                const float2* row = xp + ((int(flz) * g.ny + int(fly)) * g.nx + int(flx));
                const float2 r00 = __ldg(row), r10 = __ldg(row + g.nx);
                const float2 r01 = __ldg(row + plane), r11 = __ldg(row + plane + g.nx);
                const float c00 = fmaf(tx, r00.y - r00.x, r00.x), c10 = fmaf(tx, r10.y - r10.x, r10.x);
                const float c01 = fmaf(tx, r01.y - r01.x, r01.x), c11 = fmaf(tx, r11.y - r11.x, r11.x);
                const float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
                add(fmaf(tz, e1 - e0, e0));
            }
            for (int i = max(ib, ia); i < ns; ++i) clamped(i);
            tau = double(sum) * h;
        }
    }
    return tau;
}

__global__ void k_graded_f32(GridDev g, const float2* __restrict__ xp, double tsx, double tsy, double tsz,
                             double coeff, double step, int zlo, int zhi, float* __restrict__ out) {
    const int plane = g.nx * g.ny;
    const int i0 = zlo * plane, i1 = zhi * plane;
    const double ts[3] = {tsx, tsy, tsz};
    for (int idx = i0 + blockIdx.x * blockDim.x + threadIdx.x; idx < i1; idx += gridDim.x * blockDim.x) {
        const int x = idx % g.nx;
        const int y = (idx / g.nx) % g.ny;
        const int z = idx / plane;
        out[idx] = float(exp(-coeff * graded_tau_f32(g, xp, x, y, z, ts, step)));
    }
}

// ---- K2 as shared tap lists ("graded taps") -------------------------------------------------
// Every voxel whose ray toward the light leaves the box through a face perpendicular to axis E
// has an exit distance t1 = (face - p_E) / ts_E that depends on its E coordinate alone, hence
// the same n, h and the same sample offsets relative to its own centre: the midpoint sum
//     sum_i trilinear(p + dir (i + 1/2) h)
// is one linear functional of the density, translated, for every voxel of that plane. Grouping
// the sum by grid corner gives, with L the lane axis and O the third axis,
//     sum = sum_k  w0 rho[v+o] + w1 rho[v+o+e_L] + w2 rho[v+o+e_O] + w3 rho[v+o+e_L+e_O]
// over "column" taps o_k (the 2 x 2 (L, O) corners of a cell row; ~0.8 taps per sample instead
// of 8 corners), the same value in exact arithmetic. k_tap_build makes the tap list of every
// (E, c) plane once per level and light (FP64 weights); k_graded_cols walks it for 32
// L-consecutive voxels x K O-consecutive voxels per warp: warp-uniform tap loads, coalesced
// 2-corner (L-pair) gathers, and row j + 1 of one voxel's column is row j of the next voxel's,
// so K voxels need K + 1 gathers per tap.
//   E = y (rows x, blocks along z) and E = z (rows x, blocks along y) read x-fastest pairs;
//   E = x (voxels leaving through an x face) reads z-fastest pairs (lanes along z).
// A voxel belongs to the face it leaves through (ties: y, then z, then x). Pair records carry a
// one-voxel halo with the edge values replicated (the pair at L = -1 is {v(0), v(0)}), so the
// clamps of sample_trilinear (src/volume_grid.cpp:45-56) cost nothing: a ray that stays in the
// box only touches corners in [-1, n] on every axis. A voxel whose sample count differs from its
// plane's (len / step within rounding of an integer) marches alone. FP64 taps and sums for the
// exact build (bit-identical to the march in practice), FP32 for the production build.
template <typename W>
struct alignas(16) ColTap {
    W w[4];  // weights of (o), (o + e_L), (o + e_O), (o + e_L + e_O)
    int lin; // o_L s_L + o_E s_E + o_O s_O in the padded record strides (E offset clamped to the grid)
};

struct TapGroup {
    int tap0, n, ns, pad;  // n <= 0: no list (the plane's voxels march)
    double h, texit;
};

constexpr int kTapWarps = 4;
#ifndef SF_COLK
#define SF_COLK 8
#endif
constexpr int kColK = SF_COLK;  // voxels per lane along O: K + 1 row gathers per tap serve K voxels

// Padded pair layout of one lane axis. L = 0: x-fastest, index (x+1) + (y+1) sy + (z+1) sz over
// x in [-1, nx-1], y in [-1, ny], z in [-1, nz]; L = 2: z-fastest, (z+1) + (y+1) sy + (x+1) sx.
struct PadLayout {
    int L;
    int64_t s[3];  // strides of x, y, z
    int64_t count;
};

inline PadLayout pad_layout(int nx, int ny, int nz, int L) {
    PadLayout p;
    p.L = L;
    if (L == 0) {
        p.s[0] = 1;
        p.s[1] = nx + 1;
        p.s[2] = int64_t(nx + 1) * (ny + 2);
        p.count = p.s[2] * (nz + 2);
    } else {
        p.s[2] = 1;
        p.s[1] = nz + 1;
        p.s[0] = int64_t(nz + 1) * (ny + 2);
        p.count = p.s[0] * (nx + 2);
    }
    return p;
}

template <typename T2>
__global__ void k_pad_pairs(const float* __restrict__ v, int nx, int ny, int nz, PadLayout pl, T2* __restrict__ out) {
    const int n[3] = {nx, ny, nz};
    const int a0 = pl.L, a2 = pl.L == 0 ? 2 : 0;
    const int64_t n0 = n[a0] + 1, n1 = ny + 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < pl.count; i += int64_t(gridDim.x) * blockDim.x) {
        int c[3];
        c[a0] = int(i % n0) - 1;
        c[1] = int((i / n0) % n1) - 1;
        c[a2] = int(i / (n0 * n1)) - 1;
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = c[a] < 0 ? 0 : (c[a] > n[a] - 1 ? n[a] - 1 : c[a]);
            hi[a] = lo[a];
        }
        hi[a0] = c[a0] + 1 > n[a0] - 1 ? n[a0] - 1 : c[a0] + 1;
        T2 r;
        r.x = v[(size_t(lo[2]) * ny + lo[1]) * nx + lo[0]];
        r.y = v[(size_t(hi[2]) * ny + hi[1]) * nx + hi[0]];
        out[i] = r;
    }
}

__device__ __forceinline__ double axis_lo(const GridDev& g, int a) { return a == 0 ? g.ox : (a == 1 ? g.oy : g.oz); }
__device__ __forceinline__ double axis_hi(const GridDev& g, int a) { return a == 0 ? g.hx : (a == 1 ? g.hy : g.hz); }
__device__ __forceinline__ int axis_n(const GridDev& g, int a) { return a == 0 ? g.nx : (a == 1 ? g.ny : g.nz); }

// Light direction toward the source and its per-axis reciprocals (intersect_box's inv = 1 / d,
// inc/math.h:85-107, made once on the host: IEEE division gives the same value there).
struct LightDev {
    double ts[3];
    double inv[3];
};

inline LightDev light_dev(const double ts[3]) {
    LightDev l;
    for (int a = 0; a < 3; ++a) {
        l.ts[a] = ts[a];
        l.inv[a] = ts[a] != 0.0 ? 1.0 / ts[a] : 0.0;
    }
    return l;
}

// intersect_box's far-plane distance for axis a (ta, tb, swap)
__device__ __forceinline__ double face_exit(const GridDev& g, const LightDev& l, int a, double pa) {
    if (l.ts[a] == 0.0) return 1e300;
    const double ta = (axis_lo(g, a) - pa) * l.inv[a], tb = (axis_hi(g, a) - pa) * l.inv[a];
    return ta > tb ? ta : tb;
}

// Exit face of a voxel centre (intersect_box's t1 = min over the axes of the far-plane
// distances; the centre is inside, so the box is always hit): 1 = y, 2 = z, 0 = x; ties go to
// y, then z.
__device__ __forceinline__ int exit_face(double tx, double ty, double tz) {
    if (ty <= tz && ty <= tx) return 1;
    if (tz <= tx) return 2;
    return 0;
}

// n = max(1, ceil(len / step)) of the ray from p to p + ts t1 (src/volume_grid.cpp:64-72)
__device__ __forceinline__ int sample_count(const double p[3], const double ts[3], double t1, double step) {
    const double q[3] = {p[0] + ts[0] * t1, p[1] + ts[1] * t1, p[2] + ts[2] * t1};
    const double d[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
    const double len = sqrt(dot3(d, d));
    if (len == 0.0) return 0;
    const int ns = int(ceil(len / step));
    return ns < 1 ? 1 : ns;
}

// Group index layout: [E = y: ny planes][E = z: nz][E = x: nx].
__device__ __forceinline__ int group_index(const GridDev& g, int E, int c) {
    return E == 1 ? c : (E == 2 ? g.ny + c : g.ny + g.nz + c);
}

// One warp per (E, c) plane; lane j streams samples [j*chunk, (j+1)*chunk) keeping the eight
// corner weights of the current cell in registers and emitting a column (the cell's 2 x 2
// (L, O) corners of one E row) when that row leaves the cell; a move along L, or a jump of more
// than one cell, flushes both rows. Cells advance monotonically along every axis. A lane whose
// chunk ends in the cell the next lane starts in hands its pending weights over instead of
// emitting them (no duplicate columns at chunk seams). Pass 0 counts, pass 1 writes after a
// warp prefix sum.
template <typename W>
__global__ void __launch_bounds__(kTapWarps * 32) k_tap_build(GridDev g, LightDev lt, double step, int cap,
                                                               PadLayout plx, PadLayout plz,
                                                               TapGroup* __restrict__ groups,
                                                               ColTap<W>* __restrict__ taps) {
    const int gi = blockIdx.x * kTapWarps + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (gi >= g.nx + g.ny + g.nz) return;
    TapGroup& G = groups[gi];
    const int E = gi < g.ny ? 1 : (gi < g.ny + g.nz ? 2 : 0);
    const int c = gi - (E == 1 ? 0 : (E == 2 ? g.ny : g.ny + g.nz));
    const double* ts = lt.ts;
    if (ts[E] == 0.0) {
        if (lane == 0) G.n = 0;
        return;
    }
    // plane geometry: exit through E's far face, len, n, h, dir (as optical_depth computes them)
    const double pE = axis_lo(g, E) + (c + 0.5) * g.vs;
    const double texit = face_exit(g, lt, E, pE);
    double d[3] = {ts[0] * texit, ts[1] * texit, ts[2] * texit};
    const double len = sqrt(dot3(d, d));
    int ns = int(ceil(len / step));
    ns = ns < 1 ? 1 : ns;
    const double h = len / ns, il = 1.0 / len;
    const int L = E == 0 ? 2 : 0, O = 3 - E - L;
    const double dirL = d[L] * il, dirE = d[E] * il, dirO = d[O] * il;
    // cap bounds the lists of the planes a voxel can leave through (exit distance at most the
    // box's shortest span over |ts|); longer planes are never selected and get no list
    if (4 * ns + 4 * 32 + 8 > cap) {
        if (lane == 0) G.n = 0;
        return;
    }
    const PadLayout& pl = L == 0 ? plx : plz;
    const int64_t sL = pl.s[L], sE = pl.s[E], sO = pl.s[O];
    const int nE = axis_n(g, E);
    const double oE = axis_lo(g, E);
    const int tap0 = gi * cap;
    const int chunk = max(8, (ns + 31) / 32);
    const int i0 = min(ns, lane * chunk), i1 = min(ns, i0 + chunk);
    // cell of sample i: (L, E relative to c, O) and the fractions
    auto cell_of = [&](int i, int cc[3], double t[3]) {
        const double s = (i + 0.5) * h;
        double ul, uo, fe;
        const double pe = pE + dirE * s;
        if (g.ivs != 0.0) {
            ul = dirL * s * g.ivs;
            uo = dirO * s * g.ivs;
            fe = (pe - oE) * g.ivs - 0.5;
        } else {
            ul = dirL * s / g.vs;
            uo = dirO * s / g.vs;
            fe = (pe - oE) / g.vs - 0.5;
        }
        const double fl = floor(ul), fo = floor(uo), fE = floor(fe);
        cc[0] = int(fl);
        cc[1] = int(fE) - c;
        cc[2] = int(fo);
        t[0] = ul - fl;
        t[1] = fe - fE;
        t[2] = uo - fo;
    };
    // seams: does my last cell equal the next lane's first cell (and differ from my first)?
    int first[3] = {0, 0, 0}, last[3] = {0, 0, 0};
    double tt[3];
    if (i1 > i0) {
        cell_of(i0, first, tt);
        cell_of(i1 - 1, last, tt);
    }
    const int nf0 = __shfl_down_sync(0xffffffffu, first[0], 1), nf1 = __shfl_down_sync(0xffffffffu, first[1], 1),
              nf2 = __shfl_down_sync(0xffffffffu, first[2], 1);
    const int next_i0 = __shfl_down_sync(0xffffffffu, i0, 1), next_i1 = __shfl_down_sync(0xffffffffu, i1, 1);
    const bool hand_over = lane < 31 && i1 > i0 && next_i1 > next_i0 && last[0] == nf0 && last[1] == nf1 &&
                           last[2] == nf2 && !(first[0] == last[0] && first[1] == last[1] && first[2] == last[2]);
    const bool receive = __shfl_up_sync(0xffffffffu, hand_over ? 1 : 0, 1) && lane > 0;
    double acc[2][2][2];  // [bO][bE][bL]
    double fin[2][2][2] = {};  // pass 0's final cell weights (handed to the next lane in pass 1)
    int base = 0;
    for (int pass = 0; pass < 2; ++pass) {
        int cnt = 0;
        int C[3] = {first[0], first[1], first[2]};
#pragma unroll
        for (int bo = 0; bo < 2; ++bo)
#pragma unroll
            for (int be = 0; be < 2; ++be)
#pragma unroll
                for (int bl = 0; bl < 2; ++bl) {
                    const double v = __shfl_up_sync(0xffffffffu, fin[bo][be][bl], 1);
                    acc[bo][be][bl] = (pass == 1 && receive) ? v : 0.0;
                }
        auto emit = [&](int cl, int ce, int co, double w0, double w1, double w2, double w3) {
            int ae = c + ce;  // absolute E corner, clamped as sample_trilinear clamps it
            ae = ae < 0 ? 0 : (ae > nE - 1 ? nE - 1 : ae);
            if (pass == 1) {
                ColTap<W> t;
                t.w[0] = W(w0);
                t.w[1] = W(w1);
                t.w[2] = W(w2);
                t.w[3] = W(w3);
                t.lin = int(cl * sL + (ae - c) * sE + co * sO);
                taps[tap0 + base + cnt] = t;
            }
            ++cnt;
        };
        auto emit_row = [&](int be) {  // E row be of the current cell, both O rows
            emit(C[0], C[1] + be, C[2], acc[0][be][0], acc[0][be][1], acc[1][be][0], acc[1][be][1]);
            acc[0][be][0] = acc[0][be][1] = acc[1][be][0] = acc[1][be][1] = 0.0;
        };
        for (int i = i0; i < i1; ++i) {
            int cc[3];
            double t[3];
            cell_of(i, cc, t);
            if (cc[0] != C[0] || cc[1] != C[1] || cc[2] != C[2]) {
                const int dl = cc[0] - C[0], de = cc[1] - C[1], dO = cc[2] - C[2];
                if (dl != 0 || de > 1 || de < -1 || dO > 1 || dO < -1) {
                    emit_row(0);
                    emit_row(1);
                } else {
                    if (de == 1) {  // row bE = 0 leaves; bE = 1 becomes bE = 0
                        emit_row(0);
#pragma unroll
                        for (int bo = 0; bo < 2; ++bo) {
                            acc[bo][0][0] = acc[bo][1][0];
                            acc[bo][0][1] = acc[bo][1][1];
                            acc[bo][1][0] = acc[bo][1][1] = 0.0;
                        }
                    } else if (de == -1) {
                        emit_row(1);
#pragma unroll
                        for (int bo = 0; bo < 2; ++bo) {
                            acc[bo][1][0] = acc[bo][0][0];
                            acc[bo][1][1] = acc[bo][0][1];
                            acc[bo][0][0] = acc[bo][0][1] = 0.0;
                        }
                    }
                    C[1] = cc[1];
                    if (dO == 1) {  // O row bO = 0 leaves (as columns with only their low row)
#pragma unroll
                        for (int be = 0; be < 2; ++be) {
                            emit(C[0], C[1] + be, C[2], acc[0][be][0], acc[0][be][1], 0.0, 0.0);
                            acc[0][be][0] = acc[1][be][0];
                            acc[0][be][1] = acc[1][be][1];
                            acc[1][be][0] = acc[1][be][1] = 0.0;
                        }
                    } else if (dO == -1) {
#pragma unroll
                        for (int be = 0; be < 2; ++be) {
                            emit(C[0], C[1] + be, C[2] + 1, acc[1][be][0], acc[1][be][1], 0.0, 0.0);
                            acc[1][be][0] = acc[0][be][0];
                            acc[1][be][1] = acc[0][be][1];
                            acc[0][be][0] = acc[0][be][1] = 0.0;
                        }
                    }
                }
                C[0] = cc[0];
                C[1] = cc[1];
                C[2] = cc[2];
            }
            const double wl[2] = {1.0 - t[0], t[0]}, we[2] = {1.0 - t[1], t[1]}, wo[2] = {1.0 - t[2], t[2]};
#pragma unroll
            for (int bo = 0; bo < 2; ++bo)
#pragma unroll
                for (int be = 0; be < 2; ++be) {
                    acc[bo][be][0] += wo[bo] * we[be] * wl[0];
                    acc[bo][be][1] += wo[bo] * we[be] * wl[1];
                }
        }
        if (pass == 0) {
#pragma unroll
            for (int bo = 0; bo < 2; ++bo)
#pragma unroll
                for (int be = 0; be < 2; ++be)
#pragma unroll
                    for (int bl = 0; bl < 2; ++bl) fin[bo][be][bl] = acc[bo][be][bl];
        }
        if (i1 > i0 && !hand_over) {
            emit_row(0);
            emit_row(1);
        }
        int incl = cnt;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, dd);
            if (lane >= dd) incl += v;
        }
        base = incl - cnt;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (pass == 1 && lane == 0) G.n = total;
    }
    if (lane == 0) {
        G.tap0 = tap0;
        G.ns = ns;
        G.h = h;
        G.texit = texit;
    }
}

// The midpoint march of one voxel on the x-fastest padded pairs: the reference's FP64 operations
// (bit-identical values: the halo holds exactly the clamped corners). For the rare voxel whose
// sample count differs from its plane's.
template <typename Rec>
__device__ double march_padded(const GridDev& g, const Rec* __restrict__ px, const PadLayout& pl, const double p[3],
                               const double ts[3], double t1, double step) {
    const double q[3] = {p[0] + ts[0] * t1, p[1] + ts[1] * t1, p[2] + ts[2] * t1};
    const double d[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
    const double len = sqrt(dot3(d, d));
    if (len == 0.0) return 0.0;
    int ns = int(ceil(len / step));
    ns = ns < 1 ? 1 : ns;
    const double h = len / ns, il = 1.0 / len;
    const double dir[3] = {d[0] * il, d[1] * il, d[2] * il};
    double sum = 0.0;
    for (int i = 0; i < ns; ++i) {
        const double s = (i + 0.5) * h;
        double f[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double pa = p[a] + dir[a] * s;
            f[a] = g.ivs != 0.0 ? (pa - axis_lo(g, a)) * g.ivs - 0.5 : (pa - axis_lo(g, a)) / g.vs - 0.5;
        }
        const double fl[3] = {floor(f[0]), floor(f[1]), floor(f[2])};
        const double tx = f[0] - fl[0], ty = f[1] - fl[1], tz = f[2] - fl[2];
        const Rec* row =
            px + (int64_t(fl[0]) + 1) * pl.s[0] + (int64_t(fl[1]) + 1) * pl.s[1] + (int64_t(fl[2]) + 1) * pl.s[2];
        const Rec r00 = __ldg(row), r10 = __ldg(row + pl.s[1]);
        const Rec r01 = __ldg(row + pl.s[2]), r11 = __ldg(row + pl.s[2] + pl.s[1]);
        const double c00 = lerp1(r00.x, r00.y, tx), c10 = lerp1(r10.x, r10.y, tx);
        const double c01 = lerp1(r01.x, r01.y, tx), c11 = lerp1(r11.x, r11.y, tx);
        sum += lerp1(lerp1(c00, c10, ty), lerp1(c01, c11, ty), tz);
    }
    return sum * h;
}

// The voxels leaving through face E. A block takes 32 L-consecutive x K O-consecutive voxels on
// 8 consecutive E planes, one plane per warp: the rays of neighbouring planes are the same ray
// shifted by one voxel along E, so the warps (kept in step by the tile barriers) read the same
// record rows a tap or two apart and the block's L1 serves most of them. Each warp's tap list
// is staged through shared memory in tiles. Voxel rows z are restricted to [zlo, zhi) (a
// z-slab when the build is sharded over GPUs). Rows no owned voxel needs are redirected to a
// row that one does (no predicates in the tap loop; their sums are discarded).
constexpr int kColTile = 64;   // taps per warp per tile
constexpr int kColPlanes = 8;  // E planes (warps) per block

#ifndef SF_GRADED_MINB
#define SF_GRADED_MINB 3
#endif
template <typename W, typename Rec, int E>
__global__ void __launch_bounds__(256, SF_GRADED_MINB) k_graded_cols(GridDev g, const Rec* __restrict__ rec, PadLayout pl,
                                                        const Rec* __restrict__ recx, PadLayout plx, LightDev lt,
                                                        double coeff, double step, int zlo,
                                                        int zhi, const TapGroup* __restrict__ groups,
                                                        const ColTap<W>* __restrict__ taps, float* __restrict__ out) {
    constexpr int L = E == 0 ? 2 : 0, O = 3 - E - L, K = kColK;
    __shared__ ColTap<W> tile[kColPlanes][kColTile];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lo[3] = {0, 0, zlo}, hi[3] = {g.nx, g.ny, zhi};
    // block order: L chunk, then E plane group, then O block, so the blocks in flight cover a thin
    // O slab of the volume (their rays overlap; a small L2 working set)
    const int nch = (hi[L] - lo[L] + 31) / 32, neb = (hi[E] - lo[E] + kColPlanes - 1) / kColPlanes;
    const int ch = int(blockIdx.x % unsigned(nch));
    const int eb = int((blockIdx.x / unsigned(nch)) % unsigned(neb));
    const int ob = int(blockIdx.x / (unsigned(nch) * neb));
    const int e = lo[E] + eb * kColPlanes + warp;
    int v[3] = {0, 0, 0};
    v[L] = lo[L] + ch * 32 + lane;
    v[E] = e;
    const int o0 = lo[O] + ob * K;
    const double* ts = lt.ts;
    const bool lane_in = e < hi[E] && v[L] < hi[L];
    double p[3];
    p[L] = axis_lo(g, L) + (v[L] + 0.5) * g.vs;
    p[E] = axis_lo(g, E) + (v[E] + 0.5) * g.vs;
    const double tE = face_exit(g, lt, E, p[E]), tL = face_exit(g, lt, L, p[L]);
    TapGroup G;
    G.n = 0;
    G.tap0 = 0;
    G.ns = 0;
    G.h = 0.0;
    G.texit = 0.0;
    if (e < hi[E]) G = groups[group_index(g, E, e)];
    bool own[K], ok[K];
    bool any_own = false, any_ok = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int o = o0 + j;
        p[O] = axis_lo(g, O) + (o + 0.5) * g.vs;
        const double tO = face_exit(g, lt, O, p[O]);
        double t3[3];
        t3[L] = tL;
        t3[E] = tE;
        t3[O] = tO;
        own[j] = lane_in && o < hi[O] && exit_face(t3[0], t3[1], t3[2]) == E;
        ok[j] = own[j] && G.n > 0 && tE == G.texit && sample_count(p, ts, tE, step) == G.ns;
        any_own |= own[j];
        any_ok |= ok[j];
    }
    W acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = W(0);
    const int block_taps = __syncthreads_or(any_ok) ? 1 : 0;
    if (block_taps) {
        // row j's gather serves voxel j (low O row) and voxel j - 1 (high O row); rows no ok voxel
        // uses point at a row some ok voxel of the warp uses, so every gather stays in bounds
        const unsigned okmask = __ballot_sync(0xffffffffu, any_ok);
        const bool warp_taps = okmask != 0u;
        int vb[3] = {v[0], v[1], v[2]};
        vb[O] = o0;
        const int64_t base = (vb[0] + 1) * pl.s[0] + (vb[1] + 1) * pl.s[1] + (vb[2] + 1) * pl.s[2];
        int jfirst = K;
#pragma unroll
        for (int j = K; j >= 0; --j)
            if ((j < K && ok[j]) || (j > 0 && ok[j - 1])) jfirst = j;
        const int src = warp_taps ? __ffs(okmask) - 1 : 0;
        // 32-bit element offsets (a padded level has < 2^31 records): one add + one wide multiply-add
        // per gather
        const unsigned fallback = unsigned(__shfl_sync(0xffffffffu, base + int64_t(jfirst) * pl.s[O], src));
        unsigned rowo[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) {
            const bool need = (j < K && ok[j]) || (j > 0 && ok[j - 1]);
            rowo[j] = need ? unsigned(base + int64_t(j) * pl.s[O]) : fallback;
        }
        const ColTap<W>* tp = taps + G.tap0;
        const int n = G.n > 0 ? G.n : 0;
        int max_n = n;
        // block-wide tile rounds: the longest list of the block's planes
        {
            __shared__ int smax;
            if (threadIdx.x == 0) smax = 0;
            __syncthreads();
            if (lane == 0) atomicMax(&smax, n);
            __syncthreads();
            max_n = smax;
        }
        for (int t0 = 0; t0 < max_n; t0 += kColTile) {
            const int nt = max(0, min(kColTile, n - t0));
            __syncwarp();
            for (int i = lane; i < nt; i += 32) tile[warp][i] = tp[t0 + i];
            __syncthreads();
            if (warp_taps) {
                constexpr int U = (sizeof(W) == 4 && kColK <= 4) ? 2 : 1;  // taps in flight (registers)
                int k = 0;
                for (; k + U <= nt; k += U) {
                    ColTap<W> t[U];
                    Rec r[U][K + 1];
#pragma unroll
                    for (int u = 0; u < U; ++u) t[u] = tile[warp][k + u];
#pragma unroll
                    for (int j = 0; j <= K; ++j)
#pragma unroll
                        for (int u = 0; u < U; ++u) r[u][j] = __ldg(rec + (rowo[j] + unsigned(t[u].lin)));
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        W a = acc[j];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            a = fma(t[u].w[0], W(r[u][j].x), a);
                            a = fma(t[u].w[1], W(r[u][j].y), a);
                            a = fma(t[u].w[2], W(r[u][j + 1].x), a);
                            a = fma(t[u].w[3], W(r[u][j + 1].y), a);
                        }
                        acc[j] = a;
                    }
                }
                for (; k < nt; ++k) {
                    const ColTap<W> ta = tile[warp][k];
                    Rec ra[K + 1];
#pragma unroll
                    for (int j = 0; j <= K; ++j) ra[j] = __ldg(rec + (rowo[j] + unsigned(ta.lin)));
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        W a = acc[j];
                        a = fma(ta.w[0], W(ra[j].x), a);
                        a = fma(ta.w[1], W(ra[j].y), a);
                        a = fma(ta.w[2], W(ra[j + 1].x), a);
                        a = fma(ta.w[3], W(ra[j + 1].y), a);
                        acc[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (!any_own) return;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (!own[j]) continue;
        v[O] = o0 + j;
        p[O] = axis_lo(g, O) + (v[O] + 0.5) * g.vs;
        const double tau = ok[j] ? double(acc[j]) * G.h : march_padded<Rec>(g, recx, plx, p, ts, tE, step);
        out[(size_t(v[2]) * g.ny + v[1]) * g.nx + v[0]] = float(exp(-coeff * tau));
    }
}

struct Kernel27 {
    float k[27];
};

// K3a: conv3_replicate (src/feature_pipeline.cpp:70-92); FP64 accumulation in
// tap order dz, dy, dx.
// kFast (production build): the same taps in the same order accumulated in FP32 (fmaf).
template <bool kFast>
__global__ void k_conv3(const float* __restrict__ in, int nx, int ny, int nz, Kernel27 k, int zlo, int zhi,
                        float* __restrict__ out) {
    const size_t n = size_t(nx) * ny * zhi;
    for (size_t idx = size_t(nx) * ny * zlo + blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < n;
         idx += size_t(gridDim.x) * blockDim.x) {
        int x = int(idx % nx);
        int y = int((idx / nx) % ny);
        int z = int(idx / (size_t(nx) * ny));
        double acc = 0.0;
        float accf = 0.0f;
        int t = 0;
#pragma unroll
        for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx, ++t) {
                    int sx = clampi(x + dx, 0, nx - 1);
                    int sy = clampi(y + dy, 0, ny - 1);
                    int sz = clampi(z + dz, 0, nz - 1);
                    if (kFast)
                        accf = fmaf(k.k[t], __ldg(in + (size_t(sz) * ny + sy) * nx + sx), accf);
                    else
                        acc += double(k.k[t]) * in[(size_t(sz) * ny + sy) * nx + sx];
                }
        out[idx] = kFast ? accf : float(acc);
    }
}

constexpr int kMaxLevels = 24;
struct Levels {
    int n;
    GridDev g[kMaxLevels];
    double scale[kMaxLevels];
};

// K3b: combine_transmittance (src/feature_pipeline.cpp:94-128): for every
// level-0 voxel centre, FP64 trilinear of each convolved level, scaled, then
// accumulated in float in level order. One pass over all levels per voxel keeps
// the float accumulation order of the reference while writing the output once.
// kFast (production build): the level-0 term is the convolved value at the voxel itself (the
// trilinear at a voxel's own centre has zero weights), coarser levels are interpolated in FP32,
// and the box test is left out (level-0 centres lie inside every level's box).
__device__ __forceinline__ float trilinear_f32(const GridDev& g, float fx, float fy, float fz) {
    const float flx = floorf(fx), fly = floorf(fy), flz = floorf(fz);
    const int x0 = int(flx), y0 = int(fly), z0 = int(flz);
    float tx = fx - flx, ty = fy - fly, tz = fz - flz;
    const int xa = max(x0, 0), xb = min(x0 + 1, g.nx - 1), ya = max(y0, 0), yb = min(y0 + 1, g.ny - 1);
    const int za = max(z0, 0), zb = min(z0 + 1, g.nz - 1);
    const float* v = g.v;
    const int sy = g.nx, sz = g.nx * g.ny;
    const float c00 = fmaf(tx, __ldg(v + za * sz + ya * sy + xb) - __ldg(v + za * sz + ya * sy + xa),
                           __ldg(v + za * sz + ya * sy + xa));
    const float c10 = fmaf(tx, __ldg(v + za * sz + yb * sy + xb) - __ldg(v + za * sz + yb * sy + xa),
                           __ldg(v + za * sz + yb * sy + xa));
    const float c01 = fmaf(tx, __ldg(v + zb * sz + ya * sy + xb) - __ldg(v + zb * sz + ya * sy + xa),
                           __ldg(v + zb * sz + ya * sy + xa));
    const float c11 = fmaf(tx, __ldg(v + zb * sz + yb * sy + xb) - __ldg(v + zb * sz + yb * sy + xa),
                           __ldg(v + zb * sz + yb * sy + xa));
    const float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
    return fmaf(tz, e1 - e0, e0);
}

template <bool kFast>
__global__ void k_combine(Levels lv, GridDev base, int zlo, int zhi, float* __restrict__ out) {
    const size_t off = size_t(base.nx) * base.ny * zlo;
    const size_t n = size_t(base.nx) * base.ny * zhi;
    for (size_t idx = off + blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < n;
         idx += size_t(gridDim.x) * blockDim.x) {
        int x = int(idx % base.nx);
        int y = int((idx / base.nx) % base.ny);
        int z = int(idx / (size_t(base.nx) * base.ny));
        if (kFast) {
            // level li's voxel coordinate of this centre: (x + 0.5) / 2^li - 0.5 (exact in float)
            float acc = float(lv.scale[0] * double(__ldg(lv.g[0].v + idx)));
            float inv = 1.0f;
            for (int li = 1; li < lv.n; ++li) {
                inv *= 0.5f;
                const float v = trilinear_f32(lv.g[li], (float(x) + 0.5f) * inv - 0.5f, (float(y) + 0.5f) * inv - 0.5f,
                                              (float(z) + 0.5f) * inv - 0.5f);
                acc += float(lv.scale[li]) * v;
            }
            out[idx - off] = acc;
        } else {
            double c[3] = {base.ox + (x + 0.5) * base.vs, base.oy + (y + 0.5) * base.vs,
                           base.oz + (z + 0.5) * base.vs};
            float acc = 0.0f;
            for (int li = 0; li < lv.n; ++li) {
                double v = trilinear(lv.g[li], c[0], c[1], c[2]);
                acc += float(lv.scale[li] * v);
            }
            out[idx - off] = acc;
        }
    }
}

// K3a production form: the same 27 taps in the same order with FP32 fmaf (bit-identical to
// k_conv3<true>), one thread per (x, y) column walking kConvZ rows of z with the 3 x 3 neighbourhoods
// of planes z - 1, z, z + 1 held in registers: 9 loads per output instead of 27.
constexpr int kConvZ = 16;

__global__ void __launch_bounds__(256) k_conv3_zwin(const float* __restrict__ in, int nx, int ny, int nz, Kernel27 k,
                                                    int zlo, int zhi, float* __restrict__ out) {
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    const int z0 = zlo + blockIdx.z * kConvZ, z1 = min(z0 + kConvZ, zhi);
    if (x >= nx || y >= ny) return;
    const int xs[3] = {max(x - 1, 0), x, min(x + 1, nx - 1)};
    const int ys[3] = {max(y - 1, 0), y, min(y + 1, ny - 1)};
    float w[3][3][3];  // [plane z-1, z, z+1][dy][dx]
    auto load = [&](int zz, float (&pl)[3][3]) {
        const int zc = zz < 0 ? 0 : (zz > nz - 1 ? nz - 1 : zz);
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) pl[dy][dx] = __ldg(in + (size_t(zc) * ny + ys[dy]) * nx + xs[dx]);
    };
    load(z0 - 1, w[0]);
    load(z0, w[1]);
    for (int z = z0; z < z1; ++z) {
        load(z + 1, w[2]);
        float acc = 0.0f;
        int t = 0;
#pragma unroll
        for (int dz = 0; dz < 3; ++dz)
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int dx = 0; dx < 3; ++dx, ++t) acc = fmaf(k.k[t], w[dz][dy][dx], acc);
        out[(size_t(z) * ny + y) * nx + x] = acc;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                w[0][dy][dx] = w[1][dy][dx];
                w[1][dy][dx] = w[2][dy][dx];
            }
    }
}

// K3b production form: one thread per 2 x 2 x 2 block of level-0 voxels. For every coarser level
// the block's eight trilinear cells lie in one 3 x 3 x 3 neighbourhood of that level (the two
// fine centres of an axis fall in the same or in adjacent coarse cells), loaded once: 27 loads
// per level for eight voxels instead of 64. Each voxel's lerps are the FP32 operations of
// k_combine<true> in the same order (bit-identical).
#ifndef SF_COMBINE_MINB
#define SF_COMBINE_MINB 1
#endif
__global__ void __launch_bounds__(256, SF_COMBINE_MINB) k_combine_blk(Levels lv, GridDev base, int zlo, int zhi,
                                                     float* __restrict__ out) {
    const int bx = blockIdx.x * 32 + threadIdx.x, by = blockIdx.y * 8 + threadIdx.y;
    const int x0 = 2 * bx, y0 = 2 * by, z0 = zlo + 2 * int(blockIdx.z);
    if (x0 >= base.nx || y0 >= base.ny || z0 >= zhi) return;
    const int c0[3] = {x0, y0, z0};
    const int lim[3] = {base.nx, base.ny, zhi};
    float acc[2][2][2];  // [z][y][x]
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int x = min(x0 + k, base.nx - 1), y = min(y0 + j, base.ny - 1), z = min(z0 + i, zhi - 1);
                acc[i][j][k] = float(lv.scale[0] * double(__ldg(lv.g[0].v + (size_t(z) * base.ny + y) * base.nx + x)));
            }
    float inv = 1.0f;
    for (int li = 1; li < lv.n; ++li) {
        inv *= 0.5f;
        const GridDev& g = lv.g[li];
        const int n[3] = {g.nx, g.ny, g.nz};
        int idx[3][3];       // clamped coarse indices b, b + 1, b + 2 per axis
        float t[3][2];       // fractions of the two fine centres
        int sel[3];          // 1: the high fine centre's cell starts at b + 1
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float flo = (float(c0[a]) + 0.5f) * inv - 0.5f, fhi = (float(c0[a] + 1) + 0.5f) * inv - 0.5f;
            const float llo = floorf(flo), lhi = floorf(fhi);
            const int b = int(llo);
            t[a][0] = flo - llo;
            t[a][1] = fhi - lhi;
            sel[a] = int(lhi) - b;
#pragma unroll
            for (int q = 0; q < 3; ++q) idx[a][q] = max(0, min(b + q, n[a] - 1));
        }
        float V[3][3][3];  // [z][y][x]
#pragma unroll
        for (int qz = 0; qz < 3; ++qz)
#pragma unroll
            for (int qy = 0; qy < 3; ++qy)
#pragma unroll
                for (int qx = 0; qx < 3; ++qx)
                    V[qz][qy][qx] = __ldg(g.v + (size_t(idx[2][qz]) * g.ny + idx[1][qy]) * g.nx + idx[0][qx]);
        // x lerps of every (y', z') row for the low / high fine x
        float cx[2][3][3];  // [fine x][z'][y']
#pragma unroll
        for (int qz = 0; qz < 3; ++qz)
#pragma unroll
            for (int qy = 0; qy < 3; ++qy) {
                const float* r = V[qz][qy];
                cx[0][qz][qy] = fmaf(t[0][0], r[1] - r[0], r[0]);
                cx[1][qz][qy] = sel[0] ? fmaf(t[0][1], r[2] - r[1], r[1]) : fmaf(t[0][1], r[1] - r[0], r[0]);
            }
        const float sc = float(lv.scale[li]);
#pragma unroll
        for (int fz = 0; fz < 2; ++fz)
#pragma unroll
            for (int fy = 0; fy < 2; ++fy)
#pragma unroll
                for (int fx = 0; fx < 2; ++fx) {
                    const int oy = fy ? sel[1] : 0, oz = fz ? sel[2] : 0;
                    const float ty = t[1][fy], tz = t[2][fz];
                    // rows (y0, z0), (y1, z0), (y0, z1), (y1, z1) of this voxel's cell
                    const float c00 = oy ? (oz ? cx[fx][1][1] : cx[fx][0][1]) : (oz ? cx[fx][1][0] : cx[fx][0][0]);
                    const float c10 = oy ? (oz ? cx[fx][1][2] : cx[fx][0][2]) : (oz ? cx[fx][1][1] : cx[fx][0][1]);
                    const float c01 = oy ? (oz ? cx[fx][2][1] : cx[fx][1][1]) : (oz ? cx[fx][2][0] : cx[fx][1][0]);
                    const float c11 = oy ? (oz ? cx[fx][2][2] : cx[fx][1][2]) : (oz ? cx[fx][2][1] : cx[fx][1][1]);
                    const float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
                    acc[fz][fy][fx] += sc * fmaf(tz, e1 - e0, e0);
                }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int x = x0 + k, y = y0 + j, z = z0 + i;
                if (x < lim[0] && y < lim[1] && z < lim[2]) out[(size_t(z - zlo) * base.ny + y) * base.nx + x] = acc[i][j][k];
            }
}

__global__ void k_interleave(const float* __restrict__ a, const float* __restrict__ b,
                             float2* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = make_float2(a[i], b[i]);
}

constexpr int kMaxNodes = 64;
struct GLNodes {
    int n;
    double x[kMaxNodes];
    double w[kMaxNodes];
};

__device__ __forceinline__ double hg_phase(double g, double c) {
    double denom = 1.0 + g * g - 2.0 * g * c;
    denom = (denom < 1e-12) ? 1e-12 : denom;
    return kInv4Pi * (1.0 - g * g) / (denom * sqrt(denom));
}

// K4: PhaseTable build (src/phase.cpp:159-177 -> cap_integral :124-145), one
// thread per (g, angle, aperture) cell; 2*nodes azimuths x nodes polar nodes.
__global__ void k_phase_table(int gr, int ar, int hr, GLNodes gl, float* __restrict__ out) {
    int n = gr * ar * hr;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
        int hi = idx % hr;
        int ai = (idx / hr) % ar;
        int gi = idx / (hr * ar);
        double g = -0.99 + 1.98 * gi / double(gr - 1);
        double angle = kPi * ai / double(ar - 1);
        double cf = cos(angle);
        double half = kPi * hi / double(hr - 1);
        double v = 0.0;
        if (half > 0.0) {
            double mu_lo = cos((kPi < half) ? kPi : half);
            int n_psi = 2 * gl.n;
            double sf = 1.0 - cf * cf;
            double s_f = sqrt((0.0 < sf) ? sf : 0.0);
            double sum = 0.0;
            for (int i = 0; i < gl.n; ++i) {
                double mu = 0.5 * (1.0 + mu_lo) + 0.5 * (1.0 - mu_lo) * gl.x[i];
                double w_mu = 0.5 * (1.0 - mu_lo) * gl.w[i];
                double sm = 1.0 - mu * mu;
                double s_mu = sqrt((0.0 < sm) ? sm : 0.0);
                double inner = 0.0;
                for (int j = 0; j < n_psi; ++j) {
                    double psi = 2.0 * kPi * (j + 0.5) / n_psi;
                    double cg = clampd(cf * mu + s_f * s_mu * cos(psi), -1.0, 1.0);
                    inner += 0.0 + 1.0 * hg_phase(g, cg);
                }
                sum += w_mu * inner * (2.0 * kPi / n_psi);
            }
            v = sum;
        }
        out[idx] = float(v);
    }
}

__global__ void k_lookup_hg(const float* __restrict__ T, int gr, int ar, int hr, int64_t n,
                            const double* __restrict__ g, const double* __restrict__ a,
                            const double* __restrict__ h, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = lookup_hg(T, gr, ar, hr, g[i], a[i], h[i]);
}

__global__ void k_sample_trilinear(GridDev g, int64_t n, const double* __restrict__ pts,
                                   double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = trilinear(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

}  // namespace

void launch_pyramid_down(const sf_grid& src, sf_grid& dst, cudaStream_t s) {
    k_pyramid_down<<<grid_for(dst.count()), kBlock, 0, s>>>(src.d, src.nx, src.ny, src.nz, dst.d,
                                                           dst.nx, dst.ny, dst.nz);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

namespace {
// K2 through the shared tap lists: padded pair records of the level (x-fastest, and z-fastest
// when some rays leave through an x face), k_tap_build for every plane, then one
// k_graded_cols pass per exit face over voxel rows [zlo, zhi).
// The level's padded records of one layout: from the pyramid's cache (made on first use), else
// stream-ordered scratch that the caller frees.
template <typename Rec>
Rec* padded_records(const sf_grid& level, const PadLayout& pl, PadCache* cache, cudaStream_t s, bool& scratch) {
    const int prec = sizeof(Rec) == sizeof(double2) ? 1 : 0, lay = pl.L == 0 ? 0 : 1;
    auto fill = [&](Rec* r) {
        k_pad_pairs<Rec><<<grid_for(size_t(pl.count)), kBlock, 0, s>>>(level.d, level.nx, level.ny, level.nz, pl, r);
        SFB_CUDA(cudaGetLastError());
        count_launch();
    };
    if (!cache) {
        Rec* r = nullptr;
        SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&r), size_t(pl.count) * sizeof(Rec), s));
        fill(r);
        scratch = true;
        return r;
    }
    std::lock_guard<std::mutex> lk(cache->mu);
    scratch = false;
    if (!cache->rec[prec][lay]) {
        void* r = nullptr;
        SFB_CUDA(cudaMalloc(&r, size_t(pl.count) * sizeof(Rec)));
        cudaEvent_t ev = nullptr;
        const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            cudaFree(r);
            cuda_check(e, "cudaEventCreate");
        }
        cache->rec[prec][lay] = r;
        cache->ready[prec][lay] = ev;
        fill(static_cast<Rec*>(r));
        SFB_CUDA(cudaEventRecord(ev, s));
    } else {
        SFB_CUDA(cudaStreamWaitEvent(s, cache->ready[prec][lay], 0));
    }
    return static_cast<Rec*>(cache->rec[prec][lay]);
}

template <typename W, typename Rec>
void graded_taps(const sf_grid& level, const double ts[3], double coeff, double step, int zlo, int zhi, float* out,
                 cudaStream_t s, PadCache* cache) {
    const GridDev g = level.dev();
    // a voxel's exit distance is at most the box's shortest span over |ts_a|: it bounds the
    // sample count of every plane some voxel selects
    double T = 1e300;
    for (int a = 0; a < 3; ++a)
        if (ts[a] != 0.0) {
            const double lo = a == 0 ? g.ox : (a == 1 ? g.oy : g.oz), hi = a == 0 ? g.hx : (a == 1 ? g.hy : g.hz);
            T = std::min(T, (hi - lo) / std::fabs(ts[a]));
        }
    const int ns_max = int(std::ceil(T / step)) + 3;
    const int cap = 4 * ns_max + 4 * 32 + 16;
    const int n_groups = g.nx + g.ny + g.nz;
    const PadLayout plx = pad_layout(g.nx, g.ny, g.nz, 0), plz = pad_layout(g.nx, g.ny, g.nz, 2);
    const bool face_x = ts[0] != 0.0;
    TapGroup* groups = nullptr;
    ColTap<W>* taps = nullptr;
    Rec *px = nullptr, *pz = nullptr;
    bool px_scratch = false, pz_scratch = false;
    SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&groups), size_t(n_groups) * sizeof(TapGroup), s));
    SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&taps), size_t(n_groups) * cap * sizeof(ColTap<W>), s));
    px = padded_records<Rec>(level, plx, cache, s, px_scratch);
    if (face_x) pz = padded_records<Rec>(level, plz, cache, s, pz_scratch);
    const LightDev lt = light_dev(ts);
    k_tap_build<W><<<(n_groups + kTapWarps - 1) / kTapWarps, kTapWarps * 32, 0, s>>>(g, lt, step, cap, plx, plz, groups,
                                                                                     taps);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    const int lo[3] = {0, 0, zlo}, hi[3] = {g.nx, g.ny, zhi};
    auto blocks = [&](int E) {  // L chunks x groups of kColPlanes E planes x O blocks
        const int L = E == 0 ? 2 : 0, O = 3 - E - L;
        const int64_t tiles = int64_t((hi[L] - lo[L] + 31) / 32) * ((hi[O] - lo[O] + kColK - 1) / kColK);
        return unsigned(tiles * ((hi[E] - lo[E] + kColPlanes - 1) / kColPlanes));
    };
    if (ts[1] != 0.0) {
        k_graded_cols<W, Rec, 1><<<blocks(1), 256, 0, s>>>(
            g, px, plx, px, plx, lt, coeff, step, zlo, zhi, groups, taps, out);
        SFB_CUDA(cudaGetLastError());
        count_launch();
    }
    if (ts[2] != 0.0) {
        k_graded_cols<W, Rec, 2><<<blocks(2), 256, 0, s>>>(
            g, px, plx, px, plx, lt, coeff, step, zlo, zhi, groups, taps, out);
        SFB_CUDA(cudaGetLastError());
        count_launch();
    }
    if (face_x) {
        k_graded_cols<W, Rec, 0><<<blocks(0), 256, 0, s>>>(
            g, pz, plz, px, plx, lt, coeff, step, zlo, zhi, groups, taps, out);
        SFB_CUDA(cudaGetLastError());
        count_launch();
    }
    if (pz && pz_scratch) SFB_CUDA(cudaFreeAsync(pz, s));
    if (px_scratch) SFB_CUDA(cudaFreeAsync(px, s));
    SFB_CUDA(cudaFreeAsync(taps, s));
    SFB_CUDA(cudaFreeAsync(groups, s));
}

bool use_taps(const double ts[3]) {
    static const int mode = std::getenv("SF_GRADED") ? std::atoi(std::getenv("SF_GRADED")) : 1;  // 0: march
    (void)ts;
    return mode != 0;
}
}  // namespace

void launch_graded(const sf_grid& level, const double ts[3], double coeff, double step, int zlo, int zhi,
                   float* out, cudaStream_t s, bool fast, PadCache* cache) {
    if (zhi <= zlo) return;
    // the tap kernels address records with 32-bit element offsets
    const bool fits = pad_layout(level.nx, level.ny, level.nz, 0).count < (int64_t(1) << 31) &&
                      pad_layout(level.nx, level.ny, level.nz, 2).count < (int64_t(1) << 31);
    if (use_taps(ts) && fits) {
        if (fast)
            graded_taps<float, float2>(level, ts, coeff, step, zlo, zhi, out, s, cache);
        else
            graded_taps<double, double2>(level, ts, coeff, step, zlo, zhi, out, s, cache);
        return;
    }
    const size_t rows = size_t(level.nx) * level.ny * size_t(zhi - zlo);
    if (fast) {
        float2* xp = nullptr;
        SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xp), level.count() * sizeof(float2), s));
        k_xpair_f32<<<grid_for(level.count()), kBlock, 0, s>>>(level.d, level.nx, level.ny, level.nz, xp);
        SFB_CUDA(cudaGetLastError());
        count_launch();
        k_graded_f32<<<grid_for(rows, 128), 128, 0, s>>>(level.dev(), xp, ts[0], ts[1], ts[2], coeff, step, zlo, zhi,
                                                         out);
        SFB_CUDA(cudaGetLastError());
        count_launch();
        SFB_CUDA(cudaFreeAsync(xp, s));
        return;
    }
    double2* xp = nullptr;
    SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xp), level.count() * sizeof(double2), s));
    k_xpair_f64<<<grid_for(level.count()), kBlock, 0, s>>>(level.d, level.nx, level.ny, level.nz, xp);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    k_graded<<<grid_for(rows, 128), 128, 0, s>>>(level.dev(), xp, ts[0], ts[1], ts[2], coeff, step, zlo, zhi, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    SFB_CUDA(cudaFreeAsync(xp, s));
}

void launch_conv3(const sf_grid& in, const float k27[27], int zlo, int zhi, float* out, cudaStream_t s, bool fast) {
    if (zhi <= zlo) return;
    Kernel27 k;
    for (int i = 0; i < 27; ++i) k.k[i] = k27[i];
    static const bool v1 = std::getenv("SF_BUILD_V1") != nullptr;  // A/B: the one-thread-per-voxel kernel
    if (fast && !v1) {
        const dim3 grid((in.nx + 31) / 32, (in.ny + 7) / 8, (zhi - zlo + kConvZ - 1) / kConvZ);
        k_conv3_zwin<<<grid, dim3(32, 8), 0, s>>>(in.d, in.nx, in.ny, in.nz, k, zlo, zhi, out);
    } else {
        (fast ? k_conv3<true> : k_conv3<false>)<<<grid_for(size_t(in.nx) * in.ny * size_t(zhi - zlo)), kBlock, 0,
                                                   s>>>(in.d, in.nx, in.ny, in.nz, k, zlo, zhi, out);
    }
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_combine(const std::vector<const sf_grid*>& conv, const std::vector<float>& scales,
                    const sf_grid& base, int zlo, int zhi, float* out, cudaStream_t s, bool fast) {
    if (zhi <= zlo) return;
    if (conv.size() > size_t(kMaxLevels)) fail(SF_ERR_INVALID_ARGUMENT, "combine: too many levels");
    Levels lv{};
    lv.n = int(conv.size());
    for (int i = 0; i < lv.n; ++i) {
        lv.g[i] = conv[size_t(i)]->dev();
        lv.scale[i] = double(scales[size_t(i)]);
    }
    // the fast form needs every level to halve the previous one exactly (pyramid levels do,
    // down to 1 voxel; an odd size falls back to the FP64 form)
    bool halving = fast;
    for (int i = 1; i < lv.n && halving; ++i) {
        const sf_grid& a = *conv[size_t(i - 1)];
        const sf_grid& b = *conv[size_t(i)];
        halving = (a.nx == 2 * b.nx || (a.nx == 1 && b.nx == 1)) && (a.ny == 2 * b.ny || (a.ny == 1 && b.ny == 1)) &&
                  (a.nz == 2 * b.nz || (a.nz == 1 && b.nz == 1)) && b.vs == 2.0 * a.vs &&
                  b.origin[0] == a.origin[0] && b.origin[1] == a.origin[1] && b.origin[2] == a.origin[2];
    }
    static const bool v1 = std::getenv("SF_BUILD_V1") != nullptr;
    if (halving && !v1) {
        const dim3 grid(((base.nx + 1) / 2 + 31) / 32, ((base.ny + 1) / 2 + 7) / 8, (zhi - zlo + 1) / 2);
        k_combine_blk<<<grid, dim3(32, 8), 0, s>>>(lv, base.dev(), zlo, zhi, out);
    } else {
        (halving ? k_combine<true> : k_combine<false>)<<<grid_for(size_t(base.nx) * base.ny * size_t(zhi - zlo)),
                                                          kBlock, 0, s>>>(lv, base.dev(), zlo, zhi, out);
    }
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_interleave(const float* a, const float* b, float2* out, size_t n, cudaStream_t s) {
    k_interleave<<<grid_for(n), kBlock, 0, s>>>(a, b, out, n);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_phase_table(int gr, int ar, int hr, const std::vector<double>& nodes,
                        const std::vector<double>& weights, float* out, cudaStream_t s) {
    if (nodes.size() > size_t(kMaxNodes)) fail(SF_ERR_INVALID_ARGUMENT, "phase table: too many nodes");
    GLNodes gl{};
    gl.n = int(nodes.size());
    for (int i = 0; i < gl.n; ++i) {
        gl.x[i] = nodes[size_t(i)];
        gl.w[i] = weights[size_t(i)];
    }
    k_phase_table<<<grid_for(size_t(gr) * ar * hr, 128), 128, 0, s>>>(gr, ar, hr, gl, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_lookup_hg(const sf_phase_table& t, int64_t n, const double* g, const double* a,
                      const double* h, double* out, cudaStream_t s) {
    k_lookup_hg<<<grid_for(size_t(n)), kBlock, 0, s>>>(t.d, t.g, t.a, t.h, n, g, a, h, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_sample_trilinear(const sf_grid& g, int64_t n, const double* pts, double* out,
                             cudaStream_t s) {
    k_sample_trilinear<<<grid_for(size_t(n)), kBlock, 0, s>>>(g.dev(), n, pts, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
