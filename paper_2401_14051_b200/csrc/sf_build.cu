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

// K2: graded transmittance of one level (src/feature_pipeline.cpp:37-68) with the
// midpoint-rule optical depth (src/volume_grid.cpp:64-78), for voxel rows z in [zlo, zhi)
// (a z-slab when the build is sharded over GPUs). One thread per voxel; neighbouring
// threads march neighbouring parallel rays, so a warp's gathers stay within a few lines.
// FP64 throughout, as the reference: the kernel is FP64-pipe bound.
__global__ void k_graded(GridDev g, const double2* __restrict__ xp, double tsx, double tsy, double tsz,
                         double coeff, double step, int zlo, int zhi, float* __restrict__ out) {
    const int plane = g.nx * g.ny;
    const int i0 = zlo * plane, i1 = zhi * plane;
    const double lo[3] = {g.ox, g.oy, g.oz};
    const double hi[3] = {g.hx, g.hy, g.hz};
    const double ts[3] = {tsx, tsy, tsz};
    for (int idx = i0 + blockIdx.x * blockDim.x + threadIdx.x; idx < i1; idx += gridDim.x * blockDim.x) {
        const int x = idx % g.nx;
        const int y = (idx / g.nx) % g.ny;
        const int z = idx / plane;
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
        out[idx] = float(exp(-coeff * tau));
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

__global__ void k_graded_f32(GridDev g, const float2* __restrict__ xp, double tsx, double tsy, double tsz,
                             double coeff, double step, int zlo, int zhi, float* __restrict__ out) {
    const int plane = g.nx * g.ny;
    const int i0 = zlo * plane, i1 = zhi * plane;
    const double lo[3] = {g.ox, g.oy, g.oz};
    const double hi[3] = {g.hx, g.hy, g.hz};
    const double ts[3] = {tsx, tsy, tsz};
    for (int idx = i0 + blockIdx.x * blockDim.x + threadIdx.x; idx < i1; idx += gridDim.x * blockDim.x) {
        const int x = idx % g.nx;
        const int y = (idx / g.nx) % g.ny;
        const int z = idx / plane;
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
        out[idx] = float(exp(-coeff * tau));
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

void launch_graded(const sf_grid& level, const double ts[3], double coeff, double step, int zlo, int zhi,
                   float* out, cudaStream_t s, bool fast) {
    if (zhi <= zlo) return;
    if (fast) {
        float2* xp = nullptr;
        SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xp), level.count() * sizeof(float2), s));
        k_xpair_f32<<<grid_for(level.count()), kBlock, 0, s>>>(level.d, level.nx, level.ny, level.nz, xp);
        SFB_CUDA(cudaGetLastError());
        count_launch();
        const size_t rows = size_t(level.nx) * level.ny * size_t(zhi - zlo);
        k_graded_f32<<<grid_for(rows, 128), 128, 0, s>>>(level.dev(), xp, ts[0], ts[1], ts[2], coeff, step, zlo,
                                                         zhi, out);
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
    const size_t rows = size_t(level.nx) * level.ny * size_t(zhi - zlo);
    k_graded<<<grid_for(rows, 128), 128, 0, s>>>(level.dev(), xp, ts[0], ts[1], ts[2], coeff, step, zlo, zhi, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    SFB_CUDA(cudaFreeAsync(xp, s));
}

void launch_conv3(const sf_grid& in, const float k27[27], int zlo, int zhi, float* out, cudaStream_t s, bool fast) {
    if (zhi <= zlo) return;
    Kernel27 k;
    for (int i = 0; i < 27; ++i) k.k[i] = k27[i];
    (fast ? k_conv3<true> : k_conv3<false>)<<<grid_for(size_t(in.nx) * in.ny * size_t(zhi - zlo)), kBlock, 0, s>>>(
        in.d, in.nx, in.ny, in.nz, k, zlo, zhi, out);
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
    (halving ? k_combine<true> : k_combine<false>)<<<grid_for(size_t(base.nx) * base.ny * size_t(zhi - zlo)), kBlock, 0,
                                                      s>>>(lv, base.dev(), zlo, zhi, out);
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
