// sf_fused.cu — production front half of the query: per shading point, sample
// the 266 template features, sort/pool every (layer, feature type) and emit the
// tensor-core operands directly (K5 + K6 fused: the fp32 features stay in shared memory;
// the sorted bf16 operand blocks go to HBM for k_backbone_tc).
//
// Block = 8 consecutive queries (one 8-row group of a 128-row UMMA tile):
//  phase 1  warp w samples the template points of query q0 + w, point-parallel so a
//           warp's gathers stay inside one template footprint. Density and
//           transmittance come from xy-quad records {rho, T} at (x0, y), (x0 + 1, y),
//           (x0, y + 1), (x0 + 1, y + 1) (one 32-byte load per z corner row, k_xpair);
//           the Eq. 8 phase feature from
//           phase planes pre-blended at each lobe's g, held in shared memory.
//  phase 2  thread-per-(query, segment) register bitonic sorts (a 48-point layer is
//           split over a lane pair), sequential float sum in sorted order
//           (src/predictor.cpp:176-185) and max;
//  phase 3  every 16-byte chunk of the bf16 FC-1 feature operand rows
//           [sorted_tau, mean_tau, max_tau, 0...] goes straight into the UMMA
//           canonical layout (the 8 rows of a chunk are 128 contiguous bytes), plus
//           the fp32 {mean, max} x 3 types row of every (kind, layer) for attention.
//
// Numerics (bf16 production path only; the FP32 parity path keeps the exact
// kernels of sf_query.cu): the query base point and highlight entry are placed in
// voxel space in FP64 and split into an integer cell plus an FP32 fraction; template
// offsets, interpolation weights, lerps, phase angles and the phase bilinear are
// FP32 (relative errors ~1e-6, far inside the 3.9e-3 bf16 rounding the operands
// then undergo). Diffuse placement is a pure translation, so each diffuse point's
// voxel offset, unit axis, aperture and light-side cap integral are per-scene
// constants (made by the first blocks of k_query_prep).
#include <algorithm>
#include <cstdlib>

#include "sf_internal.h"
#include "sf_umma.cuh"

namespace sfb {

namespace {

// Block shapes of k_sample_sort: kW queries per group = warps per block, kMinB blocks per SM
// (64 registers either way, 32 warps per SM). The 32-warp block is preferred (one copy of the
// phase planes per SM and the largest L1); the 8-warp block is the fallback when its shared
// memory does not fit (very large templates).
constexpr int kWBig = 32, kMinBBig = 1, kWSmall = 8, kMinBSmall = 4;
constexpr int kSortThreadsPerSM = kWBig * 32 * kMinBBig;
static_assert(kWSmall * 32 * kMinBSmall == kSortThreadsPerSM, "both shapes: one query per warp, 32 warps per SM");

constexpr int kMaxSegs = 72;  // (kind, layer, tau) segments: 24 template layers
constexpr int kMaxChunks = 512;

struct SortDesc {
    int npts0, ntot;
    int n_segs, n_layers, n_chunks, n_tasks;
    int n_tiles;  // tiles of the operand layout (the backbone launch's batch)
    int tile0;    // first tile this launch fills; its rows / recs / feats start at row 0
    int64_t n_groups;  // 8-query groups this launch processes
    int64_t feat_stride;
    int A, H, n_planes;
    float su, sv;  // float(A - 1) / float(pi), float(H - 1) / float(pi): IEEE quotients, made once on the host
    float w[3];
    int scr_floats;
    int seg_scr[kMaxSegs];  // offset of the segment in the query scratch row
    int seg_n[kMaxSegs];
    int seg_kf[kMaxSegs];
    int64_t seg_prefix[kMaxSegs];
    uint8_t chunk_seg[kMaxChunks];
    uint8_t chunk_j[kMaxChunks];
    uint8_t task_seg[2 * kMaxSegs];  // sort tasks by network size; bit 7 = upper half of a 64-wide pair
    int debug;  // SF_DEBUG_SAMPLE_SORT (-DSF_SAMPLE_SORT_DEBUG builds): 1 skip sampling, 2 skip sort, 4 skip stores
    int mixed;                       // per-query g (C4): phase from the full table at the query's g
    int G;                           // table g resolution
    const float* table;              // [G][A][H] (mixed only)
    const float4* quad;              // the table's quad records (mixed only, see table_phase)
    int nbuf;                        // scratch buffers (2: one block barrier per group, if 3 blocks/SM still fit)
    int f16;  // bit 0: operand blocks in fp16 (SF_PRECISION_FP16) instead of bf16; bit 1: plain
              // stores (the chunk's operands stay in L2 for the backbone) instead of evict-first
};

// Bilinear lookup in a pre-blended phase plane pl[a][h] = P(a,h), rows padded to H+1 floats
// (rows a and a+1 in different banks).
__device__ __forceinline__ float plane_lookup(const float* pl, int A, int H, float sv, float ua, float half) {
    const float u = fminf(fmaxf(ua, 0.0f), float(A - 1));  // angle coordinate, see unit_coord
    int i0 = min(int(u), A - 2);
    float t = u - float(i0);
    float v = fminf(fmaxf(half, 0.0f), float(kPi)) * sv;
    int j0 = min(int(v), H - 2);
    float s = v - float(j0);
    const float* p0 = pl + i0 * (H + 1) + j0;
    const float* p1 = p0 + (H + 1);
    const float r00 = p0[0], r01 = p0[1], r10 = p1[0], r11 = p1[1];
    float a = fmaf(s, r01 - r00, r00);
    float b = fmaf(s, r11 - r10, r10);
    return fmaf(t, b - a, a);
}

// Angle coordinate of the phase table, u = angle_between(a, b) (A - 1) / pi (inc/math.h:53-56,
// src/phase.cpp:196-205), for unit vectors a and b, from t = 2 asin(|a -/+ b| / 2): u = t su, or
// (A - 1) - t su when a . b < 0 (angle = pi - t). Both branches keep the error ~1e-7 rad where
// acos of an FP32 dot product loses sqrt(eps) ~ 3e-4 rad near 0 and pi, and an FP32 angle near
// pi rounds to ulp(pi); the phase features stay within ~1e-5 of the reference's FP64 lookup
// (tests/test_gpu_reference_live.py).
__device__ __forceinline__ float unit_coord(float ax, float ay, float az, float bx, float by, float bz, float su,
                                           int A) {
    const float dot = fmaf(ax, bx, fmaf(ay, by, az * bz));
    const float sg = dot < 0.0f ? -1.0f : 1.0f;
    const float dx = fmaf(-sg, bx, ax), dy = fmaf(-sg, by, ay), dz = fmaf(-sg, bz, az);
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));  // |a -/+ b|^2 in [0, 2]
#ifdef SF_ASIN_LIBM
    const float t = 2.0f * asinf(fminf(0.5f * sqrtf(d2), 1.0f));
#else
    // x = |a -/+ b| / 2 in [0, 1/sqrt(2)]; asin(x) = x + x^3 P(x^2), P of degree 6 fitted on that
    // range (|error| <= 8e-8 rad in FP32)
    const float x = fminf(0.5f * d2 * rsqrtf(fmaxf(d2, 1e-30f)), 0.70710678f);
    const float z = x * x;
    float p = 0.08381619f;
    p = fmaf(p, z, -0.04671106f);
    p = fmaf(p, z, 0.04723444f);
    p = fmaf(p, z, 0.02576619f);
    p = fmaf(p, z, 0.04502971f);
    p = fmaf(p, z, 0.07498878f);
    p = fmaf(p, z, 0.16666670f);
    const float t = 2.0f * fmaf(x * z, p, x);
#endif
    return dot < 0.0f ? fmaf(-t, su, float(A - 1)) : t * su;
}

#ifndef SF_PLANE_PAIRS
#define SF_PLANE_PAIRS 1
#endif
// k_sample_sort's shared-memory copy of the planes as (aperture) pairs: entry (i, j) of a row
// of H + 1 float2 = {p[i][j], p[i][j + 1]}, so a bilinear lookup is two 8-byte loads instead of
// four scalar ones (the odd row stride spreads the rows over the banks). Same values, same
// arithmetic as plane_lookup.
__device__ __forceinline__ float plane_lookup_pairs(const float2* pl, int A, int H, float sv, float ua, float half) {
    const float u = fminf(fmaxf(ua, 0.0f), float(A - 1));
    int i0 = min(int(u), A - 2);
    float t = u - float(i0);
    float v = fminf(fmaxf(half, 0.0f), float(kPi)) * sv;
    int j0 = min(int(v), H - 2);
    float s = v - float(j0);
    const float2 q0 = pl[i0 * (H + 1) + j0], q1 = pl[(i0 + 1) * (H + 1) + j0];
    float a = fmaf(s, q0.y - q0.x, q0.x);
    float b = fmaf(s, q1.y - q1.x, q1.x);
    return fmaf(t, b - a, a);
}

// PhaseTable::lookup (src/phase.cpp:221-230) on the pre-blended planes.
__device__ __forceinline__ float cap_phase(const float* planes, const SortDesc& d, float ua, float half) {
    if (d.n_planes == 1) return d.w[0] * plane_lookup(planes, d.A, d.H, d.sv, ua, half);  // one lobe / iso
    float f = 0.0f;
    for (int k = 0; k < d.n_planes; ++k)
        f = fmaf(d.w[k], plane_lookup(planes + k * d.A * (d.H + 1), d.A, d.H, d.sv, ua, half), f);
    return f;
}

// PhaseTable::lookup_hg (src/phase.cpp:191-219) at a per-query g cell (gi, gt) on the full
// table [G][A][H] (L1/L2 resident): bilinear in (angle, aperture) on planes gi and gi + 1, then
// the g lerp. FP32 (production path only). The eight corners come from two 16-byte quad records
// (rows a and a + 1, each {P(gi, a, h), P(gi, a, h + 1), P(gi + 1, a, h), P(gi + 1, a, h + 1)})
// instead of eight scalar loads: same values, same arithmetic.
__device__ __forceinline__ float table_phase(const SortDesc& d, int gi, float gt, float ua, float half) {
    const int A = d.A, H = d.H;
    const float u = fminf(fmaxf(ua, 0.0f), float(A - 1));
    const int i0 = min(int(u), A - 2);
    const float t = u - float(i0);
    const float v = fminf(fmaxf(half, 0.0f), float(kPi)) * d.sv;
    const int j0 = min(int(v), H - 2);
    const float s = v - float(j0);
    const float4* qb = d.quad + (size_t(gi) * A + i0) * H + j0;
    const float4 q0 = __ldg(qb), q1 = __ldg(qb + H);
    const float r00[2] = {q0.x, q0.z}, r01[2] = {q0.y, q0.w}, r10[2] = {q1.x, q1.z}, r11[2] = {q1.y, q1.w};
    float pg[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float a = fmaf(s, r01[k] - r00[k], r00[k]), c = fmaf(s, r11[k] - r10[k], r10[k]);
        pg[k] = fmaf(t, c - a, a);
    }
    return d.w[0] * fmaf(gt, pg[1] - pg[0], pg[0]);
}

// voxel-space coordinate (s - o)/vs - 0.5 split into an integer cell base and an FP32 fraction
__device__ __forceinline__ void voxel_split(const GridDev& g, const double* s, int* base, float* frac) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double o = c == 0 ? g.ox : (c == 1 ? g.oy : g.oz);
        const double f = g.ivs != 0.0 ? (s[c] - o) * g.ivs - 0.5 : (s[c] - o) / g.vs - 0.5;
        const double fl = floor(f);
        base[c] = int(fl);
        frac[c] = float(f - fl);
    }
}

// Per-query context, computed once per query by k_query_prep (one thread per
// query) instead of redundantly by the 32 lanes of the sampling warp.
struct __align__(16) QueryCtx {  // 240 bytes: copied as 16-byte chunks
    int pb[3];               // query base cell
    float pf[3];             // query base fraction
    int eb[3];               // highlight entry cell
    float ef[3];             // highlight entry fraction
    float dpe[3];            // (entry - p) in voxels
    float t[3], b[3], a[3];  // highlight frame
    float hs;                // highlight scale in voxels per template unit
    float wf[3], iw;         // omega and 1/|omega|
    float lf[3], il;         // light and 1/|light|
    float pbox[6], ebox[6];  // in-box fraction bounds relative to pb / eb
    int ok;                  // highlight entry != p
    int same_light;          // light and medium equal query 0's (diffuse light side precomputed)
    int gi;                  // per-query g (mixed media): table g cell and weight
    float gt;
    int tiny;                // highlight template within half a voxel of its entry (see query_ctx)
    float eface[6];          // the entry's distances to the box faces (lo x, y, z, hi x, y, z), voxels
    int pad_[3];
};

static_assert(sizeof(QueryCtx) % 16 == 0, "QueryCtx is moved in 16-byte chunks");

// Phase feature factor at the query's medium: the scene's pre-blended planes, or the full
// table at the query's own g (mixed media). kPh: kPhPlanes (any number of lobes), kPhMixed (per-query
// g, full table), kPhOne (one pre-blended plane: no per-lookup lobe loop).
constexpr int kPhPlanes = 0, kPhMixed = 1, kPhOne = 2;
template <int kPh>
__device__ __forceinline__ float qphase(const float* planes, const SortDesc& d, const QueryCtx& q, float ua,
                                       float half) {
    constexpr bool kMixed = kPh == kPhMixed;
#if SF_PLANE_PAIRS
    if (kMixed) return table_phase(d, q.gi, q.gt, ua, half);
    const float2* pp = reinterpret_cast<const float2*>(planes);
    if (kPh == kPhOne || d.n_planes == 1) return d.w[0] * plane_lookup_pairs(pp, d.A, d.H, d.sv, ua, half);
    float f = 0.0f;
    for (int k = 0; k < d.n_planes; ++k)
        f = fmaf(d.w[k], plane_lookup_pairs(pp + k * d.A * (d.H + 1), d.A, d.H, d.sv, ua, half), f);
    return f;
#else
    return kMixed ? table_phase(d, q.gi, q.gt, ua, half) : cap_phase(planes, d, ua, half);
#endif
}

__device__ __forceinline__ void box_bounds(const GridDev& g, const int* base, float* box) {
    const int n[3] = {g.nx, g.ny, g.nz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        box[2 * c] = -0.5f - float(base[c]);
        box[2 * c + 1] = float(n[c] - base[c]) - 0.5f;
    }
}

__device__ __forceinline__ void query_ctx(const SceneDev& sc, const TemplateDev& ht, const double* c, QueryCtx& q) {
    const double p[3] = {c[0], c[1], c[2]}, omega[3] = {c[3], c[4], c[5]}, light[3] = {c[6], c[7], c[8]};
    const GridDev& g = sc.grid;
    voxel_split(g, p, q.pb, q.pf);
    {  // unit omega and light (normalised in FP64)
        const double iw = 1.0 / sqrt(dot3(omega, omega)), il = 1.0 / sqrt(dot3(light, light));
        for (int i = 0; i < 3; ++i) {
            q.wf[i] = float(omega[i] * iw);
            q.lf[i] = float(light[i] * il);
        }
        q.iw = q.il = 1.0f;
    }
    // light entry + highlight frame (src/feature_pipeline.cpp:130-137, src/templates.cpp:220-239)
    const double lo[3] = {g.ox, g.oy, g.oz}, hi[3] = {g.hx, g.hy, g.hz};
    double entry[3];
    light_entry(lo, hi, p, light, entry);
    voxel_split(g, entry, q.eb, q.ef);
    double span[3] = {p[0] - entry[0], p[1] - entry[1], p[2] - entry[2]};
    const double len = sqrt(dot3(span, span));
    q.ok = len > 0.0 ? 1 : 0;
    const double il = 1.0 / len;
    double axis[3] = {span[0] * il, span[1] * il, span[2] * il};
    const double od = dot3(omega, axis);
    double t[3] = {omega[0] - axis[0] * od, omega[1] - axis[1] * od, omega[2] - axis[2] * od};
    const double tl = sqrt(dot3(t, t));
    double b[3];
    if (tl > 1e-9) {
        const double it = 1.0 / tl;
        for (int i = 0; i < 3; ++i) t[i] *= it;
        b[0] = axis[1] * t[2] - axis[2] * t[1];
        b[1] = axis[2] * t[0] - axis[0] * t[2];
        b[2] = axis[0] * t[1] - axis[1] * t[0];
    } else {
        orthonormal_basis(axis, t, b);
    }
    const double ivs = g.ivs != 0.0 ? g.ivs : 1.0 / g.vs;
    for (int i = 0; i < 3; ++i) {
        q.t[i] = float(t[i]);
        q.b[i] = float(b[i]);
        q.a[i] = float(axis[i]);
    }
    q.hs = float(len / ht.gen_distance * ivs);
    // A highlight template shrunk to within half a voxel of its entry point (p on or next to the
    // face the light enters through) straddles that face at a scale the entry's FP32 voxel
    // fraction does not resolve: its points are tested against the box by their offset from the
    // entry and the entry's own distances to the faces (both accurate relative to themselves).
    q.tiny = len * ivs < 0.5 ? 1 : 0;
    for (int i = 0; i < 3; ++i) {
        q.eface[i] = float((entry[i] - lo[i]) * ivs);
        q.eface[3 + i] = float((hi[i] - entry[i]) * ivs);
        q.dpe[i] = float((entry[i] - p[i]) * ivs);  // FP64 difference: no cancellation when len is tiny
    }
    box_bounds(g, q.pb, q.pbox);
    box_bounds(g, q.eb, q.ebox);
    for (int i = 0; i < 3; ++i) {  // bases in the padded record coordinates (voxel + 1), see k_xpair
        ++q.pb[i];
        ++q.eb[i];
    }
}

// 256-bit read-only load (sm_100: LDG.E.ENL2.256): one L1 wavefront per distinct line for
// the whole 32-byte record instead of one per 16-byte half
__device__ __forceinline__ void ld_nc_256(const float4* p, float4& a, float4& b) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

// {density, transmittance} at voxel coordinate base + frac: 0 / 1 outside the box
// (sample_trilinear + TransmittanceFeatureVolume::sample), else trilinear over
// xy-quad records with the clamp-to-edge cell of src/volume_grid.cpp:45-56.
// `box` = per-base {lo, hi} fraction bounds of the closed grid box: inside iff
// lo_c <= f_c <= hi_c (lo = -0.5 - base, hi = n - 0.5 - base).
__device__ __forceinline__ void sample_rt_in(const SceneDev& sc, const int* base, bool inside, const float* f,
                                             float& rho, float& tr) {
    const GridDev& g = sc.grid;
    if (!inside) {
        rho = 0.0f;
        tr = 1.0f;
        return;
    }
    // padded record coordinates (voxel + 1, edges replicated: see k_xpair) need no clamps: a
    // clamped corner reads a record equal to its neighbour, so a + t (b - a) = a exactly
    uint32_t i0[3];
    float t[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float fl = floorf(f[c]);
        i0[c] = uint32_t(base[c] + int(fl));
        t[c] = f[c] - fl;
    }
    // the cell's two xy-quad records (z0 and z0 + 1), one 256-bit load each; record indices as
    // unsigned 32-bit sums (< 2^31 records): one IMAD.WIDE.U32 per address
    const uint32_t x0 = i0[0], z0 = i0[2], z1 = z0 + 1;
    const uint32_t b = ((x0 >> 1) << 2) + (x0 & 1) + i0[1] * g.rec_sx;
    const uint32_t ra = (z0 >> 1) * g.rec_sz + ((z0 & 1) << 1) + b, rb = (z1 >> 1) * g.rec_sz + ((z1 & 1) << 1) + b;
    const float4* v = sc.dt4;
    float4 r00, r10, r01, r11;  // r<y><z>: {rho, T}(x0), {rho, T}(x0 + 1) of row (y, z)
    ld_nc_256(v + 2 * size_t(ra), r00, r10);
    ld_nc_256(v + 2 * size_t(rb), r01, r11);
#ifdef SF_LERP_DIFF
    float c00 = fmaf(t[0], r00.z - r00.x, r00.x), c10 = fmaf(t[0], r10.z - r10.x, r10.x);
    float c01 = fmaf(t[0], r01.z - r01.x, r01.x), c11 = fmaf(t[0], r11.z - r11.x, r11.x);
    float e0 = fmaf(t[1], c10 - c00, c00), e1 = fmaf(t[1], c11 - c01, c01);
    rho = fmaf(t[2], e1 - e0, e0);
    c00 = fmaf(t[0], r00.w - r00.y, r00.y);
    c10 = fmaf(t[0], r10.w - r10.y, r10.y);
    c01 = fmaf(t[0], r01.w - r01.y, r01.y);
    c11 = fmaf(t[0], r11.w - r11.y, r11.y);
    e0 = fmaf(t[1], c10 - c00, c00);
    e1 = fmaf(t[1], c11 - c01, c01);
    tr = fmaf(t[2], e1 - e0, e0);
#else
    // (1 - t) a + t b: both fields are non-negative, so every term is, and a value much smaller
    // than its neighbours keeps its relative accuracy (a + t (b - a) loses ulp(max(a, b)))
    const float u0 = 1.0f - t[0], u1 = 1.0f - t[1], u2 = 1.0f - t[2];
    float c00 = fmaf(u0, r00.x, t[0] * r00.z), c10 = fmaf(u0, r10.x, t[0] * r10.z);
    float c01 = fmaf(u0, r01.x, t[0] * r01.z), c11 = fmaf(u0, r11.x, t[0] * r11.z);
    float e0 = fmaf(u1, c00, t[1] * c10), e1 = fmaf(u1, c01, t[1] * c11);
    rho = fmaf(u2, e0, t[2] * e1);
    c00 = fmaf(u0, r00.y, t[0] * r00.w);
    c10 = fmaf(u0, r10.y, t[0] * r10.w);
    c01 = fmaf(u0, r01.y, t[0] * r01.w);
    c11 = fmaf(u0, r11.y, t[0] * r11.w);
    e0 = fmaf(u1, c00, t[1] * c10);
    e1 = fmaf(u1, c01, t[1] * c11);
    tr = fmaf(u2, e0, t[2] * e1);
#endif
}

__device__ __forceinline__ void sample_rt(const SceneDev& sc, const int* base, const float* box, const float* f,
                                          float& rho, float& tr) {
    // non-short-circuit: one predicate chain instead of six compare-and-branch pairs
    const bool inside = (f[0] >= box[0]) & (f[0] <= box[1]) & (f[1] >= box[2]) & (f[1] <= box[3]) &
                        (f[2] >= box[4]) & (f[2] <= box[5]);
    sample_rt_in(sc, base, inside, f, rho, tr);
}

// Features of template point i (diffuse 0..npts0-1, then highlight).
template <int kPh>
__device__ __forceinline__ void point_features(const SceneDev& sc, const TemplateDev& ht, const QueryCtx& q, int i,
                                               const SortDesc& d, const float* planes, const float4* __restrict__ pre,
                                               bool same_light, float& rho, float& tr, float& ph) {
    if (i < d.npts0) {
        float4 p0, p1;  // {offset, half}, {axis, light side}: one 256-bit load
        ld_nc_256(pre + 2 * i, p0, p1);
        const float f[3] = {q.pf[0] + p0.x, q.pf[1] + p0.y, q.pf[2] + p0.z};
        sample_rt(sc, q.pb, q.pbox, f, rho, tr);
        if (p0.w < 0.0f) {
            ph = 1.0f;  // diffuse centre point (src/feature_pipeline.cpp:163-164)
            return;
        }
        const float fw = qphase<kPh>(planes, d, q, unit_coord(q.wf[0], q.wf[1], q.wf[2], p1.x, p1.y, p1.z, d.su, d.A), p0.w);
        const float fl = same_light
                             ? p1.w
                             : qphase<kPh>(planes, d, q, unit_coord(q.lf[0], q.lf[1], q.lf[2], p1.x, p1.y, p1.z, d.su, d.A), p0.w);
        ph = fw * fl;
        return;
    }
    const float4 tq = __ldg(ht.pts4 + (i - d.npts0));  // {x, y, z, cap}
    float h[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) h[c] = fmaf(q.a[c], tq.z, fmaf(q.b[c], tq.y, q.t[c] * tq.x)) * q.hs;
    const float f[3] = {q.ef[0] + h[0], q.ef[1] + h[1], q.ef[2] + h[2]};
    if (q.tiny) {  // warp-uniform (one query per warp): the box test relative to the entry
        const bool inside = (h[0] >= -q.eface[0]) & (h[0] <= q.eface[3]) & (h[1] >= -q.eface[1]) &
                            (h[1] <= q.eface[4]) & (h[2] >= -q.eface[2]) & (h[2] <= q.eface[5]);
        sample_rt_in(sc, q.eb, inside, f, rho, tr);
    } else {
        sample_rt(sc, q.eb, q.ebox, f, rho, tr);
    }
    const float dx = q.dpe[0] + h[0], dy = q.dpe[1] + h[1], dz = q.dpe[2] + h[2];
    const float dd = dx * dx + dy * dy + dz * dz;
    if (dd <= 0.0f) {
        ph = 1.0f;
        return;
    }
    const float inv = rsqrtf(dd);
    const float r = tq.w * q.hs * inv;  // cap / dist, both in voxels
    const float half = r >= 1.0f ? float(kPi) : asinf(r);
    const float ax = dx * inv, ay = dy * inv, az = dz * inv;
    ph = qphase<kPh>(planes, d, q, unit_coord(q.wf[0], q.wf[1], q.wf[2], ax, ay, az, d.su, d.A), half) *
         qphase<kPh>(planes, d, q, unit_coord(q.lf[0], q.lf[1], q.lf[2], ax, ay, az, d.su, d.A), half);
}

// Per-scene diffuse constants: pre[2i] = {offset (voxels), half angle or -1 at the
// centre}, pre[2i+1] = {unit axis, light-side cap integral for the light of query 0}.
__device__ __forceinline__ void diffuse_point(const SceneDev& sc, const TemplateDev& dt, const SortDesc& d,
                                              const float* __restrict__ planes, const double* __restrict__ queries,
                                              int i, float4* __restrict__ pre) {
    const double* qq = dt.pts + 3 * i;
    const double ts = sc.template_scale;
    const double ivs = sc.grid.ivs != 0.0 ? sc.grid.ivs : 1.0 / sc.grid.vs;
    const double ox = qq[0] * ts, oy = qq[1] * ts, oz = qq[2] * ts;
    const double dd = ox * ox + oy * oy + oz * oz;
    if (dd <= 0.0) {
        pre[2 * i] = make_float4(0.0f, 0.0f, 0.0f, -1.0f);
        pre[2 * i + 1] = make_float4(0.0f, 0.0f, 0.0f, 1.0f);
        return;
    }
    const double dist = sqrt(dd), cap = dt.caps[i] * ts;
    const float half = float(cap >= dist ? kPi : asin(cap / dist));
    const float ax = float(ox / dist), ay = float(oy / dist), az = float(oz / dist);
    // light side of the cap: angle_between(l, axis) in FP64 (inc/math.h:53-56), once per scene
    const double axis[3] = {ox / dist, oy / dist, oz / dist};
    const float ul = float(angle_between(queries + 6, axis) / kPi * (d.A - 1));
    pre[2 * i] = make_float4(float(ox * ivs), float(oy * ivs), float(oz * ivs), half);
    pre[2 * i + 1] = make_float4(ax, ay, az, cap_phase(planes, d, ul, half));
}

// Per-query preparation for the production path: make_config rows
// (src/predictor.cpp:261-274, alpha = angle_between(omega, l)) and the sampling
// context (voxel-space bases, highlight frame, in-box bounds). One thread per query; the
// block's records and config rows are staged in shared memory and stored as contiguous
// 16-byte chunks. With `dt` set, the first blocks also make the per-scene diffuse constants
// (diffuse placement is a pure translation, so axis and aperture do not depend on p).
constexpr int kPrepThreads = 128;

__global__ void __launch_bounds__(kPrepThreads)
    k_query_prep(SceneDev sc, TemplateDev ht, sf_medium_params m, int64_t n, const double* __restrict__ queries,
                 const double* __restrict__ media, double* __restrict__ cfg8, QueryCtx* __restrict__ recs,
                 const int* __restrict__ perm, const double* __restrict__ row0, TemplateDev dt, SortDesc d,
                 const float* __restrict__ planes, float4* __restrict__ pre, int diffuse_blocks) {
    if (int(blockIdx.x) < diffuse_blocks) {
        const int i = blockIdx.x * kPrepThreads + threadIdx.x;
        if (i < dt.total) diffuse_point(sc, dt, d, planes, row0, i, pre);
        return;
    }
    __shared__ __align__(16) QueryCtx s_rec[kPrepThreads];
    __shared__ __align__(16) double s_cfg[kPrepThreads * 8];
    const int64_t nblk = int64_t(gridDim.x) - diffuse_blocks;
    for (int64_t q0 = (int64_t(blockIdx.x) - diffuse_blocks) * kPrepThreads; q0 < n; q0 += nblk * kPrepThreads) {
        const int64_t q = q0 + threadIdx.x;
        if (q < n) {
            const int64_t src = perm ? int64_t(perm[q]) : q;  // processing order -> the caller's row
            const double* c = queries + 9 * src;
            QueryCtx qc;
            query_ctx(sc, ht, c, qc);
            // the diffuse light side was precomputed for the light of the batch's row 0
            qc.same_light = (!media && c[6] == row0[6] && c[7] == row0[7] && c[8] == row0[8]) ? 1 : 0;
            qc.gi = 0;
            qc.gt = 0.0f;
            if (media) {  // g axis of PhaseTable::lookup_hg (src/phase.cpp:196-205) at the query's g
                double gt;
                table_coord(media[4 * src], -0.99, 0.99, sc.phase.gr, qc.gi, gt);
                qc.gt = float(gt);
            }
            qc.pad_[0] = qc.pad_[1] = qc.pad_[2] = 0;
            s_rec[threadIdx.x] = qc;
            write_cfg8(m, media ? media + 4 * src : nullptr, c, s_cfg + 8 * threadIdx.x);
            if (!qc.ok)  // highlight placement fails (entry == p; the reference throws, src/templates.cpp:219-220):
                for (int k = 4; k < 7; ++k) s_cfg[8 * threadIdx.x + k] = __longlong_as_double(0x7ff8000000000000LL);
        }
        __syncthreads();
        const int rows = n - q0 < kPrepThreads ? int(n - q0) : kPrepThreads;
        const int4* rs = reinterpret_cast<const int4*>(s_rec);
        int4* rd = reinterpret_cast<int4*>(recs + q0);
        for (int k = threadIdx.x; k < rows * int(sizeof(QueryCtx) / 16); k += kPrepThreads) rd[k] = rs[k];
        const int4* cs = reinterpret_cast<const int4*>(s_cfg);
        int4* cd = reinterpret_cast<int4*>(cfg8 + 8 * q0);
        for (int k = threadIdx.x; k < rows * 4; k += kPrepThreads) cd[k] = cs[k];
        __syncthreads();
    }
}

// Morton interleave of a 10-bit coordinate (the query cell order below uses 6 bits per axis).
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 1023u;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// Counting sort of the queries by the Morton code of their 64^3 cell (launch_cell_order).
__global__ void k_cell_key(GridDev g, int64_t n, const double* __restrict__ queries, uint32_t* __restrict__ cells,
                           int* __restrict__ counts) {
    const double ext[3] = {g.hx - g.ox, g.hy - g.oy, g.hz - g.oz};
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) {
        uint32_t c[3];
        for (int k = 0; k < 3; ++k) {
            const double o = k == 0 ? g.ox : (k == 1 ? g.oy : g.oz);
            const double u = (queries[9 * q + k] - o) / ext[k] * 64.0;
            c[k] = uint32_t(fmin(fmax(u, 0.0), 63.0));
        }
        const uint32_t key = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);  // 18 bits
        cells[q] = key;
        atomicAdd(&counts[key], 1);
    }
}

// Exclusive scan of the cell counts in two levels: every 1024-cell tile in place (warp shuffles +
// one shared-memory pass), the tile totals into counts[kOrderCells ...] and scanned by one block.
__global__ void __launch_bounds__(1024) k_cell_tile_scan(int* __restrict__ counts) {
    __shared__ int warp_sums[32];
    const int i = blockIdx.x * 1024 + threadIdx.x;
    int total;
    const int ex = block_exclusive_scan(counts[i], warp_sums, total);
    counts[i] = ex;
    if (threadIdx.x == 0) counts[kOrderCells + blockIdx.x] = total;
}

__global__ void __launch_bounds__(kOrderCells / 1024) k_cell_sum_scan(int* __restrict__ counts) {
    __shared__ int warp_sums[32];
    int* sums = counts + kOrderCells;
    int total;
    sums[threadIdx.x] = block_exclusive_scan(sums[threadIdx.x], warp_sums, total);
}

__global__ void k_cell_scatter(int64_t n, const uint32_t* __restrict__ cells, int* __restrict__ offsets,
                               int* __restrict__ perm) {
    const int* tile_off = offsets + kOrderCells;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = cells[q];
        perm[atomicAdd(&offsets[c], 1) + tile_off[c >> 10]] = int(q);
    }
}

// xy-quad record of padded voxel (x, y, z) = voxel (x-1, y-1, z-1) with every coordinate
// clamped to the grid (edge replication; x in [0, nx], y in [0, ny], z in [0, nz + 1]):
// 32 bytes {rho, T}(x, y), {rho, T}(x+1, y), {rho, T}(x, y+1), {rho, T}(x+1, y+1) at z. The
// clamp-to-edge corners of sample_trilinear (src/volume_grid.cpp:45-56) then read replicated
// values, so the sampler has no clamps, and a trilinear cell is two 256-bit loads (z0, z0+1).
// Four records share a 128-byte line as a 2x1x2 (x, y, z) brick: a cell's two records are in
// one line when z0 is even. Index ((z/2 * PY + y) * XH + x/2) * 4 + (z&1) * 2 + (x&1).
// One thread per 128-byte brick (x pair 2xh, 2xh + 1; z pair 2zh, 2zh + 1; one y): its four
// records read three clamped x columns of two y rows at two z slices (24 loads), are staged in
// shared memory and leave as whole contiguous lines (a warp stores 512 contiguous bytes per
// instruction). 32-bit index math; every brick of the layout is written (padding bricks hold
// clamped values no lookup reads).
constexpr int kXpairThreads = 256;
__global__ void __launch_bounds__(kXpairThreads) k_xpair(const float* __restrict__ rho, const float* __restrict__ tr,
                                                         int nx, int ny, int nz, float4* __restrict__ out) {
    __shared__ float4 st[kXpairThreads * 8];
    const int XH = (nx + 2) >> 1, py = ny + 1;
    const int per_slab = XH * py;  // bricks of one z pair
    const int zh = blockIdx.y;
    const int m0 = blockIdx.x * kXpairThreads;
    const int m = m0 + threadIdx.x;
    if (m < per_slab) {
        const int y = m / XH, xh = m - y * XH;
        const int xa = min(max(2 * xh - 1, 0), nx - 1), xb = min(2 * xh, nx - 1), xc = min(2 * xh + 1, nx - 1);
        const int y0 = min(max(y - 1, 0), ny - 1), y1 = min(y, ny - 1);
        // brick: rec (dz, dx) at float4 2 (2 dz + dx), each 2 float4; slots XOR-swizzled by the
        // brick's index so the stores of a warp spread over the banks
        float4* b = st + threadIdx.x * 8;
        const int sw = threadIdx.x & 7;
#pragma unroll
        for (int dz = 0; dz < 2; ++dz) {
            const int cz = min(max(2 * zh + dz - 1, 0), nz - 1);
            const size_t r0 = (size_t(cz) * ny + y0) * nx, r1 = (size_t(cz) * ny + y1) * nx;
            const float ra0 = __ldg(rho + r0 + xa), rb0 = __ldg(rho + r0 + xb), rc0 = __ldg(rho + r0 + xc);
            const float ta0 = __ldg(tr + r0 + xa), tb0 = __ldg(tr + r0 + xb), tc0 = __ldg(tr + r0 + xc);
            const float ra1 = __ldg(rho + r1 + xa), rb1 = __ldg(rho + r1 + xb), rc1 = __ldg(rho + r1 + xc);
            const float ta1 = __ldg(tr + r1 + xa), tb1 = __ldg(tr + r1 + xb), tc1 = __ldg(tr + r1 + xc);
            // x = 2xh: corners (xa, xb); x = 2xh + 1: corners (xb, xc)
            b[(4 * dz + 0) ^ sw] = make_float4(ra0, ta0, rb0, tb0);
            b[(4 * dz + 1) ^ sw] = make_float4(ra1, ta1, rb1, tb1);
            b[(4 * dz + 2) ^ sw] = make_float4(rb0, tb0, rc0, tc0);
            b[(4 * dz + 3) ^ sw] = make_float4(rb1, tb1, rc1, tc1);
        }
    }
    __syncthreads();
    // the block's bricks are consecutive lines of one z-pair slab
    const int nb = min(kXpairThreads, per_slab - m0);
    float4* dst = out + (size_t(zh) * per_slab + m0) * 8;
    for (int k = threadIdx.x; k < nb * 8; k += kXpairThreads) __stcg(dst + k, st[(k & ~7) | ((k ^ (k >> 3)) & 7)]);
}

// Compile-time bitonic sort of P register values, descending if `desc`.
template <int P>
__device__ __forceinline__ void bitonic(float* v, bool desc) {
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const float a = v[i], b = v[l];
                    const float hi = fmaxf(a, b), lo = fminf(a, b);
                    if (((i & k) == 0) == desc) {
                        v[i] = hi;
                        v[l] = lo;
                    } else {
                        v[i] = lo;
                        v[l] = hi;
                    }
                }
            }
        }
    }
}

// Descending bitonic merge of a bitonic sequence of P values.
template <int P>
__device__ __forceinline__ void merge_desc(float* v) {
#pragma unroll
    for (int j = P >> 1; j > 0; j >>= 1) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int l = i ^ j;
            if (l > i) {
                const float a = v[i], b = v[l];
                v[i] = fmaxf(a, b);
                v[l] = fminf(a, b);
            }
        }
    }
}

// Where a sorted segment's operand row goes: chunk j (8 values = 16 bytes) of row
// `row` in the segment's [128 x kf] canonical block; pools go to the (kind, layer)
// mean/max row {mean d,p,t, max d,p,t, 0, 0}.
struct SegOut {
    uint8_t* blk;
    int row, kf, tau;
    float* mm;  // 8 floats
    int f16;    // SortDesc::f16 bits, uniform per launch
};

// Value idx of the operand row [sorted (cnt), mean, max, 0...] from the registers of
// a sorted segment (v holds positions off .. off+P-1).
template <int P>
__device__ __forceinline__ float row_value(const float* v, int off, int idx, int cnt, float mean, float mx) {
    const int r = idx - off;
    float x = idx == cnt ? mean : (idx == cnt + 1 ? mx : 0.0f);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (r == k && idx < cnt) x = v[k];
    return x;
}

// Chunks [j0, j1) of the operand row, written straight from registers (8 threads of
// consecutive query rows write one 128-byte line).
template <int P>
__device__ __forceinline__ void emit_chunks(const float* v, int off, int j0, int j1, int cnt, float mean, float mx,
                                            const SegOut& o) {
#pragma unroll
    for (int j = 0; j < (P + 2 + 15) / 16 * 2; ++j) {
        const int jj = j0 + j;
        if (jj >= j1) break;
        float v8[8];
        if (off == 0 && 8 * jj + 8 <= P) {  // fully inside the register block: static indices
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int idx = 8 * j + e;  // == 8 * jj + e when j0 == 0
                v8[e] = idx < cnt ? v[idx < P ? idx : 0] : (idx == cnt ? mean : (idx == cnt + 1 ? mx : 0.0f));
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v8[e] = row_value<P>(v, off, 8 * jj + e, cnt, mean, mx);
        }
        switch (o.f16) {
            case 0: store_chunk_stream<false>(o.blk, o.row, jj, o.kf, v8); break;
            case 1: store_chunk_stream<true>(o.blk, o.row, jj, o.kf, v8); break;
            case 2: store_chunk<false>(o.blk, o.row, jj, o.kf, v8); break;
            default: store_chunk<true>(o.blk, o.row, jj, o.kf, v8); break;
        }
    }
}

__device__ __forceinline__ void emit_pools(const SegOut& o, float mean, float mx) {
    o.mm[o.tau] = mean;
    o.mm[3 + o.tau] = mx;
    if (o.tau == 0) *reinterpret_cast<float2*>(o.mm + 6) = make_float2(0.0f, 0.0f);
}

// Batcher's odd-even merge sort of P (power of two) registers, descending, with every
// comparator that touches an index >= N dropped: positions >= N hold -INF padding, which a
// descending compare-exchange never moves, so the network sorts N values exactly (P = 32:
// 191 comparators instead of bitonic's 240; N = 24: 120; N = 12: 41; N = 6: 12).
template <int P, int N>
__device__ __forceinline__ void oem_sort_desc(float* v) {
    // comparators (a, a + k) of merge stage (p, k): a - k % p in [0, P) with (a - k % p) mod 2k < k,
    // both ends in the same 2p block (the iterative form of Batcher's network)
#pragma unroll
    for (int p = 1; p < P; p <<= 1)
#pragma unroll
        for (int k = p; k >= 1; k >>= 1)
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const int r = a - k % p, b = a + k;
                if (r >= 0 && r % (2 * k) < k && b < N && b < P && a / (2 * p) == b / (2 * p)) {
                    const float x = v[a], y = v[b];
                    v[a] = fmaxf(x, y);
                    v[b] = fminf(x, y);
                }
            }
}

// One thread sorts a segment of cnt <= N <= P values (descending), takes mean (sequential
// float sum in sorted order / cnt, src/predictor.cpp:176-185) and max, and writes the
// operand row and pools.
template <int P, int N = P>
__device__ __forceinline__ void sort_emit(const float* seg, int cnt, const SegOut& o, bool store) {
    float v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = j < cnt ? seg[j] : -INFINITY;
    oem_sort_desc<P, N>(v);
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < P; ++j)
        if (j < cnt) acc += v[j];
    const float mean = acc / float(cnt), mx = v[0];
    if (!store) return;
    emit_chunks<P>(v, 0, 0, o.kf / 8, cnt, 0.0f, 0.0f, o);  // operand row: sorted values, zero padding
    emit_pools(o, mean, mx);
}

// A lane pair sorts a 33..64-value segment: each lane sorts 32 (the upper lane
// ascending, making the 64 bitonic), one cross-lane compare-exchange, a descending
// merge per lane; the lower lane's running sum continues on the upper lane, so the
// sum is exactly sequential in sorted order. The lower lane emits chunks 0-3, the
// upper the rest (mean and max land there) and the pools.
template <int H>
__device__ __forceinline__ void sort_emit_pair(const float* seg, int cnt, bool upper, const SegOut& o, bool store) {
    // lane halves of H <= 32 values each (H = 24 for a 48-point layer: pruned 24-networks);
    // -INF padding fills each lane's 32 slots
    float v[32];
    const int base = upper ? H : 0, lim = upper ? cnt : (cnt < H ? cnt : H);
    const unsigned mask = __activemask();  // pair partners always run this branch together
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (j < H && base + j < lim) ? seg[base + j] : -INFINITY;
    oem_sort_desc<32, H>(v);
    // the upper lane's half reversed to ascending: lower desc + upper asc is one bitonic
    // sequence of 64 (the padding meets in the middle)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float a = v[j], b = v[31 - j];
        v[j] = upper ? b : a;
        v[31 - j] = upper ? a : b;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const float x = __shfl_xor_sync(mask, v[j], 1);
        v[j] = upper ? fminf(v[j], x) : fmaxf(v[j], x);
    }
    merge_desc<32>(v);
    float acc = 0.0f;
    if (!upper)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += v[j];
    acc = __shfl_xor_sync(mask, acc, 1);
    const float mx = __shfl_xor_sync(mask, v[0], 1);
    float mean = 0.0f;
    if (upper) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (32 + j < cnt) acc += v[j];
        mean = acc / float(cnt);
    }
    if (!store) return;
    if (!upper) {
        emit_chunks<32>(v, 0, 0, 4, cnt, 0.0f, 0.0f, o);
    } else {
        emit_chunks<32>(v, 32, 4, o.kf / 8, cnt, 0.0f, 0.0f, o);
        emit_pools(o, mean, mx);
    }
}

// kPh: phase lookups (kPhMixed: per-query g (C4), phase from the full table; kPhOne: one plane)
#ifdef SF_SAMPLE_SORT_DEBUG
#define SS_DEBUG(d) ((d).debug)
#else
#define SS_DEBUG(d) 0  // SF_DEBUG_SAMPLE_SORT needs a -DSF_SAMPLE_SORT_DEBUG build
#endif
template <int kPh, int kWarps, int kMinB>
__global__ void __launch_bounds__(kWarps * 32, kMinB)
    k_sample_sort(SceneDev sc, TemplateDev ht, SortDesc d, const float* __restrict__ planes_g,
                  const float4* __restrict__ pre, int64_t n, const QueryCtx* __restrict__ recs,
                  const float* __restrict__ feats, uint8_t* __restrict__ ops, float* __restrict__ mms, int* err) {
    extern __shared__ __align__(16) float sm[];
#if SF_PLANE_PAIRS
    const int plane_floats = 2 * d.n_planes * d.A * (d.H + 1);  // float2 pairs (plane_lookup_pairs)
    float* planes = sm;
    for (int i = threadIdx.x; i < plane_floats / 2; i += blockDim.x) {
        const bool last = i % (d.H + 1) == d.H;  // the row's last entry has no right neighbour (unused)
        reinterpret_cast<float2*>(planes)[i] = make_float2(planes_g[i], last ? 0.0f : planes_g[i + 1]);
    }
#else
    const int plane_floats = d.n_planes * d.A * (d.H + 1);
    float* planes = sm;
    for (int i = threadIdx.x; i < plane_floats; i += blockDim.x) planes[i] = planes_g[i];
#endif
    __shared__ int s_scr[kMaxSegs], s_n[kMaxSegs], s_kf[kMaxSegs];
    __shared__ int s_prefix[kMaxSegs];  // bytes per tile before the segment's block (< 2^31)
    __shared__ uint8_t s_task[2 * kMaxSegs];
    for (int i = threadIdx.x; i < d.n_segs; i += blockDim.x) {
        s_scr[i] = d.seg_scr[i];
        s_n[i] = d.seg_n[i];
        s_kf[i] = d.seg_kf[i];
        s_prefix[i] = int(d.seg_prefix[i]);
    }
    for (int i = threadIdx.x; i < d.n_tasks; i += blockDim.x) s_task[i] = d.task_seg[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // nbuf scratch buffers [8][scr_floats]: with two, group g+1 is sampled while g is still
    // being sorted by other warps and one block barrier per group suffices
    float* scr_buf = sm + plane_floats;
    QueryCtx* s_qc =
        reinterpret_cast<QueryCtx*>(sm + ((plane_floats + d.nbuf * kWarps * d.scr_floats + 3) & ~3));  // [2][8]
    const int64_t q_pad = int64_t(d.n_tiles) * kUmmaM;  // operand / pool layout
    const int64_t n_groups = d.n_groups;
    const int64_t qg0 = int64_t(d.tile0) * kUmmaM;      // global row of local row 0
    // per-warp prefetch of a group's query context (cp.async, 12 x 16 bytes)
    auto prefetch_ctx = [&](int64_t grp, int buf) {
        const int64_t q = grp * kWarps + warp;
        if (recs != nullptr && grp < n_groups && q < n && lane < int(sizeof(QueryCtx) / 16)) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&s_qc[buf * kWarps + warp])) + 16 * lane;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(reinterpret_cast<const char*>(recs + q) + 16 * lane)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncthreads();
    prefetch_ctx(blockIdx.x, 0);

    int it = 0;
    for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x, ++it) {
        const int64_t q0 = grp * kWarps;
        float* scr_all = scr_buf + (d.nbuf == 2 ? (it & 1) : 0) * kWarps * d.scr_floats;
        // ---- phase 1: features of query q0 + warp (warp-private; overlaps other warps' sorts)
        {
            float* scr = scr_all + warp * d.scr_floats;
            const int64_t q = q0 + warp;
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
            const QueryCtx& qc = s_qc[(it & 1) * kWarps + warp];
            prefetch_ctx(grp + gridDim.x, (it + 1) & 1);  // next group's context lands during this one
            if (q >= n || (SS_DEBUG(d) & 1)) {
                for (int i = lane; i < 3 * d.ntot; i += 32) scr[i] = 0.0f;
            } else if (recs != nullptr) {
                if (!qc.ok && lane == 0) atomicExch(err, 1);
                const bool same_light = qc.same_light != 0;
                for (int i = lane; i < d.ntot; i += 32) {
                    float rho, tr, ph;
                    point_features<kPh>(sc, ht, qc, i, d, planes, pre, same_light, rho, tr, ph);
                    scr[i] = rho;
                    scr[d.ntot + i] = tr;
                    scr[2 * d.ntot + i] = ph;
                }
            } else {
                const float* row = feats + q * d.feat_stride;
                const int n0 = d.npts0, n1 = d.ntot - d.npts0;
                for (int i = lane; i < d.ntot; i += 32)
                    for (int ch = 0; ch < 3; ++ch)
                        scr[ch * d.ntot + i] = i < n0 ? row[ch * n0 + i] : row[3 * n0 + ch * n1 + (i - n0)];
            }
        }
        __syncthreads();
        // ---- phase 2: register sorts, tasks ordered by network size; each thread writes its
        // segment's operand chunks (8 consecutive threads = 8 query rows = one 128-byte line)
        // and pools straight from registers
        const int64_t tile = d.tile0 + q0 / kUmmaM;
        const int row0 = int(q0 % kUmmaM);
        const bool store = !(SS_DEBUG(d) & 4);
        for (int t = threadIdx.x; t < ((SS_DEBUG(d) & 2) ? 0 : d.n_tasks * kWarps); t += blockDim.x) {
            const int task = s_task[t / kWarps];
            const int sg = task & 0x7f;
            const int cnt = s_n[sg];
            const bool pair = cnt > 32;
            // a 64-wide segment owns two task slots = 16 threads: (query w, half) = (t%16 / 2, t & 1)
            const int w = pair ? (t % (2 * kWarps)) >> 1 : t % kWarps;
            SegOut o;
            o.f16 = d.f16;
            o.kf = s_kf[sg];
            o.blk = ops + int64_t(s_prefix[sg]) * d.n_tiles + tile * (int64_t(kUmmaM) * o.kf * 2);
            o.row = row0 + w;
            o.tau = sg % 3;
            o.mm = mms + (int64_t(sg / 3) * q_pad + qg0 + q0 + w) * 8;
            const float* seg = scr_all + w * d.scr_floats + s_scr[sg];
            if (pair)
                cnt == 48 ? sort_emit_pair<24>(seg, cnt, t & 1, o, store)
                          : sort_emit_pair<32>(seg, cnt, t & 1, o, store);
            else if (cnt <= 8)
                cnt <= 6 ? sort_emit<8, 6>(seg, cnt, o, store) : sort_emit<8>(seg, cnt, o, store);
            else if (cnt <= 16)
                cnt <= 12 ? sort_emit<16, 12>(seg, cnt, o, store) : sort_emit<16>(seg, cnt, o, store);
            else
                cnt <= 24 ? sort_emit<32, 24>(seg, cnt, o, store) : sort_emit<32>(seg, cnt, o, store);
        }
        if (d.nbuf == 1) __syncthreads();  // the next group's sampling overwrites this scratch
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__global__ void k_blend_planes(const float* __restrict__ T, int G, int A, int H, int n_planes, double g0, double g1,
                               double g2, float* __restrict__ out) {
    const int total = n_planes * A * (H + 1);
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int k = idx / (A * (H + 1)), ah = idx % (A * (H + 1)), h = min(ah % (H + 1), H - 1), a = ah / (H + 1);
        const double g = k == 0 ? g0 : (k == 1 ? g1 : g2);
        int gi;
        double gt;
        table_coord(g, -0.99, 0.99, G, gi, gt);  // PhaseTable::lookup_hg's g axis (src/phase.cpp:196-205)
        const float* t0 = T + (size_t(gi) * A + a) * H + h;
        const float* t1 = t0 + size_t(A) * H;
        out[idx] = float((1.0 - gt) * double(t0[0]) + gt * double(t1[0]));  // the pad column repeats h = H - 1
    }
}

SortDesc make_desc(const SceneDev* sc, int n_planes, const SortLayout& L, int64_t n) {
    SortDesc d{};
    d.npts0 = L.npts[0];
    d.ntot = L.npts[0] + L.npts[1];
    d.n_layers = L.n_layers;
    d.n_tiles = int((n + kUmmaM - 1) / kUmmaM);
    d.tile0 = 0;
    d.n_groups = 0;  // set by the launcher for the chosen block shape
    d.feat_stride = 3 * int64_t(d.ntot);
    if (sc) {
        d.A = sc->phase.ar;
        d.H = sc->phase.hr;
        d.su = float(double(d.A - 1) / kPi);
        d.sv = float(d.H - 1) / float(kPi);
        d.n_planes = n_planes;
        if (sc->phase.kind == SF_PHASE_ISOTROPIC) {
            d.w[0] = 1.0f;
        } else {
            for (int k = 0; k < n_planes; ++k) d.w[k] = float(sc->phase.w[k]);
        }
    }
    int segs = 0, chunks = 0;
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < L.nl[k]; ++i)
            for (int tau = 0; tau < 3; ++tau) {
                if (segs >= kMaxSegs) fail(SF_ERR_INVALID_ARGUMENT, "sample_sort: too many layers");
                const int ch = tau == 0 ? 0 : (tau == 1 ? 2 : 1);  // {density, phase, transmittance}
                d.seg_scr[segs] = ch * d.ntot + (k == 0 ? 0 : L.npts[0]) + L.start[k][i];
                d.seg_n[segs] = L.counts[k][i];
                d.seg_kf[segs] = L.kf[k][i];
                d.seg_prefix[segs] = L.seg_prefix[k][i][tau];
                for (int j = 0; j < L.kf[k][i] / 8; ++j) {
                    if (chunks >= kMaxChunks) fail(SF_ERR_INVALID_ARGUMENT, "sample_sort: too many chunks");
                    d.chunk_seg[chunks] = uint8_t(segs);
                    d.chunk_j[chunks] = uint8_t(j);
                    ++chunks;
                }
                ++segs;
            }
    d.n_segs = segs;
    d.n_chunks = chunks;
    // Sort tasks, one slot = one network size for the group's queries (a warp of the 32-warp
    // block runs one slot; 64-wide segments take two slots as lane pairs, aligned to an even
    // slot). Slots beyond the block's threads run as a second round on the threads of the
    // first slots, so the light 16-wide tasks go first (their threads also take the
    // second-round 32/8-wide tasks), then the lane pairs (the longest), then 32 and 8.
    auto net = [](int c) { return c <= 8 ? 8 : c <= 16 ? 16 : c <= 32 ? 32 : 64; };
    std::vector<int> small, rest;
    for (int s2 = 0; s2 < segs; ++s2)
        if (net(d.seg_n[s2]) == 16) small.push_back(s2);
    int t = 0;
    for (size_t k = 0; k + (small.size() & 1) < small.size(); ++k) d.task_seg[t++] = uint8_t(small[k]);
    for (int s2 = 0; s2 < segs; ++s2)
        if (net(d.seg_n[s2]) == 64) {
            d.task_seg[t++] = uint8_t(s2);
            d.task_seg[t++] = uint8_t(s2 | 0x80);
        }
    if (small.size() & 1) d.task_seg[t++] = uint8_t(small.back());  // keeps the pairs on even slots
    for (int p : {32, 8})
        for (int s2 = 0; s2 < segs; ++s2)
            if (net(d.seg_n[s2]) == p) d.task_seg[t++] = uint8_t(s2);
    d.n_tasks = t;
    d.scr_floats = (3 * d.ntot) | 1;  // odd row stride: 8 query rows hit 8 banks
    if (const char* e = std::getenv("SF_DEBUG_SAMPLE_SORT")) d.debug = std::atoi(e);
    return d;
}

}  // namespace

void launch_blend_planes(const sf_phase_table& t, const sf_phase_model& m, float* planes, cudaStream_t s) {
    int n_planes = m.kind == SF_PHASE_ISOTROPIC ? 1 : m.n_lobes;
    double g[3] = {0, 0, 0};
    if (m.kind != SF_PHASE_ISOTROPIC)
        for (int k = 0; k < n_planes; ++k) g[k] = m.g[k];
    int total = n_planes * t.a * (t.h + 1);
    k_blend_planes<<<(total + 255) / 256, 256, 0, s>>>(t.d, t.g, t.a, t.h, n_planes, g[0], g[1], g[2], planes);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_xpair(const float* rho, const float* tr, int nx, int ny, int nz, float4* out, cudaStream_t s) {
    const int per_slab = ((nx + 2) >> 1) * (ny + 1);
    const dim3 grid(unsigned((per_slab + kXpairThreads - 1) / kXpairThreads), unsigned((nz + 3) >> 1));
    k_xpair<<<grid, kXpairThreads, 0, s>>>(rho, tr, nx, ny, nz, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_cell_order(const GridDev& g, int64_t n, const double* queries, uint32_t* cells, int* counts, int* perm,
                       cudaStream_t s) {
    if (n <= 0) return;
    if (n >= (int64_t(1) << 31)) fail(SF_ERR_INVALID_ARGUMENT, "cell order: batch too large");
    const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 16));
    SFB_CUDA(cudaMemsetAsync(counts, 0, size_t(kOrderCells) * sizeof(int), s));
    k_cell_key<<<blocks, 256, 0, s>>>(g, n, queries, cells, counts);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    k_cell_tile_scan<<<kOrderCells / 1024, 1024, 0, s>>>(counts);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    k_cell_sum_scan<<<1, kOrderCells / 1024, 0, s>>>(counts);
    SFB_CUDA(cudaGetLastError());
    count_launch();
    k_cell_scatter<<<blocks, 256, 0, s>>>(n, cells, counts, perm);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

size_t query_rec_bytes() { return sizeof(QueryCtx); }

int64_t sample_sort_round_queries() { return int64_t(sm_count()) * (kSortThreadsPerSM / 32); }

// L2 read-bandwidth probe for the sampler's roofline (bench.py): every thread streams 32-byte
// records (the sampler's load width) over an L2-resident buffer, `reps` passes.
__global__ void k_l2_probe(const float4* __restrict__ buf, size_t n32, int reps, float* __restrict__ sink) {
    float acc = 0.0f;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n32; i += stride) {
            float4 a, b;
            // volatile: the compiler may not merge the repeated loads of the `reps` loop
            asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                         : "l"(buf + 2 * i)
                         : "memory");
            acc += a.x + b.w;
        }
    if (acc == 1.2345f) sink[0] = acc;  // never true for the zeroed buffer; keeps the loads live
}

double probe_l2_read_gbs(size_t bytes, int reps) {
    const size_t n32 = bytes / 32;
    float4* buf = nullptr;
    float* sink = nullptr;
    SFB_CUDA(cudaMalloc(&buf, n32 * 32));
    SFB_CUDA(cudaMalloc(&sink, sizeof(float)));
    SFB_CUDA(cudaMemset(buf, 0, n32 * 32));
    cudaEvent_t e0, e1;
    SFB_CUDA(cudaEventCreate(&e0));
    SFB_CUDA(cudaEventCreate(&e1));
    const unsigned grid = unsigned(sm_count()) * 8;
    k_l2_probe<<<grid, 256>>>(buf, n32, 2, sink);  // warm: buffer into L2
    SFB_CUDA(cudaEventRecord(e0));
    k_l2_probe<<<grid, 256>>>(buf, n32, reps, sink);
    SFB_CUDA(cudaEventRecord(e1));
    SFB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.0f;
    SFB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(sink);
    count_launch();
    count_launch();
    return double(n32 * 32) * reps / (double(ms) * 1e-3) / 1e9;
}

// float4 units of the xy-quad layout: padded dims (nx + 1, ny + 1, nz + 2) in whole 2x1x2
// bricks, two float4 per record
size_t xpair_records(int nx, int ny, int nz) {
    return size_t((nx + 2) / 2) * size_t(ny + 1) * ((nz + 3) / 2) * 4 * 2;
}

void launch_query_prep(const SceneDev& sc, const TemplateDev& ht, const sf_medium_params& m, int64_t n,
                       const double* queries, const double* media, double* cfg8, void* recs, cudaStream_t s,
                       const int* perm, const double* row0, const TemplateDev* dt, const float* planes, int n_planes,
                       float4* pre) {
    if (n <= 0) return;
    const int diffuse_blocks = dt ? (dt->total + kPrepThreads - 1) / kPrepThreads : 0;
    SortDesc d{};
    if (dt) {
        SortLayout L{};
        d = make_desc(&sc, n_planes, L, 1);
    }
    const int64_t blocks = std::min<int64_t>((n + kPrepThreads - 1) / kPrepThreads, int64_t(sm_count()) * 16);
    k_query_prep<<<unsigned(blocks + diffuse_blocks), kPrepThreads, 0, s>>>(
        sc, ht, m, n, queries, media, cfg8, static_cast<QueryCtx*>(recs), perm, row0 ? row0 : queries,
        dt ? *dt : TemplateDev{}, d,
        planes, pre, diffuse_blocks);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_sample_sort(const SceneDev* sc, const TemplateDev* dt, const TemplateDev* ht, const float* planes,
                        int n_planes, const float4* pre, const SortLayout& L, int64_t n, const void* recs,
                        const float* feats, uint8_t* ops, float* mms, int* err, cudaStream_t s, bool mixed,
                        int64_t tile0, int64_t layout_tiles, bool f16, bool l2_keep) {
    (void)dt;  // diffuse placement comes from `pre` (k_query_prep's diffuse blocks)
    if (n <= 0) return;
    SortDesc d = make_desc(sc, n_planes, L, n);
    d.f16 = (f16 ? 1 : 0) | (l2_keep ? 2 : 0);
    if (layout_tiles > 0) {  // a window of a larger operand layout
        if (tile0 < 0 || tile0 + d.n_tiles > layout_tiles) fail(SF_ERR_INVALID_ARGUMENT, "sample_sort: tile window");
        d.tile0 = int(tile0);
        d.n_tiles = int(layout_tiles);
    }
    if (mixed && sc) {
        d.mixed = 1;
        d.G = sc->phase.gr;
        d.table = sc->phase.table;
        d.quad = sc->phase.quad;
        if (!d.quad) fail(SF_ERR_INVALID_ARGUMENT, "sample_sort: mixed media need the table's quad records");
        d.w[0] = 1.0f;  // PhaseModel::hg(g): one lobe of weight 1
    }
    auto smem_for = [&](int w, int nbuf) {
        return size_t(d.n_planes * d.A * (d.H + 1) * (SF_PLANE_PAIRS ? 2 : 1) + size_t(nbuf) * w * d.scr_floats) *
                   sizeof(float) +
               2 * size_t(w) * sizeof(QueryCtx) + 16;
    };
    static const size_t static_smem = [] {
        cudaFuncAttributes fa{};
        SFB_CUDA(cudaFuncGetAttributes(&fa, k_sample_sort<kPhMixed, kWBig, kMinBBig>));
        return fa.sharedSizeBytes;
    }();
    // Block shape: 32 warps (one block per SM) when its shared memory fits, else 8 warps x 4.
    // One scratch buffer (two block barriers per group): a second buffer, where it fits,
    // measured slower in every configuration tried; SF_SORT_NBUF=2 forces it
    // when it fits. SF_SORT_WARPS=8 forces the small shape.
    static const int force_w = std::getenv("SF_SORT_WARPS") ? std::atoi(std::getenv("SF_SORT_WARPS")) : 0;
    const size_t budget = 227 * 1024;
    const bool big = force_w != kWSmall && smem_for(kWBig, 1) + static_smem <= budget;
    const int w = big ? kWBig : kWSmall, minb = big ? kMinBBig : kMinBSmall;
    d.nbuf = 1;
    if (const char* e = std::getenv("SF_SORT_NBUF"))
        if (std::atoi(e) == 2 && minb * (smem_for(w, 2) + static_smem + 1024) <= 228 * 1024) d.nbuf = 2;
    const size_t smem = smem_for(w, d.nbuf);
    if (smem + static_smem > budget) fail(SF_ERR_INVALID_ARGUMENT, "sample_sort: templates too large for shared memory");
    const int ph = d.mixed ? kPhMixed : (d.n_planes == 1 ? kPhOne : kPhPlanes);
    auto kern = big ? (ph == kPhMixed ? k_sample_sort<kPhMixed, kWBig, kMinBBig>
                                      : (ph == kPhOne ? k_sample_sort<kPhOne, kWBig, kMinBBig>
                                                      : k_sample_sort<kPhPlanes, kWBig, kMinBBig>))
                    : (ph == kPhMixed ? k_sample_sort<kPhMixed, kWSmall, kMinBSmall>
                                      : (ph == kPhOne ? k_sample_sort<kPhOne, kWSmall, kMinBSmall>
                                                      : k_sample_sort<kPhPlanes, kWSmall, kMinBSmall>));
    if (smem > 48 * 1024)
        // (no carveout preference: the driver's choice from the occupancy need is the fastest)
        SFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int64_t window_tiles = (n + kUmmaM - 1) / kUmmaM;
    d.n_groups = window_tiles * (kUmmaM / w);
    int64_t blocks = d.n_groups;
    const int64_t cap = int64_t(sm_count()) * minb;
    if (blocks > cap) blocks = cap;
    SceneDev scd = sc ? *sc : SceneDev{};
    TemplateDev htd = ht ? *ht : TemplateDev{1, 0, nullptr, nullptr, 1.0, nullptr};
    kern<<<unsigned(blocks), w * 32, smem, s>>>(scd, htd, d, planes, pre, n, static_cast<const QueryCtx*>(recs), feats,
                                                ops, mms, err);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

__global__ void k_phase_quad(const float* __restrict__ t, int G, int A, int H, float4* __restrict__ q) {
    const int64_t n = int64_t(G) * A * H;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int h = int(i % H), a = int((i / H) % A), g = int(i / (int64_t(A) * H));
        const int h1 = min(h + 1, H - 1), g1 = min(g + 1, G - 1);
        const float* p0 = t + (int64_t(g) * A + a) * H;
        const float* p1 = t + (int64_t(g1) * A + a) * H;
        q[i] = make_float4(p0[h], p0[h1], p1[h], p1[h1]);
    }
}

const float4* phase_quad(const sf_phase_table& t, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(t.quad_mu);
    if (!t.d_quad) {
        const size_t n = size_t(t.g) * t.a * t.h;
        SFB_CUDA(cudaMalloc(&t.d_quad, n * sizeof(float4)));
        k_phase_quad<<<unsigned(std::min<size_t>((n + 255) / 256, 65535)), 256, 0, s>>>(t.d, t.g, t.a, t.h, t.d_quad);
        SFB_CUDA(cudaGetLastError());
        count_launch();
        // once per table: complete before any stream (not only `s`) may read the records
        SFB_CUDA(cudaStreamSynchronize(s));
    }
    return t.d_quad;
}

}  // namespace sfb
