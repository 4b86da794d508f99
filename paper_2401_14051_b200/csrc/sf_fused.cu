// sf_fused.cu — production front half of the query: per shading point, sample
// the 266 template features, sort/pool every (layer, feature type) and emit the
// tensor-core operands directly (K5 + K6 fused; features never reach HBM).
//
// One warp per query. Lanes evaluate template points (density + transmittance
// from the interleaved float2 volume, the Eq. 8 phase feature from pre-blended
// phase planes held in shared memory), the warp then sorts each layer segment
// descending with a 64-wide bitonic network over shuffles, sums it in sorted order
// (one lane per segment, so mean = sequential float sum / n exactly as
// src/predictor.cpp:176-185), and writes
//   * the bf16 FC-1 feature operand rows [sorted_tau, mean_tau, max_tau, 0...] of
//     every (kind, layer, tau) straight into the UMMA canonical layout of its
//     128-query tile, and
//   * the fp32 {mean, max} x 3 types row of every (kind, layer) for the attention.
//
// Numerics (bf16 production path only; the FP32 parity path keeps the exact
// kernels of sf_query.cu): positions, voxel coordinates and cell selection in
// FP64 as the reference, interpolation weights and lerps in FP32, phase angles and
// the phase-table bilinear in FP32 (survey: <= 3.2e-6 relative), all far inside
// the bf16 rounding (3.9e-3) the operands undergo.
#include <algorithm>

#include "sf_internal.h"
#include "sf_umma.cuh"

namespace sfb {

namespace {

constexpr int kWarps = 8;
constexpr int kMaxSegs = 96;
constexpr int kMaxChunks = 512;

struct SortDesc {
    int npts0, ntot;
    int n_segs, n_layers, n_chunks;
    int n_tiles;
    int64_t feat_stride;
    int A, H, n_planes;
    float w[3];
    int scr_floats;
    // per segment (kind, layer, tau)
    int seg_scr[kMaxSegs];  // offset of the segment in the warp scratch
    int seg_n[kMaxSegs];
    int seg_kf[kMaxSegs];
    int64_t seg_prefix[kMaxSegs];
    // per output chunk (16 B = 8 bf16 of one row)
    uint8_t chunk_seg[kMaxChunks];
    uint8_t chunk_j[kMaxChunks];
    uint8_t task_seg[kMaxSegs];  // segments ordered by sorting-network size
};

// Bilinear lookup in a pre-blended phase plane stored as aperture pairs
// pl[a][h] = {P(a,h), P(a,h+1)}: two 8-byte shared loads per lookup.
__device__ __forceinline__ float plane_lookup(const float2* pl, int A, int H, float angle, float half) {
    float u = fminf(fmaxf(angle, 0.0f), float(kPi)) * (float(A - 1) / float(kPi));
    int i0 = min(int(u), A - 2);
    float t = u - float(i0);
    float v = fminf(fmaxf(half, 0.0f), float(kPi)) * (float(H - 1) / float(kPi));
    int j0 = min(int(v), H - 2);
    float s = v - float(j0);
    const float2 r0 = pl[i0 * (H + 1) + j0];  // rows padded to H+1 pairs: no bank aliasing
    const float2 r1 = pl[(i0 + 1) * (H + 1) + j0];
    float a = fmaf(s, r0.y - r0.x, r0.x);
    float b = fmaf(s, r1.y - r1.x, r1.x);
    return fmaf(t, b - a, a);
}

__device__ __forceinline__ float cap_phase(const float2* planes, int n_planes, const float* w, int A, int H,
                                           float angle, float half) {
    float f = 0.0f;
    for (int k = 0; k < n_planes; ++k) f = fmaf(w[k], plane_lookup(planes + k * A * (H + 1), A, H, angle, half), f);
    return f;
}

struct QueryCtx {
    double p[3], entry[3], axis[3], t[3], b[3];
    double hscale;
    float wf[3], lf[3];
    float ww, ll;
    bool ok;
};

__device__ __forceinline__ void query_ctx(const SceneDev& sc, const TemplateDev& ht, const double* c, QueryCtx& q) {
    const double p[3] = {c[0], c[1], c[2]}, omega[3] = {c[3], c[4], c[5]}, light[3] = {c[6], c[7], c[8]};
    for (int i = 0; i < 3; ++i) {
        q.p[i] = p[i];
        q.wf[i] = float(omega[i]);
        q.lf[i] = float(light[i]);
    }
    q.ww = q.wf[0] * q.wf[0] + q.wf[1] * q.wf[1] + q.wf[2] * q.wf[2];
    q.ll = q.lf[0] * q.lf[0] + q.lf[1] * q.lf[1] + q.lf[2] * q.lf[2];
    // light entry + highlight frame (src/feature_pipeline.cpp:130-137, src/templates.cpp:220-239)
    const double lo[3] = {sc.grid.ox, sc.grid.oy, sc.grid.oz};
    const double hi[3] = {sc.grid.hx, sc.grid.hy, sc.grid.hz};
    light_entry(lo, hi, p, light, q.entry);
    double span[3] = {p[0] - q.entry[0], p[1] - q.entry[1], p[2] - q.entry[2]};
    double len = sqrt(dot3(span, span));
    q.ok = len > 0.0;
    double il = 1.0 / len;
    for (int i = 0; i < 3; ++i) q.axis[i] = span[i] * il;
    double od = dot3(omega, q.axis);
    double t[3] = {omega[0] - q.axis[0] * od, omega[1] - q.axis[1] * od, omega[2] - q.axis[2] * od};
    double tl = sqrt(dot3(t, t));
    if (tl > 1e-9) {
        double it = 1.0 / tl;
        for (int i = 0; i < 3; ++i) q.t[i] = t[i] * it;
        q.b[0] = q.axis[1] * q.t[2] - q.axis[2] * q.t[1];
        q.b[1] = q.axis[2] * q.t[0] - q.axis[0] * q.t[2];
        q.b[2] = q.axis[0] * q.t[1] - q.axis[1] * q.t[0];
    } else {
        orthonormal_basis(q.axis, q.t, q.b);
    }
    q.hscale = len / ht.gen_distance;
}

// density, transmittance and phase feature of template point i (0..ntot)
__device__ __forceinline__ void point_features(const SceneDev& sc, const TemplateDev& dt, const TemplateDev& ht,
                                               const QueryCtx& q, int i, int npts0, const float2* planes,
                                               const float2* pre, bool use_pre, const SortDesc& d, float& rho,
                                               float& tr, float& ph) {
    double s[3];
    double cap;
    if (i < npts0) {
        const double* qq = dt.pts + 3 * i;
        for (int c = 0; c < 3; ++c) s[c] = q.p[c] + qq[c] * sc.template_scale;
        cap = dt.caps[i] * sc.template_scale;
    } else {
        const int li = i - npts0;
        const double* qq = ht.pts + 3 * li;
        for (int c = 0; c < 3; ++c) {
            double v = q.t[c] * qq[0] + q.b[c] * qq[1];
            v = v + q.axis[c] * qq[2];
            s[c] = q.entry[c] + v * q.hscale;
        }
        cap = ht.caps[li] * q.hscale;
    }
    const GridDev& g = sc.grid;
    if (!in_box(g, s[0], s[1], s[2])) {
        rho = 0.0f;
        tr = 1.0f;
    } else {
        // FP64 cell selection exactly as sample_trilinear; FP32 weights and lerps.
        // x-pair records hold {rho, T} at x0 and clamp(x0 + 1): one 16-byte load per
        // (y, z) corner row; a cell clamped at the low x edge has tx forced to 0.
        double fx, fy, fz;
        if (g.ivs != 0.0) {
            fx = (s[0] - g.ox) * g.ivs - 0.5;
            fy = (s[1] - g.oy) * g.ivs - 0.5;
            fz = (s[2] - g.oz) * g.ivs - 0.5;
        } else {
            fx = (s[0] - g.ox) / g.vs - 0.5;
            fy = (s[1] - g.oy) / g.vs - 0.5;
            fz = (s[2] - g.oz) / g.vs - 0.5;
        }
        const double flx = floor(fx), fly = floor(fy), flz = floor(fz);
        int x0 = int(flx), y0 = int(fly), z0 = int(flz);
        float tx = float(fx - flx), ty = float(fy - fly), tz = float(fz - flz);
        if (x0 < 0) tx = 0.0f;
        const int y1 = clampi(y0 + 1, 0, g.ny - 1), z1 = clampi(z0 + 1, 0, g.nz - 1);
        x0 = clampi(x0, 0, g.nx - 1);
        y0 = clampi(y0, 0, g.ny - 1);
        z0 = clampi(z0, 0, g.nz - 1);
        const size_t sy = size_t(g.nx), sz = size_t(g.nx) * g.ny;
        const float4* v = sc.dt4 + x0;
        const float4 r00 = __ldg(v + z0 * sz + y0 * sy), r10 = __ldg(v + z0 * sz + y1 * sy);
        const float4 r01 = __ldg(v + z1 * sz + y0 * sy), r11 = __ldg(v + z1 * sz + y1 * sy);
        float c00 = fmaf(tx, r00.z - r00.x, r00.x), c10 = fmaf(tx, r10.z - r10.x, r10.x);
        float c01 = fmaf(tx, r01.z - r01.x, r01.x), c11 = fmaf(tx, r11.z - r11.x, r11.x);
        float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
        rho = fmaf(tz, e1 - e0, e0);
        c00 = fmaf(tx, r00.w - r00.y, r00.y);
        c10 = fmaf(tx, r10.w - r10.y, r10.y);
        c01 = fmaf(tx, r01.w - r01.y, r01.y);
        c11 = fmaf(tx, r11.w - r11.y, r11.y);
        e0 = fmaf(ty, c10 - c00, c00);
        e1 = fmaf(ty, c11 - c01, c01);
        tr = fmaf(tz, e1 - e0, e0);
    }
    const float dx = float(s[0] - q.p[0]), dy = float(s[1] - q.p[1]), dz = float(s[2] - q.p[2]);
    const float dd = dx * dx + dy * dy + dz * dz;
    if (dd <= 0.0f) {
        ph = 1.0f;  // diffuse centre point (src/feature_pipeline.cpp:163-164)
        return;
    }
    const float inv = rsqrtf(dd);
    const float ax = dx * inv, ay = dy * inv, az = dz * inv;
    const float aa = ax * ax + ay * ay + az * az;
    const float cw = (q.wf[0] * ax + q.wf[1] * ay + q.wf[2] * az) * rsqrtf(q.ww * aa);
    const float aw = acosf(fminf(fmaxf(cw, -1.0f), 1.0f));
    float half, fl;
    if (use_pre && i < npts0) {
        const float2 pr = pre[i];  // translation-invariant diffuse aperture and light side
        half = pr.x;
        fl = pr.y;
    } else {
        const float capf = float(cap), dist = dd * inv;
        half = capf >= dist ? float(kPi) : asinf(capf / dist);
        const float cl = (q.lf[0] * ax + q.lf[1] * ay + q.lf[2] * az) * rsqrtf(q.ll * aa);
        fl = cap_phase(planes, d.n_planes, d.w, d.A, d.H, acosf(fminf(fmaxf(cl, -1.0f), 1.0f)), half);
    }
    ph = cap_phase(planes, d.n_planes, d.w, d.A, d.H, aw, half) * fl;
}

// pre[i] = {half angle, light-side cap integral} of diffuse point i for the light of
// query 0 (axis = q_i/|q_i| and aperture asin(cap/|q_i ts|) do not depend on p).
__global__ void k_diffuse_light(SceneDev sc, TemplateDev dt, SortDesc d, const float2* __restrict__ planes,
                                const double* __restrict__ queries, float2* __restrict__ pre) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dt.total) return;
    const double* qq = dt.pts + 3 * i;
    const double ts = sc.template_scale;
    const float dx = float(qq[0] * ts), dy = float(qq[1] * ts), dz = float(qq[2] * ts);
    const float dd = dx * dx + dy * dy + dz * dz;
    if (dd <= 0.0f) {
        pre[i] = make_float2(float(kPi), 1.0f);
        return;
    }
    const float inv = rsqrtf(dd), dist = dd * inv;
    const float ax = dx * inv, ay = dy * inv, az = dz * inv;
    const float aa = ax * ax + ay * ay + az * az;
    const float capf = float(dt.caps[i] * ts);
    const float half = capf >= dist ? float(kPi) : asinf(capf / dist);
    const float lx = float(queries[6]), ly = float(queries[7]), lz = float(queries[8]);
    const float ll = lx * lx + ly * ly + lz * lz;
    const float cl = (lx * ax + ly * ay + lz * az) * rsqrtf(ll * aa);
    pre[i] = make_float2(half, cap_phase(planes, d.n_planes, d.w, d.A, d.H,
                                         acosf(fminf(fmaxf(cl, -1.0f), 1.0f)), half));
}

__global__ void k_xpair(const float2* __restrict__ v, int nx, int ny, int nz, float4* __restrict__ out) {
    const size_t n = size_t(nx) * ny * nz;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const int x = int(i % nx);
        const float2 a = v[i], b = v[x + 1 < nx ? i + 1 : i];
        out[i] = make_float4(a.x, a.y, b.x, b.y);
    }
}

// Descending bitonic network on P (power of two) register values; all indices are
// compile-time so the segment never leaves registers.
template <int P>
__device__ __forceinline__ void bitonic_desc(float* v) {
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
                    if ((i & k) == 0) {
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

// Sort one segment (cnt <= P values at seg) in registers, write it back sorted and
// return mean (sequential float sum in sorted order / cnt) and max.
template <int P>
__device__ __forceinline__ void sort_segment(float* seg, int cnt, float& mean, float& mx) {
    float v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = j < cnt ? seg[j] : -INFINITY;
    bitonic_desc<P>(v);
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < P; ++j)
        if (j < cnt) acc += v[j];
#pragma unroll
    for (int j = 0; j < P; ++j)
        if (j < cnt) seg[j] = v[j];
    mean = acc / float(cnt);
    mx = v[0];
}

// Block = 8 consecutive queries (one 8-row group of a UMMA tile).
//  phase 1: warp w samples the 266 template points of query q0 + w (point-parallel,
//           so a warp's gathers stay inside one template's footprint);
//  phase 2: thread-per-(query, segment) register sorts, tasks ordered by network
//           size so a warp runs one network;
//  phase 3: the 8 rows of every 16-byte operand chunk are 128 contiguous bytes of
//           the canonical layout, so each warp store is fully coalesced.
__global__ void __launch_bounds__(kWarps * 32, 3)
    k_sample_sort(SceneDev sc, TemplateDev dt, TemplateDev ht, SortDesc d, const float2* __restrict__ planes_g,
                  const float2* __restrict__ pre, int64_t n, const double* __restrict__ queries,
                  const float* __restrict__ feats, uint8_t* __restrict__ ops, float* __restrict__ mms, int* err) {
    extern __shared__ __align__(16) float sm[];
    const int plane_floats = 2 * d.n_planes * d.A * (d.H + 1);
    float2* planes = reinterpret_cast<float2*>(sm);
    for (int i = threadIdx.x; i < plane_floats / 2; i += blockDim.x) planes[i] = planes_g[i];
    // segment / chunk tables in shared memory (lane-divergent indices would serialize
    // constant-bank loads)
    __shared__ int s_scr[kMaxSegs], s_n[kMaxSegs], s_kf[kMaxSegs];
    __shared__ int64_t s_prefix[kMaxSegs];
    __shared__ uint8_t s_cseg[kMaxChunks], s_cj[kMaxChunks], s_task[kMaxSegs];
    for (int i = threadIdx.x; i < d.n_segs; i += blockDim.x) {
        s_scr[i] = d.seg_scr[i];
        s_n[i] = d.seg_n[i];
        s_kf[i] = d.seg_kf[i];
        s_prefix[i] = d.seg_prefix[i];
        s_task[i] = d.task_seg[i];
    }
    for (int i = threadIdx.x; i < d.n_chunks; i += blockDim.x) {
        s_cseg[i] = d.chunk_seg[i];
        s_cj[i] = d.chunk_j[i];
    }
    // light of query 0: diffuse light sides in `pre` are valid for queries with that light
    double l_ref[3] = {0, 0, 0};
    if (queries != nullptr && n > 0)
        for (int c = 0; c < 3; ++c) l_ref[c] = queries[6 + c];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* scr_all = sm + plane_floats;                        // [8][scr_floats]
    float* pools = scr_all + kWarps * d.scr_floats;            // [8][n_segs][2]
    const int64_t q_pad = int64_t(d.n_tiles) * kUmmaM;
    const int64_t n_groups = q_pad / kWarps;
    __syncthreads();

    for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
        const int64_t q0 = grp * kWarps;
        // ---- phase 1: features
        {
            float* scr = scr_all + warp * d.scr_floats;
            const int64_t q = q0 + warp;
            if (q >= n) {
                for (int i = lane; i < 3 * d.ntot; i += 32) scr[i] = 0.0f;
            } else if (feats == nullptr) {
                QueryCtx qc;
                const double* qr = queries + 9 * q;
                query_ctx(sc, ht, qr, qc);
                if (!qc.ok && lane == 0) atomicExch(err, 1);
                const bool use_pre = pre != nullptr && qr[6] == l_ref[0] && qr[7] == l_ref[1] && qr[8] == l_ref[2];
                for (int i = lane; i < d.ntot; i += 32) {
                    float rho, tr, ph;
                    point_features(sc, dt, ht, qc, i, d.npts0, planes, pre, use_pre, d, rho, tr, ph);
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
        // ---- phase 2: per-(query, segment) register sorts + pools
        for (int t = threadIdx.x; t < d.n_segs * kWarps; t += blockDim.x) {
            const int s = s_task[t / kWarps], w = t % kWarps;
            float* seg = scr_all + w * d.scr_floats + s_scr[s];
            const int cnt = s_n[s];
            float mean, mx;
            if (cnt <= 8)
                sort_segment<8>(seg, cnt, mean, mx);
            else if (cnt <= 16)
                sort_segment<16>(seg, cnt, mean, mx);
            else if (cnt <= 32)
                sort_segment<32>(seg, cnt, mean, mx);
            else
                sort_segment<64>(seg, cnt, mean, mx);
            pools[(w * d.n_segs + s) * 2] = mean;
            pools[(w * d.n_segs + s) * 2 + 1] = mx;
        }
        __syncthreads();
        // ---- phase 3: outputs
        const int64_t tile = q0 / kUmmaM;
        const int row0 = int(q0 % kUmmaM);
        for (int t = threadIdx.x; t < d.n_chunks * kWarps; t += blockDim.x) {
            const int c = t / kWarps, w = t % kWarps;
            const int s = s_cseg[c], j = s_cj[c];
            const float* seg = scr_all + w * d.scr_floats + s_scr[s];
            const float* pl = pools + (w * d.n_segs + s) * 2;
            const int cnt = s_n[s], kf = s_kf[s];
            float v8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int idx = 8 * j + e;
                v8[e] = idx < cnt ? seg[idx] : (idx == cnt ? pl[0] : (idx == cnt + 1 ? pl[1] : 0.0f));
            }
            uint8_t* blk = ops + s_prefix[s] * d.n_tiles + tile * (int64_t(kUmmaM) * kf * 2);
            store_chunk(blk, row0 + w, j, kf, v8);
        }
        for (int t = threadIdx.x; t < d.n_layers * kWarps; t += blockDim.x) {
            const int l = t / kWarps, w = t % kWarps;
            const float* pl = pools + (w * d.n_segs + 3 * l) * 2;  // segments 3l + tau
            float4* o = reinterpret_cast<float4*>(mms + (int64_t(l) * q_pad + q0 + w) * 8);
            o[0] = make_float4(pl[0], pl[2], pl[4], pl[1]);
            o[1] = make_float4(pl[3], pl[5], 0.0f, 0.0f);
        }
        __syncthreads();
    }
}

__global__ void k_blend_planes(const float* __restrict__ T, int G, int A, int H, int n_planes, double g0, double g1,
                               double g2, float2* __restrict__ out) {
    const int total = n_planes * A * H;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int k = idx / (A * H), ah = idx % (A * H), h = ah % H, a = ah / H;
        const double g = k == 0 ? g0 : (k == 1 ? g1 : g2);
        int gi;
        double gt;
        table_coord(g, -0.99, 0.99, G, gi, gt);  // PhaseTable::lookup_hg's g axis (src/phase.cpp:196-205)
        const float* t0 = T + size_t(gi) * A * H + ah;
        const float* t1 = t0 + size_t(A) * H;
        const int dh = h + 1 < H ? 1 : 0;
        const float v0 = float((1.0 - gt) * double(t0[0]) + gt * double(t1[0]));
        const float v1 = float((1.0 - gt) * double(t0[dh]) + gt * double(t1[dh]));
        out[(k * A + a) * (H + 1) + h] = make_float2(v0, v1);
    }
}

SortDesc make_desc(const SceneDev* sc, int n_planes, const SortLayout& L, int64_t n) {
    SortDesc d{};
    d.npts0 = L.npts[0];
    d.ntot = L.npts[0] + L.npts[1];
    d.n_layers = L.n_layers;
    d.n_tiles = int((n + kUmmaM - 1) / kUmmaM);
    d.feat_stride = 3 * int64_t(d.ntot);
    if (sc) {
        d.A = sc->phase.ar;
        d.H = sc->phase.hr;
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
    auto net = [](int c) { return c <= 8 ? 8 : c <= 16 ? 16 : c <= 32 ? 32 : 64; };
    int t = 0;
    for (int p : {64, 32, 16, 8})
        for (int s2 = 0; s2 < segs; ++s2)
            if (net(d.seg_n[s2]) == p) d.task_seg[t++] = uint8_t(s2);
    // odd row stride: the 8 query rows of a sort task group hit 8 different banks
    d.scr_floats = (3 * d.ntot) | 1;
    return d;
}

}  // namespace

void launch_blend_planes(const sf_phase_table& t, const sf_phase_model& m, float* planes, cudaStream_t s) {
    int n_planes = m.kind == SF_PHASE_ISOTROPIC ? 1 : m.n_lobes;
    double g[3] = {0, 0, 0};
    if (m.kind != SF_PHASE_ISOTROPIC)
        for (int k = 0; k < n_planes; ++k) g[k] = m.g[k];
    int total = n_planes * t.a * t.h;
    k_blend_planes<<<(total + 255) / 256, 256, 0, s>>>(t.d, t.g, t.a, t.h, n_planes, g[0], g[1], g[2],
                                                        reinterpret_cast<float2*>(planes));
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_xpair(const float2* dt, int nx, int ny, int nz, float4* out, cudaStream_t s) {
    const size_t n = size_t(nx) * ny * nz;
    k_xpair<<<unsigned(std::min<size_t>((n + 255) / 256, size_t(sm_count()) * 32)), 256, 0, s>>>(dt, nx, ny, nz,
                                                                                                 out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_diffuse_light(const SceneDev& sc, const TemplateDev& dt, const float* planes, int n_planes,
                          const double* queries, float2* pre, cudaStream_t s) {
    SortLayout L{};
    SortDesc d = make_desc(&sc, n_planes, L, 1);
    k_diffuse_light<<<(dt.total + 127) / 128, 128, 0, s>>>(sc, dt, d, reinterpret_cast<const float2*>(planes),
                                                           queries, pre);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_sample_sort(const SceneDev* sc, const TemplateDev* dt, const TemplateDev* ht, const float* planes,
                        int n_planes, const float2* pre, const SortLayout& L, int64_t n, const double* queries,
                        const float* feats, uint8_t* ops, float* mms, int* err, cudaStream_t s) {
    if (n <= 0) return;
    SortDesc d = make_desc(sc, n_planes, L, n);
    const size_t smem = size_t(2 * d.n_planes * d.A * (d.H + 1) + kWarps * d.scr_floats + kWarps * d.n_segs * 2 + 2) *
                        sizeof(float);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        SFB_CUDA(cudaFuncSetAttribute(k_sample_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = smem;
    }
    const int64_t q_pad = int64_t(d.n_tiles) * kUmmaM;
    int64_t blocks = q_pad / kWarps;
    int64_t cap = int64_t(sm_count()) * 3;
    if (blocks > cap) blocks = cap;
    SceneDev scd = sc ? *sc : SceneDev{};
    TemplateDev dtd = dt ? *dt : TemplateDev{};
    TemplateDev htd = ht ? *ht : TemplateDev{1, 0, nullptr, nullptr, 1.0};
    k_sample_sort<<<unsigned(blocks), kWarps * 32, smem, s>>>(scd, dtd, htd, d,
                                                              reinterpret_cast<const float2*>(planes), pre, n,
                                                              queries, feats, ops, mms, err);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
