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

__device__ __forceinline__ void warp_sort64_desc(float& v0, float& v1, int lane) {
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                float a = fmaxf(v0, v1), b = fminf(v0, v1);
                v0 = a;
                v1 = b;
            } else {
                float o0 = __shfl_xor_sync(0xffffffffu, v0, j);
                float o1 = __shfl_xor_sync(0xffffffffu, v1, j);
                const bool lower = (lane & j) == 0;
                const bool d0 = (lane & k) == 0, d1 = ((lane + 32) & k) == 0;
                v0 = (lower == d0) ? fmaxf(v0, o0) : fminf(v0, o0);
                v1 = (lower == d1) ? fmaxf(v1, o1) : fminf(v1, o1);
            }
        }
    }
}

__device__ __forceinline__ float plane_lookup(const float* pl, int A, int H, float angle, float half) {
    float u = fminf(fmaxf(angle, 0.0f), float(kPi)) * (float(A - 1) / float(kPi));
    int i0 = min(int(u), A - 2);
    float t = u - float(i0);
    float v = fminf(fmaxf(half, 0.0f), float(kPi)) * (float(H - 1) / float(kPi));
    int j0 = min(int(v), H - 2);
    float s = v - float(j0);
    const float* r0 = pl + i0 * H + j0;
    const float* r1 = r0 + H;
    float a = fmaf(s, r0[1] - r0[0], r0[0]);
    float b = fmaf(s, r1[1] - r1[0], r1[0]);
    return fmaf(t, b - a, a);
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
                                               const QueryCtx& q, int i, int npts0, const float* planes,
                                               const SortDesc& d, float& rho, float& tr, float& ph) {
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
        Cell c = cell_of(g, s[0], s[1], s[2]);
        const float tx = float(c.tx), ty = float(c.ty), tz = float(c.tz);
        const size_t sy = size_t(g.nx), sz = size_t(g.nx) * g.ny;
        const float2* v = sc.dt;
        float2 a000 = __ldg(v + c.z0 * sz + c.y0 * sy + c.x0), a100 = __ldg(v + c.z0 * sz + c.y0 * sy + c.x1);
        float2 a010 = __ldg(v + c.z0 * sz + c.y1 * sy + c.x0), a110 = __ldg(v + c.z0 * sz + c.y1 * sy + c.x1);
        float2 a001 = __ldg(v + c.z1 * sz + c.y0 * sy + c.x0), a101 = __ldg(v + c.z1 * sz + c.y0 * sy + c.x1);
        float2 a011 = __ldg(v + c.z1 * sz + c.y1 * sy + c.x0), a111 = __ldg(v + c.z1 * sz + c.y1 * sy + c.x1);
        float c00 = fmaf(tx, a100.x - a000.x, a000.x), c10 = fmaf(tx, a110.x - a010.x, a010.x);
        float c01 = fmaf(tx, a101.x - a001.x, a001.x), c11 = fmaf(tx, a111.x - a011.x, a011.x);
        float e0 = fmaf(ty, c10 - c00, c00), e1 = fmaf(ty, c11 - c01, c01);
        rho = fmaf(tz, e1 - e0, e0);
        c00 = fmaf(tx, a100.y - a000.y, a000.y);
        c10 = fmaf(tx, a110.y - a010.y, a010.y);
        c01 = fmaf(tx, a101.y - a001.y, a001.y);
        c11 = fmaf(tx, a111.y - a011.y, a011.y);
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
    const float dist = sqrtf(dd);
    const float capf = float(cap);
    const float half = capf >= dist ? float(kPi) : asinf(capf / dist);
    const float inv = 1.0f / dist;
    const float ax = dx * inv, ay = dy * inv, az = dz * inv;
    const float aa = ax * ax + ay * ay + az * az;
    float cw = (q.wf[0] * ax + q.wf[1] * ay + q.wf[2] * az) * rsqrtf(q.ww * aa);
    float cl = (q.lf[0] * ax + q.lf[1] * ay + q.lf[2] * az) * rsqrtf(q.ll * aa);
    const float aw = acosf(fminf(fmaxf(cw, -1.0f), 1.0f));
    const float al = acosf(fminf(fmaxf(cl, -1.0f), 1.0f));
    float fw = 0.0f, fl = 0.0f;
    for (int k = 0; k < d.n_planes; ++k) {
        const float* pl = planes + k * d.A * d.H;
        fw = fmaf(d.w[k], plane_lookup(pl, d.A, d.H, aw, half), fw);
        fl = fmaf(d.w[k], plane_lookup(pl, d.A, d.H, al, half), fl);
    }
    ph = fw * fl;
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
    k_sample_sort(SceneDev sc, TemplateDev dt, TemplateDev ht, SortDesc d, const float* __restrict__ planes_g,
                  int64_t n, const double* __restrict__ queries, const float* __restrict__ feats,
                  uint8_t* __restrict__ ops, float* __restrict__ mms, int* err) {
    extern __shared__ __align__(16) float sm[];
    const int plane_floats = d.n_planes * d.A * d.H;
    for (int i = threadIdx.x; i < plane_floats; i += blockDim.x) sm[i] = planes_g[i];
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
                query_ctx(sc, ht, queries + 9 * q, qc);
                if (!qc.ok && lane == 0) atomicExch(err, 1);
                for (int i = lane; i < d.ntot; i += 32) {
                    float rho, tr, ph;
                    point_features(sc, dt, ht, qc, i, d.npts0, sm, d, rho, tr, ph);
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
            const int s = d.task_seg[t / kWarps], w = t % kWarps;
            float* seg = scr_all + w * d.scr_floats + d.seg_scr[s];
            const int cnt = d.seg_n[s];
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
            const int s = d.chunk_seg[c], j = d.chunk_j[c];
            const float* seg = scr_all + w * d.scr_floats + d.seg_scr[s];
            const float* pl = pools + (w * d.n_segs + s) * 2;
            const int cnt = d.seg_n[s], kf = d.seg_kf[s];
            float v8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int idx = 8 * j + e;
                v8[e] = idx < cnt ? seg[idx] : (idx == cnt ? pl[0] : (idx == cnt + 1 ? pl[1] : 0.0f));
            }
            uint8_t* blk = ops + d.seg_prefix[s] * d.n_tiles + tile * (int64_t(kUmmaM) * kf * 2);
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
                               double g2, float* __restrict__ out) {
    int total = n_planes * A * H;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        int k = idx / (A * H), ah = idx % (A * H);
        double g = k == 0 ? g0 : (k == 1 ? g1 : g2);
        int gi;
        double gt;
        table_coord(g, -0.99, 0.99, G, gi, gt);
        out[idx] = float((1.0 - gt) * double(T[size_t(gi) * A * H + ah]) + gt * double(T[size_t(gi + 1) * A * H + ah]));
    }
}

}  // namespace

void launch_blend_planes(const sf_phase_table& t, const sf_phase_model& m, float* planes, cudaStream_t s) {
    int n_planes = m.kind == SF_PHASE_ISOTROPIC ? 1 : m.n_lobes;
    double g[3] = {0, 0, 0};
    if (m.kind != SF_PHASE_ISOTROPIC)
        for (int k = 0; k < n_planes; ++k) g[k] = m.g[k];
    int total = n_planes * t.a * t.h;
    k_blend_planes<<<(total + 255) / 256, 256, 0, s>>>(t.d, t.g, t.a, t.h, n_planes, g[0], g[1], g[2], planes);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_sample_sort(const SceneDev* sc, const TemplateDev* dt, const TemplateDev* ht, const float* planes,
                        int n_planes, const SortLayout& L, int64_t n, const double* queries, const float* feats,
                        uint8_t* ops, float* mms, int* err, cudaStream_t s) {
    if (n <= 0) return;
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
    {
        auto net = [](int c) { return c <= 8 ? 8 : c <= 16 ? 16 : c <= 32 ? 32 : 64; };
        int t = 0;
        for (int p : {64, 32, 16, 8})
            for (int s2 = 0; s2 < segs; ++s2)
                if (net(d.seg_n[s2]) == p) d.task_seg[t++] = uint8_t(s2);
    }
    d.scr_floats = (3 * d.ntot + 3) / 4 * 4;
    const size_t smem =
        size_t(d.n_planes * d.A * d.H + kWarps * d.scr_floats + kWarps * segs * 2) * sizeof(float);
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
    k_sample_sort<<<unsigned(blocks), kWarps * 32, smem, s>>>(scd, dtd, htd, d, planes, n, queries, feats, ops,
                                                              mms, err);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
