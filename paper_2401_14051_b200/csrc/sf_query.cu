// sf_query.cu — per-shading-point kernels: template placement + feature
// sampling (K5), per-layer sort / pool (K6), the FP32 SIMT backbone forward that
// reproduces the reference's sequential FP32 arithmetic (K7-fp32), and decode.
//
// The feature kernel gathers density and transmittance from ONE interleaved
// float2 level-0 volume ({rho, T} share the lattice, src/feature_pipeline.cpp:
// 107-112 and :159-160), so each trilinear corner is a single 8-byte load; the
// phase table (1 MiB at 64x128x32) stays L2-resident.
#include <algorithm>
#include <mutex>

#include "sf_internal.h"
#include "sf_exact.cuh"

namespace sfb {

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(size_t n, int block = kBlock) {
    size_t g = (n + block - 1) / block;
    return unsigned(g > 0x7fffffff ? 0x7fffffff : (g == 0 ? 1 : g));
}

// K5: sample_features (src/feature_pipeline.cpp:139-172) for a batch of queries.
// Thread = (query, template point); output rows are SoA per block:
// out[q*row_stride + col_offset + {0,1,2}*total + i] = {density, trans, phase}.
__global__ void k_sample_features(SceneDev sc, TemplateDev td, int64_t n,
                                  const double* __restrict__ queries, const double* __restrict__ media,
                                  float* __restrict__ out, int64_t row_stride, int64_t col_offset, int* err) {
    int64_t total = int64_t(n) * td.total;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        int64_t qi = idx / td.total;
        int i = int(idx - qi * td.total);
        float* o = out + qi * row_stride + col_offset;
        float rho, tr, f;
        if (!exact_point_features(sc, td, i, queries + 9 * qi, media ? media + 4 * qi : nullptr, rho, tr, f)) {
            atomicExch(err, 1);
            o[i] = o[td.total + i] = o[2 * td.total + i] = __int_as_float(0x7fc00000);
            continue;
        }
        o[i] = rho;
        o[td.total + i] = tr;
        o[2 * td.total + i] = f;
    }
}

__global__ void k_place_template(SceneDev sc, TemplateDev td, int64_t n,
                                 const double* __restrict__ p, const double* __restrict__ omega,
                                 const double* __restrict__ entry, double* __restrict__ pts,
                                 double* __restrict__ caps, int* err) {
    int64_t total = int64_t(n) * td.total;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        int64_t qi = idx / td.total;
        int i = int(idx - qi * td.total);
        const double* pq = p + 3 * qi;
        const double* q = td.pts + 3 * i;
        double* s = pts + 3 * idx;
        if (td.kind == 0) {
            for (int c = 0; c < 3; ++c) s[c] = pq[c] + q[c] * sc.template_scale;
            caps[idx] = td.caps[i] * sc.template_scale;
            continue;
        }
        const double* e = entry + 3 * qi;
        const double* w = omega + 3 * qi;
        double span[3] = {pq[0] - e[0], pq[1] - e[1], pq[2] - e[2]};
        double len = sqrt(dot3(span, span));
        if (len <= 0.0) {
            atomicExch(err, 1);
            continue;
        }
        double il = 1.0 / len;
        double axis[3] = {span[0] * il, span[1] * il, span[2] * il};
        double od = dot3(w, axis);
        double t[3] = {w[0] - axis[0] * od, w[1] - axis[1] * od, w[2] - axis[2] * od};
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
        for (int c = 0; c < 3; ++c) {
            double v = t[c] * q[0] + b[c] * q[1];
            v = v + axis[c] * q[2];
            s[c] = e[c] + v * scale;
        }
        caps[idx] = td.caps[i] * scale;
    }
}

// ---- sort / pool (src/predictor.cpp:153-191) --------------------------------------
constexpr int kMaxSegs = 96;
constexpr int kMaxLayerPoints = 64;
struct SegTable {
    int n_segs;
    int n[kMaxSegs];        // points in the layer
    int src[kMaxSegs];      // column of the first value in the feature row
    int dst[kMaxSegs];      // slice offset of the sorted run (then mean, max)
};

// K6: one thread per (query, kind, layer, tau); insertion sort descending, then
// float mean in sorted order and max = first element. Slices are stored
// [slice_col][query] so the backbone's per-query reads coalesce across a warp.
__global__ void k_slice(SegTable st, int64_t n, int64_t feat_stride,
                        const float* __restrict__ feats, float* __restrict__ slices) {
    int64_t total = n * st.n_segs;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        int64_t q = idx % n;
        int seg = int(idx / n);
        int cnt = st.n[seg];
        const float* src = feats + q * feat_stride + st.src[seg];
        float a[kMaxLayerPoints];
        for (int j = 0; j < cnt; ++j) {
            float v = src[j];
            int k = j - 1;
            while (k >= 0 && a[k] < v) {
                a[k + 1] = a[k];
                --k;
            }
            a[k + 1] = v;
        }
        float acc = 0.0f;
        for (int j = 0; j < cnt; ++j) acc += a[j];
        float* dst = slices + int64_t(st.dst[seg]) * n + q;
        for (int j = 0; j < cnt; ++j) dst[int64_t(j) * n] = a[j];
        dst[int64_t(cnt) * n] = acc / float(cnt);
        dst[int64_t(cnt + 1) * n] = a[0];
    }
}

// ---- FP32 backbone (src/predictor.cpp:206-235, 352-409; src/neural.cpp:86-122) ------
struct NetDesc {
    int nl[2];
    int counts[2][16];
    int slice_off[2][16];  // slice column of (kind, layer) group
    int W, M, H;
    int literal;
    double gamma;
    int64_t stack_off[2][3];
    int64_t merge_off, cross_off, head_off[3];
};

__device__ __forceinline__ float relu(float v) { return (v < 0.0f) ? 0.0f : v; }
// 1/(1+exp(-v)) in float; exp rounded from FP64 so it matches the correctly
// rounded expf of the CPU reference (src/neural.cpp:190-193).
__device__ __forceinline__ float sigmoid_ref(float v) {
    return 1.0f / (1.0f + float(exp(double(-v))));
}

// Tape<float>::dense: acc = b; acc += w*x (no contraction; built --fmad=false).
template <int MAXM>
__device__ __forceinline__ void dense_f32(const float* __restrict__ W, const float* __restrict__ b,
                                          int m, int n, const float* x, float* y) {
    for (int i = 0; i < m; ++i) {
        float acc = __ldg(b + i);
        const float* row = W + int64_t(i) * n;
        for (int j = 0; j < n; ++j) acc += __ldg(row + j) * x[j];
        y[i] = acc;
    }
}

__device__ void run_stack_f32(const NetDesc& nd, const float* __restrict__ P, int k, int tau,
                              const float* cfgv, const float* __restrict__ slices, int64_t n,
                              int64_t q, float g_mean, float alpha, float* o_out) {
    const int W = nd.W;
    int64_t off = nd.stack_off[k][tau];
    float o[64], o_att[64], u[64], t2[64], x[160];
    dense_f32<64>(P + off, P + off + W * 7, W, 7, cfgv, o);
    off += W * 7 + W;
    for (int j = 0; j < W; ++j) o[j] = relu(o[j]);
    for (int i = 0; i < nd.nl[k]; ++i) {
        const int cnt = nd.counts[k][i];
        const float* sl = slices + int64_t(nd.slice_off[k][i]) * n + q;
        // tau blocks of (cnt + 2): sorted, mean, max
        float v[8];
        for (int t = 0; t < 3; ++t) {
            v[t] = sl[int64_t(t * (cnt + 2) + cnt) * n];
            v[3 + t] = sl[int64_t(t * (cnt + 2) + cnt + 1) * n];
        }
        v[6] = g_mean;
        v[7] = alpha;
        float w;
        if (nd.literal) {
            float acc = 0.0f;
            for (int j = 0; j < 8; ++j) acc += (v[j] < 0.0f) ? 0.0f : v[j];
            w = sigmoid_ref(acc / 8.0f);
        } else {
            float h[4], w3[3];
            dense_f32<4>(P + off, P + off + 32, 4, 8, v, h);
            for (int j = 0; j < 4; ++j) h[j] = relu(h[j]);
            dense_f32<3>(P + off + 36, P + off + 48, 3, 4, h, w3);
            w = sigmoid_ref(w3[tau]);
            off += 51;
        }
        for (int j = 0; j < W; ++j) o_att[j] = o[j] * w;
        const int K = W + cnt + 2;
        for (int j = 0; j < W; ++j) x[j] = o_att[j];
        const float* st = sl + int64_t(tau * (cnt + 2)) * n;
        for (int j = 0; j < cnt + 2; ++j) x[W + j] = st[int64_t(j) * n];
        dense_f32<64>(P + off, P + off + int64_t(W) * K, W, K, x, u);
        off += int64_t(W) * K + W;
        for (int j = 0; j < W; ++j) u[j] = relu(u[j]);
        dense_f32<64>(P + off, P + off + W * W, W, W, u, t2);
        off += W * W + W;
        for (int j = 0; j < W; ++j) o[j] = relu(t2[j]) + o_att[j];
    }
    for (int j = 0; j < W; ++j) o_out[j] = o[j];
}

__global__ void __launch_bounds__(128) k_backbone_fp32(NetDesc nd, const float* __restrict__ P,
                                                       int64_t n, const float* __restrict__ slices,
                                                       const double* __restrict__ cfg8,
                                                       float* __restrict__ y_out,
                                                       double* __restrict__ F_out) {
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x) {
        const double* c8 = cfg8 + 8 * q;
        int ng = int(c8[0]);
        float g_mean = 0.0f;
        for (int i = 0; i < ng; ++i) g_mean += float(c8[1 + i]);
        if (ng > 0) g_mean /= float(double(ng));
        float alpha = float(c8[7]);
        float cfgv[7] = {0.0f, 0.0f, 0.0f, float(c8[4]), float(c8[5]), float(c8[6]), float(c8[7])};
        for (int i = 0; i < ng && i < 3; ++i) cfgv[i] = float(c8[1 + i]);
        const int W = nd.W, M = nd.M, H = nd.H;
        float merged[3 * 128], cat[128], od[64], oh[64], h1[128], h2[128], y[3];
        for (int t = 0; t < 3; ++t) {
            run_stack_f32(nd, P, 0, t, cfgv, slices, n, q, g_mean, alpha, od);
            run_stack_f32(nd, P, 1, t, cfgv, slices, n, q, g_mean, alpha, oh);
            for (int j = 0; j < W; ++j) {
                cat[j] = od[j];
                cat[W + j] = oh[j];
            }
            const float* mW = P + nd.merge_off + int64_t(t) * (int64_t(M) * 2 * W + M);
            dense_f32<128>(mW, mW + int64_t(M) * 2 * W, M, 2 * W, cat, merged + t * M);
            for (int j = 0; j < M; ++j) merged[t * M + j] = relu(merged[t * M + j]);
        }
        dense_f32<128>(P + nd.cross_off, P + nd.cross_off + int64_t(M) * 3 * M, M, 3 * M, merged,
                       h1);
        for (int j = 0; j < M; ++j) h1[j] = relu(h1[j]);
        dense_f32<128>(P + nd.head_off[0], P + nd.head_off[0] + int64_t(H) * M, H, M, h1, h2);
        for (int j = 0; j < H; ++j) h2[j] = relu(h2[j]);
        dense_f32<128>(P + nd.head_off[1], P + nd.head_off[1] + int64_t(H) * H, H, H, h2, h1);
        for (int j = 0; j < H; ++j) h1[j] = relu(h1[j]);
        dense_f32<3>(P + nd.head_off[2], P + nd.head_off[2] + 3 * H, 3, H, h1, y);
        for (int c = 0; c < 3; ++c) {
            y[c] = fabsf(y[c]);
            if (y_out) y_out[3 * q + c] = y[c];
            // decode_prediction (src/predictor.cpp:406-409)
            if (F_out) F_out[3 * q + c] = pow(c8[4 + c], nd.gamma) * expm1(double(y[c]));
        }
    }
}

// Exact FP32 backbone, warp-cooperative: a warp runs kQPW queries, lane j owns output
// neurons j and j + 32 of every dense layer. Each neuron is still accumulated in the
// reference's order (acc = b; acc += w * x over the inputs in order, src/neural.cpp:95-101,
// no contraction), so the results are those of k_backbone_fp32; what changes is the
// parallelism (32 lanes per query instead of one thread) and the weight traffic: weights
// are read transposed ([in][out], one coalesced 128-byte row per input) once per warp for
// kQPW queries. Widths <= 64.
constexpr int kQPW = 4;
constexpr int kXs = 200;  // per-query input buffer (fc1 <= 32 + 64 + 2, cross 3M <= 192)

struct Acc2 {
    float v[kQPW][2];
};

// acc[q][h] = b[j] + sum_k WT[k][j] * x[q][k] for j = lane + 32 h < m (exact order)
__device__ __forceinline__ void dense_warp(const float* __restrict__ WT, const float* __restrict__ b, int m, int K,
                                           const float (*x)[kXs], int lane, Acc2& acc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const float bj = j < m ? __ldg(b + j) : 0.0f;
#pragma unroll
        for (int q = 0; q < kQPW; ++q) acc.v[q][h] = bj;
    }
    for (int k = 0; k < K; ++k) {
        const float w0 = lane < m ? __ldg(WT + int64_t(k) * m + lane) : 0.0f;
        const float w1 = lane + 32 < m ? __ldg(WT + int64_t(k) * m + lane + 32) : 0.0f;
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {
            const float xk = x[q][k];
            acc.v[q][0] += w0 * xk;
            acc.v[q][1] += w1 * xk;
        }
    }
}

__global__ void __launch_bounds__(128) k_backbone_fp32w(NetDesc nd, const float* __restrict__ P,
                                                        const float* __restrict__ PT, int64_t n,
                                                        const float* __restrict__ slices,
                                                        const double* __restrict__ cfg8, float* __restrict__ y_out,
                                                        double* __restrict__ F_out) {
    __shared__ float xs_all[4][2][kQPW][kXs];  // [warp][ping-pong][query][input]
    __shared__ float keep_all[4][kQPW][3 * 64 + 2 * 64];  // merged (3M) then od | oh (2W)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float(*xa)[kXs] = xs_all[warp][0];
    float(*xb)[kXs] = xs_all[warp][1];
    float(*keep)[3 * 64 + 2 * 64] = keep_all[warp];
    const int W = nd.W, M = nd.M, H = nd.H;
    const int64_t n_warps = (n + kQPW - 1) / kQPW;
    for (int64_t wi = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; wi < n_warps;
         wi += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int64_t q0 = wi * kQPW;
        float cfgv[kQPW][7], g_mean[kQPW], alpha[kQPW];
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {  // cfg_vector (src/predictor.cpp:193-202); padded rows repeat the last
            const int64_t qq = q0 + q < n ? q0 + q : n - 1;
            const double* c8 = cfg8 + 8 * qq;
            const int ng = int(c8[0]);
            g_mean[q] = 0.0f;
            for (int i = 0; i < ng; ++i) g_mean[q] += float(c8[1 + i]);
            if (ng > 0) g_mean[q] /= float(double(ng));
            alpha[q] = float(c8[7]);
            for (int i = 0; i < 3; ++i) cfgv[q][i] = i < ng ? float(c8[1 + i]) : 0.0f;
            for (int i = 0; i < 4; ++i) cfgv[q][3 + i] = float(c8[4 + i]);
        }
        for (int t = 0; t < 3; ++t) {
            for (int k = 0; k < 2; ++k) {
                int64_t off = nd.stack_off[k][t];
                // conditioning layer o = relu(W_init cfg + b) (run_stack, src/predictor.cpp:206-212)
#pragma unroll
                for (int q = 0; q < kQPW; ++q)
                    if (lane < 7) xa[q][lane] = cfgv[q][lane];
                __syncwarp();
                Acc2 o;
                dense_warp(PT + off, P + off + W * 7, W, 7, xa, lane, o);
                off += W * 7 + W;
#pragma unroll
                for (int q = 0; q < kQPW; ++q) {
                    o.v[q][0] = relu(o.v[q][0]);
                    o.v[q][1] = relu(o.v[q][1]);
                }
                for (int i = 0; i < nd.nl[k]; ++i) {
                    const int cnt = nd.counts[k][i];
                    float wq[kQPW];
#pragma unroll
                    for (int q = 0; q < kQPW; ++q) {  // channel attention, redundantly per lane
                        const int64_t qq = q0 + q < n ? q0 + q : n - 1;
                        const float* sl = slices + int64_t(nd.slice_off[k][i]) * n + qq;
                        float v[8];
                        for (int c = 0; c < 3; ++c) {
                            v[c] = sl[int64_t(c * (cnt + 2) + cnt) * n];
                            v[3 + c] = sl[int64_t(c * (cnt + 2) + cnt + 1) * n];
                        }
                        v[6] = g_mean[q];
                        v[7] = alpha[q];
                        if (nd.literal) {
                            float acc = 0.0f;
                            for (int j = 0; j < 8; ++j) acc += (v[j] < 0.0f) ? 0.0f : v[j];
                            wq[q] = sigmoid_ref(acc / 8.0f);
                        } else {
                            float hh[4], w3[3];
                            dense_f32<4>(P + off, P + off + 32, 4, 8, v, hh);
                            for (int j = 0; j < 4; ++j) hh[j] = relu(hh[j]);
                            dense_f32<3>(P + off + 36, P + off + 48, 3, 4, hh, w3);
                            wq[q] = sigmoid_ref(w3[t]);
                        }
                    }
                    if (!nd.literal) off += 51;
                    // fc1 input [o_att | sorted_tau, mean, max]
                    Acc2 oa;
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < kQPW; ++q) {
                        const int64_t qq = q0 + q < n ? q0 + q : n - 1;
                        oa.v[q][0] = o.v[q][0] * wq[q];
                        oa.v[q][1] = o.v[q][1] * wq[q];
                        if (lane < W) xa[q][lane] = oa.v[q][0];
                        if (lane + 32 < W) xa[q][lane + 32] = oa.v[q][1];
                        const float* st = slices + int64_t(nd.slice_off[k][i] + t * (cnt + 2)) * n + qq;
                        for (int j = lane; j < cnt + 2; j += 32) xa[q][W + j] = st[int64_t(j) * n];
                    }
                    __syncwarp();
                    const int K = W + cnt + 2;
                    Acc2 u;
                    dense_warp(PT + off, P + off + int64_t(W) * K, W, K, xa, lane, u);
                    off += int64_t(W) * K + W;
#pragma unroll
                    for (int q = 0; q < kQPW; ++q) {
                        if (lane < W) xb[q][lane] = relu(u.v[q][0]);
                        if (lane + 32 < W) xb[q][lane + 32] = relu(u.v[q][1]);
                    }
                    __syncwarp();
                    Acc2 t2;
                    dense_warp(PT + off, P + off + W * W, W, W, xb, lane, t2);
                    off += W * W + W;
#pragma unroll
                    for (int q = 0; q < kQPW; ++q) {
                        o.v[q][0] = relu(t2.v[q][0]) + oa.v[q][0];
                        o.v[q][1] = relu(t2.v[q][1]) + oa.v[q][1];
                    }
                }
                // od (k = 0) / oh (k = 1) -> the merge input [od | oh]
#pragma unroll
                for (int q = 0; q < kQPW; ++q) {
                    if (lane < W) keep[q][3 * 64 + k * W + lane] = o.v[q][0];
                    if (lane + 32 < W) keep[q][3 * 64 + k * W + lane + 32] = o.v[q][1];
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < kQPW; ++q)
                for (int j = lane; j < 2 * W; j += 32) xa[q][j] = keep[q][3 * 64 + j];
            __syncwarp();
            const int64_t mo = nd.merge_off + int64_t(t) * (int64_t(M) * 2 * W + M);
            Acc2 mg;
            dense_warp(PT + mo, P + mo + int64_t(M) * 2 * W, M, 2 * W, xa, lane, mg);
#pragma unroll
            for (int q = 0; q < kQPW; ++q) {
                if (lane < M) keep[q][t * M + lane] = relu(mg.v[q][0]);
                if (lane + 32 < M) keep[q][t * M + lane + 32] = relu(mg.v[q][1]);
            }
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < kQPW; ++q)
            for (int j = lane; j < 3 * M; j += 32) xa[q][j] = keep[q][j];
        __syncwarp();
        Acc2 h;
        dense_warp(PT + nd.cross_off, P + nd.cross_off + int64_t(M) * 3 * M, M, 3 * M, xa, lane, h);
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {
            if (lane < M) xb[q][lane] = relu(h.v[q][0]);
            if (lane + 32 < M) xb[q][lane + 32] = relu(h.v[q][1]);
        }
        __syncwarp();
        dense_warp(PT + nd.head_off[0], P + nd.head_off[0] + int64_t(H) * M, H, M, xb, lane, h);
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {
            if (lane < H) xa[q][lane] = relu(h.v[q][0]);
            if (lane + 32 < H) xa[q][lane + 32] = relu(h.v[q][1]);
        }
        __syncwarp();
        dense_warp(PT + nd.head_off[1], P + nd.head_off[1] + int64_t(H) * H, H, H, xa, lane, h);
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {
            if (lane < H) xb[q][lane] = relu(h.v[q][0]);
            if (lane + 32 < H) xb[q][lane + 32] = relu(h.v[q][1]);
        }
        __syncwarp();
        dense_warp(PT + nd.head_off[2], P + nd.head_off[2] + 3 * H, 3, H, xb, lane, h);
#pragma unroll
        for (int q = 0; q < kQPW; ++q) {
            const int64_t qq = q0 + q;
            if (lane < 3 && qq < n) {
                const float yc = fabsf(h.v[q][0]);
                if (y_out) y_out[3 * qq + lane] = yc;
                // decode_prediction (src/predictor.cpp:406-409)
                if (F_out) F_out[3 * qq + lane] = pow(cfg8[8 * qq + 4 + lane], nd.gamma) * expm1(double(yc));
            }
        }
        __syncwarp();
    }
}

// make_config (src/predictor.cpp:261-274): g params + albedo of the medium,
// alpha = angle_between(omega, light) per query.
__global__ void k_make_cfg8(sf_medium_params m, int64_t n, const double* __restrict__ queries,
                            const double* __restrict__ media, double* __restrict__ cfg8) {
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x) {
        const double* c = queries + 9 * q;
        double* o = cfg8 + 8 * q;
        write_cfg8(m, media ? media + 4 * q : nullptr, c, o);
    }
}

}  // namespace

SceneDev scene_dev(const sf_grid& density, const sf_grid& tvol, const float2* dt,
                   const sf_phase_model& m, const sf_phase_table& t, double ts) {
    SceneDev s{};
    s.grid = density.dev();
    s.dt = dt;
    s.tvol = tvol.d;
    s.phase.kind = m.kind;
    s.phase.n_lobes = m.n_lobes;
    for (int k = 0; k < 3; ++k) {
        s.phase.w[k] = m.weight[k];
        s.phase.g[k] = m.g[k];
    }
    s.phase.table = t.d;
    s.phase.gr = t.g;
    s.phase.ar = t.a;
    s.phase.hr = t.h;
    s.phase.quad = t.d_quad;
    s.template_scale = ts;
    return s;
}

TemplateDev template_dev(const sf_template& t) {
    return TemplateDev{t.kind, t.total, t.d_points, t.d_caps, t.gen_distance, t.d_pts4};
}

void launch_sample_features(const SceneDev& sc, const TemplateDev& td, int64_t n,
                            const double* queries, const double* media, float* out, int64_t row_stride,
                            int64_t col_offset, int* err, cudaStream_t s) {
    if (n <= 0) return;
    k_sample_features<<<grid_for(size_t(n) * td.total, 128), 128, 0, s>>>(
        sc, td, n, queries, media, out, row_stride, col_offset, err);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_place_template(const sf_template& t, int64_t n, const double* p,
                           const double* omega, const double* entry, double ts, double* pts,
                           double* caps, int* err, cudaStream_t s) {
    if (n <= 0) return;
    SceneDev sc{};
    sc.template_scale = ts;
    k_place_template<<<grid_for(size_t(n) * t.total), kBlock, 0, s>>>(sc, template_dev(t), n, p,
                                                                       omega, entry, pts, caps, err);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

int64_t slices_per_query(const sf_backbone_config& c) {
    int64_t s = 0;
    for (int i = 0; i < c.n_diffuse_layers; ++i) s += 3 * (c.diffuse_counts[i] + 2);
    for (int i = 0; i < c.n_highlight_layers; ++i) s += 3 * (c.highlight_counts[i] + 2);
    return s;
}

static void seg_table(const sf_backbone_config& c, SegTable& st, NetDesc* nd) {
    st.n_segs = 0;
    int nd_total = 0, nh_total = 0;
    for (int i = 0; i < c.n_diffuse_layers; ++i) nd_total += c.diffuse_counts[i];
    for (int i = 0; i < c.n_highlight_layers; ++i) nh_total += c.highlight_counts[i];
    int dst = 0;
    for (int k = 0; k < 2; ++k) {
        int nl = k == 0 ? c.n_diffuse_layers : c.n_highlight_layers;
        const int* counts = k == 0 ? c.diffuse_counts : c.highlight_counts;
        int ntot = k == 0 ? nd_total : nh_total;
        int base = k == 0 ? 0 : 3 * nd_total;
        int start = 0;
        for (int i = 0; i < nl; ++i) {
            if (nd) nd->slice_off[k][i] = dst;
            for (int tau = 0; tau < 3; ++tau) {
                // tau order {density, phase, transmittance}; feature channels are
                // {density, transmittance, phase} (src/predictor.cpp:168-169).
                int ch = tau == 0 ? 0 : (tau == 1 ? 2 : 1);
                if (st.n_segs >= kMaxSegs) fail(SF_ERR_INVALID_ARGUMENT, "too many template layers");
                st.n[st.n_segs] = counts[i];
                st.src[st.n_segs] = base + ch * ntot + start;
                st.dst[st.n_segs] = dst;
                ++st.n_segs;
                dst += counts[i] + 2;
            }
            start += counts[i];
        }
    }
}

void launch_slice(const sf_backbone_config& c, int64_t n, const float* feats, float* slices,
                  cudaStream_t s) {
    if (n <= 0) return;
    for (int i = 0; i < c.n_diffuse_layers; ++i)
        if (c.diffuse_counts[i] > kMaxLayerPoints) fail(SF_ERR_INVALID_ARGUMENT, "layer too large");
    for (int i = 0; i < c.n_highlight_layers; ++i)
        if (c.highlight_counts[i] > kMaxLayerPoints) fail(SF_ERR_INVALID_ARGUMENT, "layer too large");
    SegTable st{};
    seg_table(c, st, nullptr);
    int64_t stride = 0;
    for (int i = 0; i < c.n_diffuse_layers; ++i) stride += 3 * c.diffuse_counts[i];
    for (int i = 0; i < c.n_highlight_layers; ++i) stride += 3 * c.highlight_counts[i];
    k_slice<<<grid_for(size_t(n) * st.n_segs), kBlock, 0, s>>>(st, n, stride, feats, slices);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

// d_paramsT: the canonical parameters with every dense W [out][in] of the backbone stored
// transposed [in][out] at the same offset (biases and attention records unchanged), built
// once per backbone on first FP32 use.
static void prepare_transposed(sf_backbone& b, const NetDesc& nd, cudaStream_t s) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (b.d_paramsT) return;
    std::vector<float> P(size_t(b.layout.total)), T;
    SFB_CUDA(cudaMemcpyAsync(P.data(), b.d_params, P.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
    SFB_CUDA(cudaStreamSynchronize(s));
    T = P;
    auto tr = [&](int64_t off, int rows, int cols) {  // W [rows][cols] -> [cols][rows]
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) T[size_t(off + int64_t(c) * rows + r)] = P[size_t(off + int64_t(r) * cols + c)];
    };
    const int W = nd.W, M = nd.M, H = nd.H;
    for (int k = 0; k < 2; ++k)
        for (int t = 0; t < 3; ++t) {  // walk_params order (src/predictor.cpp:62-109)
            int64_t off = nd.stack_off[k][t];
            tr(off, W, 7);
            off += W * 7 + W;
            for (int i = 0; i < nd.nl[k]; ++i) {
                if (!nd.literal) off += 51;
                const int K = W + nd.counts[k][i] + 2;
                tr(off, W, K);
                off += int64_t(W) * K + W;
                tr(off, W, W);
                off += W * W + W;
            }
        }
    for (int t = 0; t < 3; ++t) tr(nd.merge_off + int64_t(t) * (int64_t(M) * 2 * W + M), M, 2 * W);
    tr(nd.cross_off, M, 3 * M);
    tr(nd.head_off[0], H, M);
    tr(nd.head_off[1], H, H);
    tr(nd.head_off[2], 3, H);
    float* d = nullptr;
    SFB_CUDA(cudaMalloc(&d, T.size() * sizeof(float)));
    SFB_CUDA(cudaMemcpy(d, T.data(), T.size() * sizeof(float), cudaMemcpyHostToDevice));
    b.d_paramsT = d;
}

void launch_backbone_fp32(const sf_backbone& b, int64_t n, const float* slices,
                          const double* cfg8, float* y, double* F, cudaStream_t s) {
    if (n <= 0) return;
    const sf_backbone_config& c = b.cfg;
    if (c.width > 64 || c.merge_width > 128 || c.head_width > 128)
        fail(SF_ERR_INVALID_ARGUMENT, "fp32 backbone: width>64 or merge/head width>128 unsupported");
    NetDesc nd{};
    SegTable st{};
    seg_table(c, st, &nd);
    nd.nl[0] = c.n_diffuse_layers;
    nd.nl[1] = c.n_highlight_layers;
    for (int i = 0; i < 16; ++i) {
        nd.counts[0][i] = c.diffuse_counts[i];
        nd.counts[1][i] = c.highlight_counts[i];
    }
    nd.W = c.width;
    nd.M = c.merge_width;
    nd.H = c.head_width;
    nd.literal = c.literal_attention;
    nd.gamma = c.gamma;
    for (int k = 0; k < 2; ++k)
        for (int t = 0; t < 3; ++t) nd.stack_off[k][t] = b.layout.stack_off[k][t];
    nd.merge_off = b.layout.merge_off;
    nd.cross_off = b.layout.cross_off;
    for (int l = 0; l < 3; ++l) nd.head_off[l] = b.layout.head_off[l];
    if (c.width <= 64 && c.merge_width <= 64 && c.head_width <= 64) {  // warp-cooperative kernel
        prepare_transposed(const_cast<sf_backbone&>(b), nd, s);
        const int64_t warps = (n + kQPW - 1) / kQPW;
        const int64_t blocks = std::min<int64_t>((warps + 3) / 4, int64_t(sm_count()) * 16);
        k_backbone_fp32w<<<unsigned(blocks), 128, 0, s>>>(nd, b.d_params, b.d_paramsT, n, slices, cfg8, y, F);
    } else {
        k_backbone_fp32<<<grid_for(size_t(n), 128), 128, 0, s>>>(nd, b.d_params, n, slices, cfg8, y, F);
    }
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_make_cfg8(const sf_medium_params& m, int64_t n, const double* queries, const double* media,
                      double* cfg8, cudaStream_t s) {
    if (n <= 0) return;
    k_make_cfg8<<<grid_for(size_t(n)), kBlock, 0, s>>>(m, n, queries, media, cfg8);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
