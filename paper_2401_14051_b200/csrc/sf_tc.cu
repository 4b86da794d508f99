// sf_tc.cu — the backbone forward on 5th-generation tensor cores (tcgen05).
//
// One CTA = one tile of 128 shading points = UMMA_M. Thread t owns query row t,
// which is also TMEM lane t, so each epilogue is a private tcgen05.ld of the
// thread's own accumulator row. The reference network (src/predictor.cpp:206-235,
// 352-387) becomes a chain of tcgen05.mma GEMMs D[128 x N] (fp32, TMEM) = A * W^T:
//
//   FC-1  = [o_att | sorted_tau, mean, max] W1^T as two MMAs into one accumulator:
//           A_att (K=32, written by the threads) x W1[:, :32]  +
//           F     (K=pad16(n+2), bulk-copied, produced by k_sample_sort) x W1[:, 32:]
//   FC-2  (N=32, K=32), per-type merge (N=64, K=64), cross merge accumulated
//   chunk by chunk as each merged_tau appears (3 x K=64), head 0/1 (N=64, K=64).
//
// The reference's W[out][in] row-major is exactly UMMA's K-major B operand, so
// weights are packed once (tc_prepare) into the no-swizzle canonical layout.
// Everything a step needs — its weight blob, the tile's sorted-feature operand
// block and mean/max block, and the step's small FP32 SIMT parameters (attention
// 8->4->3, biases, the 7->32 conditioning layer, the 64->3 output layer) — is one
// bundle of cp.async.bulk copies into a 3-slot SMEM ring completing on one
// mbarrier; bundle j+2 is in flight while step j runs, so no global load sits on
// the per-layer critical path. The step program lives in the kernel parameters.
//
// Precision: bf16 GEMM operands (weights, o_att, features, u, merges), fp32
// accumulation, fp32 bias / activation / residual / attention (tests/bf16_emulation.py).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "sf_internal.h"
#include "sf_umma.cuh"

namespace sfb {

namespace {

constexpr int kThreads = 128;   // one thread per query row / TMEM lane
constexpr int kTmemCols = 256;  // fc1 [0,32) fc2 [32,64) merge/head [64,128) cross [128,192)
constexpr int kSlots = 3;
constexpr int kSlotBytes = 28672;
// FC-1 bundle layout
constexpr int kSlotW1a = 0, kSlotW1b = 2048, kSlotFeat = 6144, kSlotMM = 22528;
constexpr int kSlotAtt = 26624;   // [52] attention W1 b1 W2 b2 (+pad), [32] FC-1 bias
constexpr int kSlotInit = 27136;  // [224] conditioning W, [32] b (first layer of a stack)
// 64-wide bundles: weights at 0, bias at 8192, head2 W/b at 8448 (head-1 bundle)
constexpr int kSlotBias = 8192, kSlotHead2 = 8448;
constexpr int kMaxSteps = 96;
constexpr int kMaxCopies = 6;

struct Copy {
    int32_t kind;    // 0 packed parameters (absolute), 1 sorted-feature blocks, 2 mean/max blocks
    uint32_t dst;    // byte offset in the slot
    uint32_t bytes;
    uint32_t pad;
    int64_t a;       // kind 0: byte offset; kind 1: per-tile prefix bytes (x n_tiles); kind 2: layer index
    int64_t stride;  // per-tile stride in bytes
};

struct Step {
    int32_t ncopy;
    uint32_t total;
    int32_t k2;  // K of the (second) GEMM operand
    int32_t pad;
    Copy c[kMaxCopies];
};

struct TcDesc {
    int nl[2];
    int counts[2][16];
    int literal;
    double gamma;
    int n_steps;
    int prof;  // SF_DEBUG_TC: CTA 0 / thread 0 accumulates clock64 per phase into g_tc_prof
    Step steps[kMaxSteps];
};

__device__ unsigned long long g_tc_prof[16];

struct TcPack {
    uint8_t* d_blobs = nullptr;
    TcDesc desc{};
};

struct Ring {
    uint8_t* slot[kSlots];
    uint64_t* full;  // [kSlots]
    uint64_t* mma;
    uint32_t par[kSlots];
    uint32_t mpar;
    int step;
};

__device__ __forceinline__ void issue_step(const Ring& r, const TcDesc& d, int j, const uint8_t* wpk,
                                           const uint8_t* ops, const uint8_t* mms, int tile, int n_tiles) {
    if (j >= d.n_steps) return;
    const Step& s = d.steps[j];
    const int slot = j % kSlots;
    uint64_t* bar = &r.full[slot];
    mbar_expect_tx(bar, s.total);
    for (int c = 0; c < s.ncopy; ++c) {
        const Copy& cp = s.c[c];
        const uint8_t* src;
        if (cp.kind == 0)
            src = wpk + cp.a;
        else if (cp.kind == 1)
            src = ops + cp.a * n_tiles + int64_t(tile) * cp.stride;
        else
            src = mms + cp.a * int64_t(n_tiles) * 4096 + int64_t(tile) * 4096;
        bulk_g2s(r.slot[slot] + cp.dst, src, cp.bytes, bar);
    }
}

// Wait for the current step's bundle (all threads read parameters from it).
__device__ __forceinline__ uint8_t* acquire(Ring& r) {
    const int slot = r.step % kSlots;
    mbar_wait(&r.full[slot], r.par[slot]);
    r.par[slot] ^= 1;
    return r.slot[slot];
}

// Issue the step's MMAs (thread 0) after prefetching bundle j+2, then wait.
// a0/k0 x weights at w0, then optionally a1/k1 x weights at w1 into the same columns.
__device__ __forceinline__ void run_mma(Ring& r, const TcDesc& d, const uint8_t* wpk, const uint8_t* ops,
                                        const uint8_t* mms, int tile, int n_tiles, uint32_t tmem_d, int n,
                                        uint32_t a0, int k0, uint32_t w0, uint32_t a1, int k1, uint32_t w1,
                                        bool accumulate) {
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        tc_fence_after();
        // ring slot (j+2)%3 was last used by step j-1, whose MMA and readers are done
        issue_step(r, d, r.step + kSlots - 1, wpk, ops, mms, tile, n_tiles);
        const uint32_t id = idesc_bf16(n);
        for (int k = 0; k < k0 / 16; ++k)
            umma_bf16(tmem_d, smem_desc(a0 + k * 256, 128, k0 * 16), smem_desc(w0 + k * 256, 128, k0 * 16), id,
                      (accumulate || k > 0) ? 1u : 0u);
        for (int k = 0; k < k1 / 16; ++k)
            umma_bf16(tmem_d, smem_desc(a1 + k * 256, 128, k1 * 16), smem_desc(w1 + k * 256, 128, k1 * 16), id,
                      1u);
        umma_commit(r.mma);
    }
    mbar_wait(r.mma, r.mpar);
    r.mpar ^= 1;
    r.step += 1;
    tc_fence_after();
}

__device__ __forceinline__ float relu(float v) { return v > 0.0f ? v : 0.0f; }

// y = W x + b from shared memory (broadcast reads), FP32
template <int M, int N>
__device__ __forceinline__ void dense_s(const float* W, const float* b, const float* x, float* y) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        float acc = b[i];
#pragma unroll
        for (int j = 0; j < N; ++j) acc = fmaf(W[i * N + j], x[j], acc);
        y[i] = acc;
    }
}

__global__ void __launch_bounds__(kThreads, 2)
    k_backbone_tc(const __grid_constant__ TcDesc d, const uint8_t* __restrict__ wpk, const uint8_t* __restrict__ ops,
                  const uint8_t* __restrict__ mms, int n_tiles, int64_t n, const double* __restrict__ cfg8,
                  float* __restrict__ y_out, double* __restrict__ F_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[kSlots + 1];
    __shared__ uint32_t tmem_slot;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
    const bool prof = d.prof && blockIdx.x == 0 && tid == 0;
    long long t_last = clock64();
    const long long t_start = t_last;
#define PROF(k)                                                             \
    if (prof) {                                                             \
        long long t_now = clock64();                                        \
        atomicAdd(&g_tc_prof[k], (unsigned long long)(t_now - t_last));     \
        t_last = t_now;                                                     \
    }
    const int64_t q = int64_t(tile) * kUmmaM + tid;
    const bool live = q < n;

    uintptr_t base = (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023);
    uint8_t* a_att = reinterpret_cast<uint8_t*>(base);  // [128 x 32]
    uint8_t* a2 = a_att + kUmmaM * 32 * 2;              // [128 x 64]
    Ring r;
    r.slot[0] = a2 + kUmmaM * 64 * 2;
    for (int s = 1; s < kSlots; ++s) r.slot[s] = r.slot[s - 1] + kSlotBytes;
    r.full = bars;
    r.mma = bars + kSlots;
    for (int s = 0; s < kSlots; ++s) r.par[s] = 0;
    r.mpar = 0;
    r.step = 0;

    if (warp == 0) tmem_alloc(&tmem_slot, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s <= kSlots; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (tid == 0)
        for (int j = 0; j < kSlots - 1; ++j) issue_step(r, d, j, wpk, ops, mms, tile, n_tiles);
    const uint32_t lane = uint32_t(warp * 32) << 16;
    const uint32_t s_att = smem_u32(a_att), s_a2 = smem_u32(a2);

    // conditioning (cfg_vector, src/predictor.cpp:193-202)
    float cfgv[7] = {0, 0, 0, 0, 0, 0, 0};
    float g_mean = 0.0f, alpha = 0.0f;
    double alb[3] = {0.5, 0.5, 0.5};
    if (live) {
        const double* c8 = cfg8 + 8 * q;
        int ng = int(c8[0]);
        for (int i = 0; i < ng; ++i) g_mean += float(c8[1 + i]);
        if (ng > 0) g_mean /= float(double(ng));
        alpha = float(c8[7]);
        for (int i = 0; i < ng && i < 3; ++i) cfgv[i] = float(c8[1 + i]);
        for (int i = 0; i < 4; ++i) cfgv[3 + i] = float(c8[4 + i]);
        alb[0] = c8[4];
        alb[1] = c8[5];
        alb[2] = c8[6];
    }

    uint32_t od_pk[16];
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            float o[32];
            for (int i = 0; i < d.nl[kind]; ++i) {
                PROF(7);
                uint8_t* slot = acquire(r);
                PROF(0);
                const uint32_t s_slot = smem_u32(slot);
                const float* prm = reinterpret_cast<const float*>(slot + kSlotAtt);
                if (i == 0) {  // conditioning layer o = relu(W_init cfg + b)
                    const float* ini = reinterpret_cast<const float*>(slot + kSlotInit);
                    dense_s<32, 7>(ini, ini + 224, cfgv, o);
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] = relu(o[j]);
                }
                // channel attention (src/neural.cpp:473-491) from the tile's mean/max block
                const float4* mm = reinterpret_cast<const float4*>(slot + kSlotMM) + tid * 2;
                const float4 m0 = mm[0], m1 = mm[1];
                const float v[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, g_mean, alpha};
                float w;
                if (d.literal) {
                    float acc = 0.0f;
                    for (int j = 0; j < 8; ++j) acc += relu(v[j]);
                    w = 1.0f / (1.0f + __expf(-(acc / 8.0f)));
                } else {
                    float h[4], w3[3];
                    dense_s<4, 8>(prm, prm + 32, v, h);
#pragma unroll
                    for (int j = 0; j < 4; ++j) h[j] = relu(h[j]);
                    dense_s<3, 4>(prm + 36, prm + 48, h, w3);
                    w = 1.0f / (1.0f + __expf(-w3[tau]));
                }
                float oa[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) oa[j] = o[j] * w;
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk(a_att, tid, c, 32, oa + 8 * c);
                PROF(1);
                const int kf = d.steps[r.step].k2;
                run_mma(r, d, wpk, ops, mms, tile, n_tiles, tmem + 0, 32, s_att, 32, s_slot + kSlotW1a,
                        s_slot + kSlotFeat, kf, s_slot + kSlotW1b, false);
                PROF(2);
                // FC-1 epilogue: u = relu(acc + b1) -> bf16 operand of FC-2
                const float* b1 = prm + 52;
                float acc[32];
                tmem_ld32(tmem + lane + 0, acc);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + b1[8 * c + e]);
                    store_chunk(a2, tid, c, 32, v8);
                }
                PROF(3);
                uint8_t* slot2 = acquire(r);
                PROF(4);
                run_mma(r, d, wpk, ops, mms, tile, n_tiles, tmem + 32, 32, s_a2, 32, smem_u32(slot2), 0, 0, 0,
                        false);
                PROF(5);
                // FC-2 epilogue + residual: o = relu(acc + b2) + o_att (fp32)
                const float* b2 = reinterpret_cast<const float*>(slot2 + 2048);
                tmem_ld32(tmem + lane + 32, acc);
#pragma unroll
                for (int j = 0; j < 32; ++j) o[j] = relu(acc[j] + b2[j]) + oa[j];
                PROF(6);
            }
            if (kind == 0) {
#pragma unroll
                for (int j = 0; j < 16; ++j) od_pk[j] = pack_bf16(o[2 * j], o[2 * j + 1]);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(a2 + canon_off(tid, 8 * c, 64)) =
                        make_uint4(od_pk[4 * c], od_pk[4 * c + 1], od_pk[4 * c + 2], od_pk[4 * c + 3]);
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk(a2, tid, 4 + c, 64, o + 8 * c);
            }
        }
        // merged_tau = relu(W_m [od; oh] + b)
        uint8_t* slot = acquire(r);
        run_mma(r, d, wpk, ops, mms, tile, n_tiles, tmem + 64, 64, s_a2, 64, smem_u32(slot), 0, 0, 0, false);
        const float* bm = reinterpret_cast<const float*>(slot + kSlotBias);
        for (int half = 0; half < 2; ++half) {
            float acc[32];
            tmem_ld32(tmem + lane + 64 + 32 * half, acc);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + bm[32 * half + 8 * c + e]);
                store_chunk(a2, tid, half * 4 + c, 64, v8);
            }
        }
        // cross += W_c[:, 64 tau : 64 tau + 64] merged_tau (accumulated in TMEM)
        slot = acquire(r);
        run_mma(r, d, wpk, ops, mms, tile, n_tiles, tmem + 128, 64, s_a2, 64, smem_u32(slot), 0, 0, 0, tau > 0);
        if (tau == 2) {  // the last cross bundle carries the cross bias
            const float* bc = reinterpret_cast<const float*>(slot + kSlotBias);
            float h[32];
            for (int half = 0; half < 2; ++half) {
                tmem_ld32(tmem + lane + 128 + 32 * half, h);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = relu(h[8 * c + e] + bc[32 * half + 8 * c + e]);
                    store_chunk(a2, tid, half * 4 + c, 64, v8);
                }
            }
        }
    }
    // head 0 / 1 (64 -> 64, relu); head 2 (64 -> 3) SIMT from the head-1 bundle
    float h[64];
    for (int l = 0; l < 2; ++l) {
        uint8_t* slot = acquire(r);
        run_mma(r, d, wpk, ops, mms, tile, n_tiles, tmem + 64, 64, s_a2, 64, smem_u32(slot), 0, 0, 0, false);
        const float* bh = reinterpret_cast<const float*>(slot + kSlotBias);
        tmem_ld32(tmem + lane + 64, h);
        tmem_ld32(tmem + lane + 96, h + 32);
#pragma unroll
        for (int j = 0; j < 64; ++j) h[j] = relu(h[j] + bh[j]);
        if (l == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) store_chunk(a2, tid, c, 64, h + 8 * c);
        } else {
            const float* h2 = reinterpret_cast<const float*>(slot + kSlotHead2);
            float y[3];
            dense_s<3, 64>(h2, h2 + 192, h, y);
            if (live) {
                for (int c = 0; c < 3; ++c) {
                    float yc = fabsf(y[c]);
                    if (y_out) y_out[3 * q + c] = yc;
                    if (F_out) F_out[3 * q + c] = pow(alb[c], d.gamma) * expm1(double(yc));  // decode_prediction
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, kTmemCols);
    if (prof) atomicAdd(&g_tc_prof[8], (unsigned long long)(clock64() - t_start));
#undef PROF
}

// ---- host-side packing ------------------------------------------------------------

// B operand of one GEMM: rows = N outputs, cols [col0, col0+cols) of W (leading dim ld), zero padded to Kp.
uint32_t pack_blob(std::vector<uint8_t>& buf, const float* W, int rows, int cols, int ld, int col0, int Kp) {
    size_t off = (buf.size() + 127) & ~size_t(127);
    size_t bytes = size_t(rows) * Kp * 2;
    buf.resize(off + bytes, 0);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < Kp; ++k) {
            float v = k < cols ? W[size_t(r) * ld + col0 + k] : 0.0f;
            __nv_bfloat16 h = __float2bfloat16_rn(v);
            std::memcpy(&buf[off + canon_off(r, k, Kp)], &h, 2);
        }
    return uint32_t(off);
}

// FP32 parameters (16-byte aligned, padded to a multiple of 16 bytes).
uint32_t pack_f32(std::vector<uint8_t>& buf, const std::vector<float>& v) {
    size_t off = (buf.size() + 127) & ~size_t(127);
    size_t bytes = (v.size() * 4 + 15) & ~size_t(15);
    buf.resize(off + bytes, 0);
    std::memcpy(&buf[off], v.data(), v.size() * 4);
    return uint32_t(off);
}

uint32_t f32_bytes(size_t n) { return uint32_t((n * 4 + 15) & ~size_t(15)); }

Copy pcopy(uint32_t off, uint32_t bytes, uint32_t dst) { return Copy{0, dst, bytes, 0, int64_t(off), 0}; }

std::vector<float> slice(const std::vector<float>& P, int64_t off, size_t n) {
    return std::vector<float>(P.begin() + off, P.begin() + off + int64_t(n));
}

}  // namespace

bool tc_supported(const sf_backbone_config& c) {
    if (c.width != 32 || c.merge_width != 64 || c.head_width != 64) return false;
    if (c.n_diffuse_layers * 6 + c.n_highlight_layers * 6 + 3 * 2 + 2 > kMaxSteps) return false;
    for (int i = 0; i < c.n_diffuse_layers; ++i)
        if (c.diffuse_counts[i] + 2 > 64) return false;
    for (int i = 0; i < c.n_highlight_layers; ++i)
        if (c.highlight_counts[i] + 2 > 64) return false;
    return true;
}

SortLayout sort_layout(const sf_backbone_config& c) {
    SortLayout L{};
    L.nl[0] = c.n_diffuse_layers;
    L.nl[1] = c.n_highlight_layers;
    int64_t prefix = 0;
    int layer = 0;
    for (int k = 0; k < 2; ++k) {
        const int* counts = k == 0 ? c.diffuse_counts : c.highlight_counts;
        int start = 0;
        for (int i = 0; i < L.nl[k]; ++i) {
            L.counts[k][i] = counts[i];
            L.start[k][i] = start;
            L.kf[k][i] = (counts[i] + 2 + 15) / 16 * 16;
            L.mm_layer[k][i] = layer++;
            start += counts[i];
            for (int t = 0; t < 3; ++t) {
                L.seg_prefix[k][i][t] = prefix;  // bytes per tile before this segment
                prefix += int64_t(kUmmaM) * L.kf[k][i] * 2;
            }
        }
        L.npts[k] = start;
    }
    L.tile_bytes = prefix;
    L.n_layers = layer;
    return L;
}

void tc_prepare(sf_backbone& b, cudaStream_t s) {
    if (b.tc) return;
    const sf_backbone_config& c = b.cfg;
    const BackboneLayout& L = b.layout;
    const SortLayout S = sort_layout(c);
    std::vector<float> P(size_t(L.total));
    SFB_CUDA(cudaMemcpyAsync(P.data(), b.d_params, P.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
    SFB_CUDA(cudaStreamSynchronize(s));
    auto pk = std::make_unique<TcPack>();
    std::vector<uint8_t> buf;
    std::vector<Step> steps;
    const int W = 32;
    auto push = [&](Step st) {
        st.total = 0;
        for (int k = 0; k < st.ncopy; ++k) st.total += st.c[k].bytes;
        steps.push_back(st);
    };
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            const int64_t init_off = L.stack_off[kind][tau];
            int64_t off = init_off + W * 7 + W;
            for (int i = 0; i < S.nl[kind]; ++i) {
                std::vector<float> simt(84, 0.0f);  // [W1 32, b1 4, W2 12, b2 3, pad] + FC-1 bias [32]
                if (!c.literal_attention) {
                    for (int k = 0; k < 51; ++k) simt[size_t(k)] = P[size_t(off + k)];
                    off += 51;
                }
                const int cnt = S.counts[kind][i];
                const int K = W + cnt + 2, kf = S.kf[kind][i];
                for (int k = 0; k < W; ++k) simt[size_t(52 + k)] = P[size_t(off + int64_t(W) * K + k)];
                Step st{};
                st.k2 = kf;
                st.c[0] = pcopy(pack_blob(buf, P.data() + off, W, W, K, 0, W), W * W * 2, kSlotW1a);
                st.c[1] = pcopy(pack_blob(buf, P.data() + off, W, cnt + 2, K, W, kf), uint32_t(W * kf * 2), kSlotW1b);
                st.c[2] = Copy{1, uint32_t(kSlotFeat), uint32_t(kUmmaM * kf * 2), 0, S.seg_prefix[kind][i][tau],
                               int64_t(kUmmaM) * kf * 2};
                st.c[3] = Copy{2, uint32_t(kSlotMM), uint32_t(kUmmaM * 8 * 4), 0, S.mm_layer[kind][i], 4096};
                st.c[4] = pcopy(pack_f32(buf, simt), f32_bytes(simt.size()), kSlotAtt);
                st.ncopy = 5;
                if (i == 0) {  // conditioning layer of the stack
                    std::vector<float> ini = slice(P, init_off, size_t(W * 7 + W));
                    st.c[5] = pcopy(pack_f32(buf, ini), f32_bytes(ini.size()), kSlotInit);
                    st.ncopy = 6;
                }
                push(st);
                off += int64_t(W) * K + W;
                Step s2{};
                s2.k2 = W;
                s2.c[0] = pcopy(pack_blob(buf, P.data() + off, W, W, W, 0, W), W * W * 2, 0);
                s2.c[1] = pcopy(pack_f32(buf, slice(P, off + W * W, W)), f32_bytes(W), 2048);
                s2.ncopy = 2;
                push(s2);
                off += W * W + W;
            }
        }
        const int64_t mo = L.merge_off + int64_t(tau) * (64 * 64 + 64);
        Step sm{};
        sm.k2 = 64;
        sm.c[0] = pcopy(pack_blob(buf, P.data() + mo, 64, 64, 64, 0, 64), 8192, 0);
        sm.c[1] = pcopy(pack_f32(buf, slice(P, mo + 64 * 64, 64)), f32_bytes(64), kSlotBias);
        sm.ncopy = 2;
        push(sm);
        Step sc{};
        sc.k2 = 64;
        sc.c[0] = pcopy(pack_blob(buf, P.data() + L.cross_off, 64, 64, 192, 64 * tau, 64), 8192, 0);
        sc.ncopy = 1;
        if (tau == 2) {
            sc.c[1] = pcopy(pack_f32(buf, slice(P, L.cross_off + 64 * 192, 64)), f32_bytes(64), kSlotBias);
            sc.ncopy = 2;
        }
        push(sc);
    }
    for (int l = 0; l < 2; ++l) {
        Step sh{};
        sh.k2 = 64;
        sh.c[0] = pcopy(pack_blob(buf, P.data() + L.head_off[l], 64, 64, 64, 0, 64), 8192, 0);
        sh.c[1] = pcopy(pack_f32(buf, slice(P, L.head_off[l] + 64 * 64, 64)), f32_bytes(64), kSlotBias);
        sh.ncopy = 2;
        if (l == 1) {
            std::vector<float> h2 = slice(P, L.head_off[2], 3 * 64 + 3);
            sh.c[2] = pcopy(pack_f32(buf, h2), f32_bytes(h2.size()), kSlotHead2);
            sh.ncopy = 3;
        }
        push(sh);
    }
    if (steps.size() > size_t(kMaxSteps)) fail(SF_ERR_INVALID_ARGUMENT, "tc backbone: too many layers");
    TcDesc& d = pk->desc;
    d.nl[0] = S.nl[0];
    d.nl[1] = S.nl[1];
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < S.nl[k]; ++i) d.counts[k][i] = S.counts[k][i];
    d.literal = c.literal_attention;
    d.gamma = c.gamma;
    d.n_steps = int(steps.size());
    for (size_t j = 0; j < steps.size(); ++j) d.steps[j] = steps[j];
    d.prof = std::getenv("SF_DEBUG_TC") != nullptr;
    SFB_CUDA(cudaMalloc(&pk->d_blobs, buf.size()));
    SFB_CUDA(cudaMemcpy(pk->d_blobs, buf.data(), buf.size(), cudaMemcpyHostToDevice));
    b.tc = pk.release();
}

void tc_release(sf_backbone& b) {
    auto pk = static_cast<TcPack*>(b.tc);
    if (!pk) return;
    cudaFree(pk->d_blobs);
    delete pk;
    b.tc = nullptr;
}

void launch_backbone_tc(const sf_backbone& b, int64_t n, const uint8_t* ops, const float* mms, const double* cfg8,
                        float* y, double* F, cudaStream_t s) {
    if (n <= 0) return;
    auto pk = static_cast<const TcPack*>(b.tc);
    const size_t smem = 1024 + kUmmaM * 32 * 2 + kUmmaM * 64 * 2 + size_t(kSlots) * kSlotBytes;
    static bool attr_set = false;
    if (!attr_set) {
        SFB_CUDA(cudaFuncSetAttribute(k_backbone_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_set = true;
    }
    const int n_tiles = int((n + kUmmaM - 1) / kUmmaM);
    k_backbone_tc<<<n_tiles, kThreads, smem, s>>>(pk->desc, pk->d_blobs, ops, reinterpret_cast<const uint8_t*>(mms),
                                                  n_tiles, n, cfg8, y, F);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void tc_read_prof(unsigned long long* out) {
    SFB_CUDA(cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(unsigned long long) * 16));
    unsigned long long z[16] = {};
    SFB_CUDA(cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z)));
}

}  // namespace sfb
