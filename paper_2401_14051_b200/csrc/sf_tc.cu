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
// Everything a step needs (weight blob, the tile's sorted-feature operand block
// and its mean/max block) is one bundle of cp.async.bulk copies into a 3-slot
// SMEM ring completing on one mbarrier; bundle j+2 is in flight while step j
// runs. The SIMT pieces (7->32 conditioning layer, 8->4->3 channel attention,
// 64->3 output layer) and the residual stream stay FP32 on the CUDA cores.
//
// Precision: bf16 GEMM operands (weights, o_att, features, u, merges), fp32
// accumulation, fp32 bias / activation / residual (tests/bf16_emulation.py).
#include <cstring>
#include <vector>

#include "sf_internal.h"
#include "sf_umma.cuh"

namespace sfb {

namespace {

constexpr int kThreads = 128;     // one thread per query row / TMEM lane
constexpr int kTmemCols = 256;    // fc1 [0,32) fc2 [32,64) merge/head [64,128) cross [128,192)
constexpr int kSlots = 3;
constexpr int kSlotBytes = 27648;
constexpr int kSlotW1a = 0, kSlotW1b = 2048, kSlotFeat = 6144, kSlotMM = 22528;
constexpr int kMaxSteps = 96;

struct Copy {
    int32_t kind;     // 0 weights (absolute), 1 sorted-feature blocks, 2 mean/max blocks
    uint32_t dst;     // byte offset in the slot
    uint32_t bytes;
    uint32_t pad;
    int64_t a;        // kind 0: byte offset; kind 1: per-tile prefix bytes (x n_tiles); kind 2: layer index
    int64_t stride;   // per-tile stride in bytes (0 for weights)
};

struct Step {
    int32_t ncopy;
    uint32_t total;
    int32_t k2;       // K of the second GEMM operand (fc1 feature part) or the only GEMM's K
    int32_t pad;
    Copy c[4];
};

struct TcDesc {
    int nl[2];
    int counts[2][16];
    int W, M, H;
    int literal;
    double gamma;
    int64_t stack_off[2][3];
    int64_t merge_off, cross_off, head_off[3];
    int n_steps;
};

struct TcPack {
    uint8_t* d_blobs = nullptr;
    Step* d_steps = nullptr;
    TcDesc desc{};
    std::vector<Step> steps;
};

struct Ring {
    uint8_t* slot[kSlots];
    uint64_t* full;   // [kSlots]
    uint64_t* mma;
    uint32_t par[kSlots];
    uint32_t mpar;
    int step;
};

__device__ __forceinline__ void issue_step(const Ring& r, const Step* __restrict__ steps, int n_steps, int j,
                                           const uint8_t* wpk, const uint8_t* ops, const uint8_t* mms,
                                           int tile, int n_tiles) {
    if (j >= n_steps) return;
    const Step& s = steps[j];
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

// Wait for step j's bundle (all threads: some read the mean/max block).
__device__ __forceinline__ uint8_t* acquire(Ring& r) {
    const int slot = r.step % kSlots;
    mbar_wait(&r.full[slot], r.par[slot]);
    r.par[slot] ^= 1;
    return r.slot[slot];
}

// Issue the step's MMAs (thread 0), prefetch bundle j+2, wait for completion.
// a0/k0: first GEMM operand (SMEM) x slot weights at w0; optional second
// operand a1/k1 x slot weights at w1, accumulating into the same columns.
__device__ __forceinline__ void run_mma(Ring& r, const Step* steps, int n_steps, const uint8_t* wpk,
                                        const uint8_t* ops, const uint8_t* mms, int tile, int n_tiles,
                                        uint32_t tmem_d, int n, uint32_t a0, int k0, uint32_t w0, uint32_t a1,
                                        int k1, uint32_t w1, bool accumulate) {
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t id = idesc_bf16(n);
        for (int k = 0; k < k0 / 16; ++k)
            umma_bf16(tmem_d, smem_desc(a0 + k * 256, 128, k0 * 16), smem_desc(w0 + k * 256, 128, k0 * 16), id,
                      (accumulate || k > 0) ? 1u : 0u);
        for (int k = 0; k < k1 / 16; ++k)
            umma_bf16(tmem_d, smem_desc(a1 + k * 256, 128, k1 * 16), smem_desc(w1 + k * 256, 128, k1 * 16), id,
                      1u);
        umma_commit(r.mma);
        issue_step(r, steps, n_steps, r.step + kSlots - 1, wpk, ops, mms, tile, n_tiles);
    }
    mbar_wait(r.mma, r.mpar);
    r.mpar ^= 1;
    r.step += 1;
    tc_fence_after();
}

__device__ __forceinline__ float relu(float v) { return v > 0.0f ? v : 0.0f; }

__device__ __forceinline__ void dense_simt(const float* __restrict__ W, const float* __restrict__ b, int m,
                                           int n, const float* x, float* y) {
    for (int i = 0; i < m; ++i) {
        float acc = __ldg(b + i);
        const float* row = W + i * n;
        for (int j = 0; j < n; ++j) acc = fmaf(__ldg(row + j), x[j], acc);
        y[i] = acc;
    }
}

__global__ void __launch_bounds__(kThreads, 2)
    k_backbone_tc(TcDesc d, const Step* __restrict__ steps, const float* __restrict__ P,
                  const uint8_t* __restrict__ wpk, const uint8_t* __restrict__ ops, const uint8_t* __restrict__ mms,
                  int n_tiles, int64_t n, const double* __restrict__ cfg8, float* __restrict__ y_out,
                  double* __restrict__ F_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[kSlots + 1];
    __shared__ uint32_t tmem_slot;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
    const int64_t q = int64_t(tile) * kUmmaM + tid;
    const bool live = q < n;
    constexpr int W = 32;

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
        for (int j = 0; j < kSlots - 1; ++j) issue_step(r, steps, d.n_steps, j, wpk, ops, mms, tile, n_tiles);
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
            int64_t off = d.stack_off[kind][tau];
            float o[32];
            dense_simt(P + off, P + off + W * 7, W, 7, cfgv, o);
            off += W * 7 + W;
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = relu(o[j]);
            for (int i = 0; i < d.nl[kind]; ++i) {
                const int cnt = d.counts[kind][i];
                uint8_t* slot = acquire(r);
                const uint32_t s_slot = smem_u32(slot);
                // channel attention (src/neural.cpp:473-491) from the tile's mean/max block
                const float* mm = reinterpret_cast<const float*>(slot + kSlotMM) + tid * 8;
                float v[8] = {mm[0], mm[1], mm[2], mm[3], mm[4], mm[5], g_mean, alpha};
                float w;
                if (d.literal) {
                    float acc = 0.0f;
                    for (int j = 0; j < 8; ++j) acc += relu(v[j]);
                    w = 1.0f / (1.0f + __expf(-(acc / 8.0f)));
                } else {
                    float h[4], w3[3];
                    dense_simt(P + off, P + off + 32, 4, 8, v, h);
                    for (int j = 0; j < 4; ++j) h[j] = relu(h[j]);
                    dense_simt(P + off + 36, P + off + 48, 3, 4, h, w3);
                    w = 1.0f / (1.0f + __expf(-w3[tau]));
                    off += 51;
                }
                float oa[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) oa[j] = o[j] * w;
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk(a_att, tid, c, 32, oa + 8 * c);
                const int kf = steps[r.step].k2;
                run_mma(r, steps, d.n_steps, wpk, ops, mms, tile, n_tiles, tmem + 0, 32, s_att, 32,
                        s_slot + kSlotW1a, s_slot + kSlotFeat, kf, s_slot + kSlotW1b, false);
                // FC-1 epilogue: u = relu(acc + b1) -> bf16 operand of FC-2
                const float* b1 = P + off + int64_t(W) * (W + cnt + 2);
                float acc[32];
                tmem_ld32(tmem + lane + 0, acc);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + __ldg(b1 + 8 * c + e));
                    store_chunk(a2, tid, c, 32, v8);
                }
                off += int64_t(W) * (W + cnt + 2) + W;
                uint8_t* slot2 = acquire(r);
                run_mma(r, steps, d.n_steps, wpk, ops, mms, tile, n_tiles, tmem + 32, 32, s_a2, 32,
                        smem_u32(slot2), 0, 0, 0, false);
                // FC-2 epilogue + residual: o = relu(acc + b2) + o_att (fp32)
                const float* b2 = P + off + W * W;
                tmem_ld32(tmem + lane + 32, acc);
#pragma unroll
                for (int j = 0; j < 32; ++j) o[j] = relu(acc[j] + __ldg(b2 + j)) + oa[j];
                off += W * W + W;
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
        run_mma(r, steps, d.n_steps, wpk, ops, mms, tile, n_tiles, tmem + 64, 64, s_a2, 64, smem_u32(slot), 0, 0,
                0, false);
        const float* bm = P + d.merge_off + int64_t(tau) * (64 * 64 + 64) + 64 * 64;
        for (int half = 0; half < 2; ++half) {
            float acc[32];
            tmem_ld32(tmem + lane + 64 + 32 * half, acc);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + __ldg(bm + 32 * half + 8 * c + e));
                store_chunk(a2, tid, half * 4 + c, 64, v8);
            }
        }
        // cross += W_c[:, 64 tau : 64 tau + 64] merged_tau (accumulated in TMEM)
        slot = acquire(r);
        run_mma(r, steps, d.n_steps, wpk, ops, mms, tile, n_tiles, tmem + 128, 64, s_a2, 64, smem_u32(slot), 0,
                0, 0, tau > 0);
    }
    float h[64];
    {
        const float* bc = P + d.cross_off + 64 * 192;
        tmem_ld32(tmem + lane + 128, h);
        tmem_ld32(tmem + lane + 160, h + 32);
#pragma unroll
        for (int j = 0; j < 64; ++j) h[j] = relu(h[j] + __ldg(bc + j));
    }
    for (int l = 0; l < 2; ++l) {
#pragma unroll
        for (int c = 0; c < 8; ++c) store_chunk(a2, tid, c, 64, h + 8 * c);
        uint8_t* slot = acquire(r);
        run_mma(r, steps, d.n_steps, wpk, ops, mms, tile, n_tiles, tmem + 64, 64, s_a2, 64, smem_u32(slot), 0, 0,
                0, false);
        const float* bh = P + d.head_off[l] + 64 * 64;
        tmem_ld32(tmem + lane + 64, h);
        tmem_ld32(tmem + lane + 96, h + 32);
#pragma unroll
        for (int j = 0; j < 64; ++j) h[j] = relu(h[j] + __ldg(bh + j));
    }
    float y[3];
    dense_simt(P + d.head_off[2], P + d.head_off[2] + 3 * 64, 3, 64, h, y);
    if (live) {
        for (int c = 0; c < 3; ++c) {
            float yc = fabsf(y[c]);
            if (y_out) y_out[3 * q + c] = yc;
            if (F_out) F_out[3 * q + c] = pow(alb[c], d.gamma) * expm1(double(yc));  // decode_prediction
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, kTmemCols);
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

Copy wcopy(uint32_t off, uint32_t bytes, uint32_t dst) { return Copy{0, dst, bytes, 0, int64_t(off), 0}; }

}  // namespace

bool tc_supported(const sf_backbone_config& c) {
    if (c.width != 32 || c.merge_width != 64 || c.head_width != 64) return false;
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
    auto pk = new TcPack();
    std::vector<uint8_t> buf;
    std::vector<Step>& steps = pk->steps;
    const int W = 32;
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            int nl = S.nl[kind];
            int64_t off = L.stack_off[kind][tau] + W * 7 + W;
            for (int i = 0; i < nl; ++i) {
                if (!c.literal_attention) off += 51;
                const int cnt = S.counts[kind][i];
                const int K = W + cnt + 2, kf = S.kf[kind][i];
                uint32_t oa = pack_blob(buf, P.data() + off, W, W, K, 0, W);
                uint32_t ob = pack_blob(buf, P.data() + off, W, cnt + 2, K, W, kf);
                Step st{};
                st.ncopy = 4;
                st.k2 = kf;
                st.c[0] = wcopy(oa, W * W * 2, kSlotW1a);
                st.c[1] = wcopy(ob, uint32_t(W * kf * 2), kSlotW1b);
                st.c[2] = Copy{1, kSlotFeat, uint32_t(kUmmaM * kf * 2), 0, S.seg_prefix[kind][i][tau],
                               int64_t(kUmmaM) * kf * 2};
                st.c[3] = Copy{2, kSlotMM, uint32_t(kUmmaM * 8 * 4), 0, S.mm_layer[kind][i], 4096};
                steps.push_back(st);
                off += int64_t(W) * K + W;
                uint32_t o2 = pack_blob(buf, P.data() + off, W, W, W, 0, W);
                Step s2{};
                s2.ncopy = 1;
                s2.k2 = W;
                s2.c[0] = wcopy(o2, W * W * 2, 0);
                steps.push_back(s2);
                off += W * W + W;
            }
        }
        Step sm{};
        sm.ncopy = 1;
        sm.k2 = 64;
        sm.c[0] = wcopy(pack_blob(buf, P.data() + L.merge_off + int64_t(tau) * (64 * 64 + 64), 64, 64, 64, 0, 64),
                        8192, 0);
        steps.push_back(sm);
        Step sc{};
        sc.ncopy = 1;
        sc.k2 = 64;
        sc.c[0] = wcopy(pack_blob(buf, P.data() + L.cross_off, 64, 64, 192, 64 * tau, 64), 8192, 0);
        steps.push_back(sc);
    }
    for (int l = 0; l < 2; ++l) {
        Step sh{};
        sh.ncopy = 1;
        sh.k2 = 64;
        sh.c[0] = wcopy(pack_blob(buf, P.data() + L.head_off[l], 64, 64, 64, 0, 64), 8192, 0);
        steps.push_back(sh);
    }
    if (steps.size() > size_t(kMaxSteps)) fail(SF_ERR_INVALID_ARGUMENT, "tc backbone: too many layers");
    for (Step& st : steps) {
        st.total = 0;
        for (int k = 0; k < st.ncopy; ++k) st.total += st.c[k].bytes;
    }
    TcDesc& d = pk->desc;
    d.nl[0] = S.nl[0];
    d.nl[1] = S.nl[1];
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < S.nl[k]; ++i) d.counts[k][i] = S.counts[k][i];
    d.W = c.width;
    d.M = c.merge_width;
    d.H = c.head_width;
    d.literal = c.literal_attention;
    d.gamma = c.gamma;
    for (int k = 0; k < 2; ++k)
        for (int t = 0; t < 3; ++t) d.stack_off[k][t] = L.stack_off[k][t];
    d.merge_off = L.merge_off;
    d.cross_off = L.cross_off;
    for (int l = 0; l < 3; ++l) d.head_off[l] = L.head_off[l];
    d.n_steps = int(steps.size());
    SFB_CUDA(cudaMalloc(&pk->d_blobs, buf.size()));
    SFB_CUDA(cudaMemcpy(pk->d_blobs, buf.data(), buf.size(), cudaMemcpyHostToDevice));
    SFB_CUDA(cudaMalloc(&pk->d_steps, steps.size() * sizeof(Step)));
    SFB_CUDA(cudaMemcpy(pk->d_steps, steps.data(), steps.size() * sizeof(Step), cudaMemcpyHostToDevice));
    b.tc = pk;
}

void launch_backbone_tc(const sf_backbone& b, int64_t n, const uint8_t* ops, const float* mms,
                        const double* cfg8, float* y, double* F, cudaStream_t s) {
    if (n <= 0) return;
    auto pk = static_cast<const TcPack*>(b.tc);
    const size_t smem = 1024 + kUmmaM * 32 * 2 + kUmmaM * 64 * 2 + size_t(kSlots) * kSlotBytes;
    static bool attr_set = false;
    if (!attr_set) {
        SFB_CUDA(cudaFuncSetAttribute(k_backbone_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_set = true;
    }
    const int n_tiles = int((n + kUmmaM - 1) / kUmmaM);
    k_backbone_tc<<<n_tiles, kThreads, smem, s>>>(pk->desc, pk->d_steps, b.d_params, pk->d_blobs, ops,
                                                  reinterpret_cast<const uint8_t*>(mms), n_tiles, n, cfg8, y, F);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void tc_release(sf_backbone& b) {
    auto pk = static_cast<TcPack*>(b.tc);
    if (!pk) return;
    cudaFree(pk->d_blobs);
    cudaFree(pk->d_steps);
    delete pk;
    b.tc = nullptr;
}

}  // namespace sfb
