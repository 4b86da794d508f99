// sf_tc.cu — the backbone forward on 5th-generation tensor cores (tcgen05).
//
// One CTA = one tile of 128 shading points = UMMA_M. Thread t owns query row t,
// which is also TMEM lane t, so each epilogue is a private tcgen05.ld of the
// thread's own accumulator row. The reference network (src/predictor.cpp:206-235,
// 352-387) becomes a chain of tcgen05.mma GEMMs D[128 x N] (fp32, TMEM) = A * W^T:
//
//   FC-1  = [o_att | sorted_tau, mean, max] W1^T as two MMAs into one accumulator:
//           A_att (K=32, written by the threads) x W1[:, :32]  +
//           F     (K=pad16(n), bulk-copied, produced by k_sample_sort) x W1[:, 32:32+n]
//           and the layer's (mean, max) x W1's last two columns as an fp32 rank-2
//           update in the epilogue (keeps K small and the pools unrounded)
//   FC-2  (N=32, K=32), per-type merge (N=64, K=64), cross merge accumulated
//   chunk by chunk as each merged_tau appears (3 x K=64), head 0/1 (N=64, K=64).
//
// The reference's W[out][in] row-major is exactly UMMA's K-major B operand, so
// weights are packed once (tc_prepare) into the no-swizzle canonical layout.
// Everything a step needs — its weight blob, the tile's sorted-feature operand
// block and mean/max block, and the step's small FP32 SIMT parameters (attention
// 8->4->3, biases, the 7->32 conditioning layer, the 64->3 output layer) — is one
// bundle of cp.async.bulk copies into a ring of SMEM slots completing on one
// mbarrier; every consumer warp releases a slot the moment it is done with it (the
// step's MMA completed, its biases already in registers), so the next bundle lands
// while the layer's epilogue runs. The step program is read from global memory by the
// producer warp. The per-layer chain (MMA -> epilogue -> MMA) is latency-bound, so
// throughput comes from independent chains per SM: three CTAs (RingTri).
//
// Precision: bf16 GEMM operands (weights, o_att, features, u, merges), fp32
// accumulation, fp32 bias / activation / residual / attention (tests/bf16_emulation.py).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "sf_internal.h"
#include "sf_umma.cuh"

namespace sfb {

namespace {

constexpr int kConsumers = 128;             // one thread per query row / TMEM lane
constexpr int kThreads = kConsumers + 32;    // + one producer warp issuing the bundle copies
// TMEM: fc1 [0,32) fc2 [32,64); merge / head [0,64) once a type's stacks are done; cross [64,128)
constexpr int kTmemCols = 128;
constexpr int kColMerge = 0, kColCross = 64;
// Ring geometry (compile-time, so every bundle read has a constant offset): slots of the
// network's largest FC-1 bundle. Layers of up to 48 points: RingTri, 2 slots of 17,792 B
// (~70 KB of shared memory, 128 TMEM columns, <= 128 registers: three CTAs = three
// independent layer chains per SM; a slot is refilled as soon as every warp is done with
// it); up to 64 points: RingWide, 3 slots of 23,552 B, two CTAs per SM.
struct RingNarrow {
    static constexpr int NS = 4, SB = 17792, OF = 5120, OB = 17408, KF = 48, MINB = 2;
};
struct RingWide {
    static constexpr int NS = 3, SB = 23552, OF = 6144, OB = 22528, KF = 64, MINB = 2;
};
// two slots, ~70 KB: three CTAs (three independent chains) per SM
struct RingTri {
    static constexpr int NS = 2, SB = 17792, OF = 5120, OB = 17408, KF = 48, MINB = 3;
};
// FC-1 bundle: W1[:, :32], W1[:, 32:], the tile's sorted-feature block, FC-1 bias
// (the sorted-feature block at RC::OF, b1 + W1's mean / max columns at RC::OB)
constexpr int kSlotW1a = 0, kSlotW1b = 2048;
// FC-2 bundle: W2, bias. 64-wide bundles: weights, bias, head2 W/b (head-1 bundle)
constexpr int kSlotB2 = 2048, kSlotBias = 8192, kSlotHead2 = 8448;
constexpr int kSlotWmHi = 4096;  // merge bundle: W_m[:, 0:32] at 0, W_m[:, 32:64] here
// Attention payload of the NEXT FC-1 step, carried by the bundle of the step before it so
// the attention weight is computed while that step's MMA runs: the tile's mean/max block,
// [52] attention W1 b1 W2 b2 (+pad), [224 + 32] conditioning W/b (first layer of a stack).
constexpr int kPayMM = 9728, kPayAtt = 13824, kPayInit = 14080;
template <class RC>
constexpr bool ring_ok() {
    return kSlotW1b + 32 * RC::KF * 2 <= RC::OF && RC::OF + kUmmaM * RC::KF * 2 <= RC::OB && RC::OB + 384 <= RC::SB &&
           kPayInit + 1024 <= RC::SB && RC::OF % 128 == 0 && RC::SB % 128 == 0;
}
static_assert(ring_ok<RingNarrow>() && ring_ok<RingWide>() && ring_ok<RingTri>(), "slot layout");
template <class RC>
constexpr size_t ring_smem() {
    return 1024 + 2 * kUmmaM * 32 * 2 + kUmmaM * 64 * 2 + size_t(RC::NS) * RC::SB;
}
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
    int32_t k2;   // K of the (second) GEMM operand
    int32_t cls;  // k_backbone_rr: 0 big ring (FC-1 bundles), 1 small ring
    Copy c[kMaxCopies];
};

static_assert(sizeof(Copy) == 32 && sizeof(Step) == 16 + 32 * kMaxCopies, "step program is read as int4 words");

struct TcDesc {
    int nl[2];
    int counts[2][16];
    int literal;
    double gamma;
    int n_steps;
    int prof;  // SF_DEBUG_TC (builds with -DSF_TC_PROFILE): CTA 0 / thread 0 accumulates clock64 per phase
    const Step* steps;  // step program in global memory (read through the L1 by the issuing thread)
};

__device__ unsigned long long g_tc_prof[16];

struct TcPack {
    uint8_t* d_blobs = nullptr;
    TcDesc desc{};
    bool narrow = false;  // RingNarrow / RingTri (every layer <= 48 points) else RingWide
    bool tri = false;     // RingTri may run it (same layout as RingNarrow; chosen per launch)
    bool rr = false;      // k_backbone_rr's program (desc_rr) was built
    TcDesc desc_rr{};
};

struct Ring {
    uint8_t* base;
    uint64_t* full;   // [NS] bundle landed (producer expect_tx + bulk copies)
    uint64_t* empty;  // [NS] bundle consumed (consumer thread 0)
    uint64_t* mma;    // MMA completion (tcgen05.commit)
    uint32_t mpar;
};

// Producer: the copies of one step into ring slot j % NS. The step program is in
// global memory; the whole descriptor is fetched with independent loads (one L2 round
// trip) before the producer waits for the slot, so only the copies remain to issue.
struct StepRegs {
    int4 w[1 + 2 * kMaxCopies];
};

__device__ __forceinline__ void load_step(const TcDesc& d, int j, StepRegs& sr) {
    const int4* p = reinterpret_cast<const int4*>(d.steps + j);
#pragma unroll
    for (int k = 0; k < 1 + 2 * kMaxCopies; ++k) sr.w[k] = __ldg(p + k);
}

template <class RC>
__device__ __forceinline__ void issue_step(const Ring& r, const StepRegs& sr, int j, const uint8_t* wpk,
                                           const uint8_t* ops, const uint8_t* mms, int tile, int n_tiles) {
    const int slot = j % RC::NS;
    uint64_t* bar = &r.full[slot];
    mbar_expect_tx(bar, uint32_t(sr.w[0].y));
#pragma unroll
    for (int c = 0; c < kMaxCopies; ++c) {
        if (c >= sr.w[0].x) break;
        const int4 c0 = sr.w[1 + 2 * c], c1 = sr.w[2 + 2 * c];
        const int kind = c0.x;
        const uint32_t dst = uint32_t(c0.y), bytes = uint32_t(c0.z);
        const int64_t a = (int64_t(uint32_t(c1.y)) << 32) | uint32_t(c1.x);
        const int64_t stride = (int64_t(uint32_t(c1.w)) << 32) | uint32_t(c1.z);
        const uint8_t* src;
        if (kind == 0)
            src = wpk + a;
        else if (kind == 1)
            src = ops + a * n_tiles + int64_t(tile) * stride;
        else
            src = mms + a * int64_t(n_tiles) * 4096 + int64_t(tile) * 4096;
        bulk_g2s(r.base + slot * RC::SB + dst, src, bytes, bar);
    }
}

#ifdef SF_TC_WATCHDOG
// Debug builds: a wait that has not completed after ~1 s records who waited on what in
// g_tc_prof[14..15] and gives up, so a protocol deadlock ends the kernel with a diagnosis.
__device__ void wd_wait(uint64_t* bar, uint32_t parity, int code, int j) {
    const long long t0 = clock64();
    while (true) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) return;
        if (clock64() - t0 > 2000000000ll) {
            if (atomicCAS(&g_tc_prof[15], 0ull, 1ull + blockIdx.x) == 0ull)
                g_tc_prof[14] = uint64_t(code) | (uint64_t(j) << 8) | (uint64_t(parity) << 24) |
                                (uint64_t(threadIdx.x) << 32);
            return;
        }
    }
}
#define SF_WAIT(bar, par, code, j) wd_wait(bar, par, code, j)
#else
#define SF_WAIT(bar, par, code, j) mbar_wait(bar, par)
#endif

template <class RC>
__device__ __forceinline__ uint8_t* wait_full(const Ring& r, int j) {
    const int slot = j % RC::NS;
    SF_WAIT(&r.full[slot], uint32_t(j / RC::NS) & 1u, 1, j);
    return r.base + slot * RC::SB;
}

// Every consumer warp, once step j's bundle is dead for it (its MMA completed and the warp's
// last read of the slot done): one arrival per warp, so a slot is refilled as early as possible.
template <class RC>
__device__ __forceinline__ void release(const Ring& r, int j) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&r.empty[j % RC::NS]);
}

// Operands written by the consumer threads -> visible to the tensor core; then thread 0 issues.
__device__ __forceinline__ void mma_sync() {
    fence_proxy_async();
    tc_fence_before();
    consumer_bar_sync();
    tc_fence_after();
}

__device__ __forceinline__ void mma_wait(Ring& r) {
    SF_WAIT(r.mma, r.mpar, 3, 0);
    r.mpar ^= 1;
    tc_fence_after();
}

// D[128 x n] (+)= A[128 x k] * W[n x k]^T, both K-major canonical; one UMMA per 16 K.
template <bool kH>
__device__ __forceinline__ void issue_gemm(uint32_t tmem_d, int n, uint32_t a, int k, uint32_t w, bool accumulate) {
    const uint32_t id = idesc16(n, kH);
    const uint64_t da = smem_desc(a, 128, k * 16), dw = smem_desc(w, 128, k * 16);
    for (int s = 0; s < k / 16; ++s)  // +256 B per K step = +16 in the start-address field
        umma_bf16(tmem_d, da + 16u * s, dw + 16u * s, id, (accumulate || s > 0) ? 1u : 0u);
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

struct RowCtx {
    float cfgv[7];
    float g_mean, alpha;
    int literal;
};

// Channel attention weight of type tau (src/neural.cpp:473-491) from a bundle's payload.
// Also returns the layer's pools of type tau (mean, max: the fp32 part of its FC-1).
template <int kMM = kPayMM, int kAtt = kPayAtt>
__device__ __forceinline__ float attention(const uint8_t* slot, int tau, const RowCtx& rc, float2& pool) {
    const float4* mm = reinterpret_cast<const float4*>(slot + kMM) + threadIdx.x * 2;
    const float4 m0 = mm[0], m1 = mm[1];
    const float v[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, rc.g_mean, rc.alpha};
    pool = tau == 0 ? make_float2(m0.x, m0.w) : (tau == 1 ? make_float2(m0.y, m1.x) : make_float2(m0.z, m1.y));
    if (rc.literal) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += relu(v[j]);
        return 1.0f / (1.0f + __expf(-(acc / 8.0f)));
    }
    const float* prm = reinterpret_cast<const float*>(slot + kAtt);
    float h[4], w3[3];
    dense_s<4, 8>(prm, prm + 32, v, h);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = relu(h[j]);
    dense_s<3, 4>(prm + 36, prm + 48, h, w3);
    const float z = tau == 0 ? w3[0] : (tau == 1 ? w3[1] : w3[2]);
    return 1.0f / (1.0f + __expf(-z));
}

// First layer of a stack: o = relu(W_init cfg + b) (src/predictor.cpp:206-212), o_att = w o.
template <int kMM = kPayMM, int kAtt = kPayAtt, int kInit = kPayInit>
__device__ __forceinline__ void stack_start(const uint8_t* slot, int tau, const RowCtx& rc, float* oa, float2& pool) {
    const float* ini = reinterpret_cast<const float*>(slot + kInit);
    const float w = attention<kMM, kAtt>(slot, tau, rc, pool);
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // 8 outputs at a time: bounds the loads the compiler hoists
        float o[8];
        dense_s<8, 7>(ini + 56 * g, ini + 224 + 8 * g, rc.cfgv, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) oa[8 * g + j] = relu(o[j]) * w;
        asm volatile("" ::: "memory");
    }
}

template <bool kH>
__device__ __forceinline__ void store_row32(uint8_t* a, const float* v) {
#pragma unroll
    for (int c = 0; c < 4; ++c) store_chunk<kH>(a, threadIdx.x, c, 32, v + 8 * c);
}

// kH: fp16 GEMM operands (SF_PRECISION_FP16), else bf16; fp32 accumulation either way
#ifndef SF_TC_EARLY_B2
#define SF_TC_EARLY_B2 1
#endif
template <bool kH, class RC>
__global__ void __launch_bounds__(kThreads, RC::MINB)
    k_backbone_tc(const TcDesc d, const uint8_t* __restrict__ wpk, const uint8_t* __restrict__ ops,
                  const uint8_t* __restrict__ mms, int n_tiles, int64_t n, const double* __restrict__ cfg8,
                  float* __restrict__ y_out, double* __restrict__ F_out, const int* __restrict__ perm,
                  int f_stage) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[2 * RC::NS + 1];
    __shared__ uint32_t tmem_slot;
    __shared__ int s_kf[2][16];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
#ifdef SF_TC_PROFILE
    const bool prof = d.prof && blockIdx.x == 0 && tid == 0;
    long long t_last = clock64();
    const long long t_start = t_last;
#define PROF(k)                                                             \
    if (prof) {                                                             \
        long long t_now = clock64();                                        \
        atomicAdd(&g_tc_prof[k], (unsigned long long)(t_now - t_last));     \
        t_last = t_now;                                                     \
    }
#else
#define PROF(k)
#endif

    // 1024-byte aligned in the shared window; derived from smem_raw by pointer arithmetic so the
    // compiler keeps the shared address space (LDS/STS, not generic LD/ST, for every ring read)
    uint8_t* a_att = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // [128 x 32] o_att of FC-1
    uint8_t* a_od = a_att + kUmmaM * 32 * 2;            // [128 x 32] diffuse stack output (merge, K 0-31)
    uint8_t* a2 = a_od + kUmmaM * 32 * 2;               // [128 x 64] FC-2 / merge (K 32-63) / cross / head
    Ring r;
    r.base = a2 + kUmmaM * 64 * 2;
    r.full = bars;
    r.empty = bars + RC::NS;
    r.mma = bars + 2 * RC::NS;
    r.mpar = 0;

    if (warp == 0) tmem_alloc(&tmem_slot, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < 2 * RC::NS + 1; ++s)
            mbar_init(&bars[s], s >= RC::NS && s < 2 * RC::NS ? kConsumers / 32 : 1);  // empty: per warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) s_kf[tid >> 4][tid & 15] = (d.counts[tid >> 4][tid & 15] + 15) / 16 * 16;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == kConsumers / 32) {  // producer warp: keeps the ring full, off the critical path
        if ((tid & 31) == 0) {
            StepRegs cur, nxt;
            load_step(d, 0, cur);
            for (int j = 0; j < d.n_steps; ++j) {
                if (j + 1 < d.n_steps) load_step(d, j + 1, nxt);  // in flight across the slot wait
                if (j >= RC::NS) SF_WAIT(&r.empty[j % RC::NS], uint32_t(j / RC::NS - 1) & 1u, 2, j);
                issue_step<RC>(r, cur, j, wpk, ops, mms, tile, n_tiles);
                cur = nxt;
            }
        }
        return;
    }

    const int64_t q = int64_t(tile) * kUmmaM + tid;
    const bool live = q < n;
    const uint32_t tmem = tmem_slot;
    const uint32_t lane = uint32_t(warp * 32) << 16;
    const uint32_t s_att = smem_u32(a_att), s_od = smem_u32(a_od), s_a2 = smem_u32(a2);

    // conditioning (cfg_vector, src/predictor.cpp:193-202)
    RowCtx rc;
    for (int i = 0; i < 7; ++i) rc.cfgv[i] = 0.0f;
    rc.g_mean = 0.0f;
    rc.alpha = 0.0f;
    rc.literal = d.literal;
    if (live) {
        const double* c8 = cfg8 + 8 * q;
        int ng = int(c8[0]);
        for (int i = 0; i < ng; ++i) rc.g_mean += float(c8[1 + i]);
        if (ng > 0) rc.g_mean /= float(double(ng));
        rc.alpha = float(c8[7]);
        for (int i = 0; i < ng && i < 3; ++i) rc.cfgv[i] = float(c8[1 + i]);
        for (int i = 0; i < 4; ++i) rc.cfgv[3 + i] = float(c8[4 + i]);
    }

    float oa[32];  // o_att of the current layer (fp32 residual); its bf16 copy is a_att
    float2 pool;   // the current layer's (mean, max) of its feature type
    // step 0: payload of the first FC-1 step
    stack_start(wait_full<RC>(r, 0), 0, rc, oa, pool);
    release<RC>(r, 0);
    store_row32<kH>(a_att, oa);
    int j = 1;
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            const int nl = kind == 0 ? d.nl[0] : d.nl[1];
            for (int i = 0; i < nl; ++i) {
                // FC-1 = [o_att | sorted_tau, mean, max] W1^T
                PROF(7);
                const uint8_t* s1 = wait_full<RC>(r, j);
                PROF(0);
                mma_sync();
                if (tid == 0) {
                    const uint32_t b1s = smem_u32(s1);
                    issue_gemm<kH>(tmem + 0, 32, s_att, 32, b1s + kSlotW1a, false);
                    issue_gemm<kH>(tmem + 0, 32, b1s + RC::OF, s_kf[kind][i], b1s + kSlotW1b, true);
                    umma_commit(r.mma);
                }
                // while the MMA runs: the FC-1 bias with the layer's fp32 mean / max columns
                float be[32];
                {
                    const float* b1 = reinterpret_cast<const float*>(s1 + RC::OB);  // b1, W1 mean / max cols
#pragma unroll
                    for (int e = 0; e < 32; ++e) be[e] = fmaf(pool.x, b1[32 + e], fmaf(pool.y, b1[64 + e], b1[e]));
                }
                mma_wait(r);
                release<RC>(r, j);  // W1 / features consumed, bias in registers
                PROF(1);
                // FC-1 epilogue: u = relu(acc + b1) -> bf16 operand of FC-2
                {
                    float acc[32];
                    tmem_ld32(tmem + lane + 0, acc);
#pragma unroll
                    for (int e = 0; e < 32; ++e) acc[e] = relu(acc[e] + be[e]);
                    store_row32<kH>(a2, acc);
                }
                PROF(2);
                const uint8_t* s2 = wait_full<RC>(r, j + 1);
                PROF(3);
                mma_sync();
                if (tid == 0) {
                    issue_gemm<kH>(tmem + 32, 32, s_a2, 32, smem_u32(s2), false);
                    umma_commit(r.mma);
                }
                PROF(4);
                // while FC-2 runs: the next FC-1's attention weight (payload of this bundle)
                const bool last = i == nl - 1;
                float w_next = 0.0f;
                float2 pool_next = pool;
                if (!last) w_next = attention(s2, tau, rc, pool_next);
                float b2r[32];  // FC-2 bias into registers while the MMA runs
#if SF_TC_EARLY_B2
                {
                    const float4* b2 = reinterpret_cast<const float4*>(s2 + kSlotB2);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float4 v = b2[e];
                        b2r[4 * e] = v.x;
                        b2r[4 * e + 1] = v.y;
                        b2r[4 * e + 2] = v.z;
                        b2r[4 * e + 3] = v.w;
                    }
                }
#endif
                PROF(5);
                mma_wait(r);
                if (!(last && kind == 0) && SF_TC_EARLY_B2) release<RC>(r, j + 1);  // else after the stack start
                PROF(6);
                // FC-2 epilogue + residual: o = relu(acc + b2) + o_att (fp32)
                float o[32];
                {
                    tmem_ld32(tmem + lane + 32, o);
#if !SF_TC_EARLY_B2
                    for (int e = 0; e < 32; ++e) b2r[e] = reinterpret_cast<const float*>(s2 + kSlotB2)[e];
#endif
                    PROF(9);
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = relu(o[e] + b2r[e]) + oa[e];
                }
                pool = pool_next;
                if (!last) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) oa[e] = o[e] * w_next;
                    PROF(10);
                    store_row32<kH>(a_att, oa);
                    PROF(11);
                } else if (kind == 0) {  // od: K 0-31 of the merge input
                    store_row32<kH>(a_od, o);
                    stack_start(s2, tau, rc, oa, pool);  // highlight stack (once per type: not overlapped)
                    if (SF_TC_EARLY_B2) release<RC>(r, j + 1);
                    store_row32<kH>(a_att, oa);
                } else {  // oh: K 32-63 of the merge input
                    store_row32<kH>(a2, o);
                }
                if (!SF_TC_EARLY_B2) release<RC>(r, j + 1);
                j += 2;
            }
        }
        // merged_tau = relu(W_m [od; oh] + b)
        {
            const uint8_t* sm = wait_full<RC>(r, j);
            mma_sync();
            if (tid == 0) {
                issue_gemm<kH>(tmem + kColMerge, 64, s_od, 32, smem_u32(sm), false);
                issue_gemm<kH>(tmem + kColMerge, 64, s_a2, 32, smem_u32(sm) + kSlotWmHi, true);
                umma_commit(r.mma);
            }
            mma_wait(r);
            const float* bm = reinterpret_cast<const float*>(sm + kSlotBias);
            for (int half = 0; half < 2; ++half) {
                float acc[32];
                tmem_ld32(tmem + lane + kColMerge + 32 * half, acc);
#pragma unroll
                for (int e = 0; e < 32; ++e) acc[e] = relu(acc[e] + bm[32 * half + e]);
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk<kH>(a2, tid, half * 4 + c, 64, acc + 8 * c);
            }
            release<RC>(r, j);
            ++j;
        }
        // cross += W_c[:, 64 tau : 64 tau + 64] merged_tau (accumulated in TMEM)
        {
            const uint8_t* sc = wait_full<RC>(r, j);
            mma_sync();
            if (tid == 0) {
                issue_gemm<kH>(tmem + kColCross, 64, s_a2, 64, smem_u32(sc), tau > 0);
                umma_commit(r.mma);
            }
            if (tau < 2) {  // next type's first diffuse layer, while the cross MMA runs
                stack_start(sc, tau + 1, rc, oa, pool);
                store_row32<kH>(a_att, oa);
            }
            mma_wait(r);
            if (tau == 2) {  // the last cross bundle carries the cross bias
                const float* bc = reinterpret_cast<const float*>(sc + kSlotBias);
                for (int half = 0; half < 2; ++half) {
                    float h[32];
                    tmem_ld32(tmem + lane + kColCross + 32 * half, h);
#pragma unroll
                    for (int e = 0; e < 32; ++e) h[e] = relu(h[e] + bc[32 * half + e]);
#pragma unroll
                    for (int c = 0; c < 4; ++c) store_chunk<kH>(a2, tid, half * 4 + c, 64, h + 8 * c);
                }
            }
            release<RC>(r, j);
            ++j;
        }
    }
    // head 0 / 1 (64 -> 64, relu); head 2 (64 -> 3) SIMT from the head-1 bundle
    for (int l = 0; l < 2; ++l) {
        const uint8_t* sh = wait_full<RC>(r, j);
        mma_sync();
        if (tid == 0) {
            issue_gemm<kH>(tmem + kColMerge, 64, s_a2, 64, smem_u32(sh), false);
            umma_commit(r.mma);
        }
        mma_wait(r);
        const float* bh = reinterpret_cast<const float*>(sh + kSlotBias);
        float h[64];
        tmem_ld32(tmem + lane + kColMerge, h);
        tmem_ld32(tmem + lane + kColMerge + 32, h + 32);
#pragma unroll
        for (int e = 0; e < 64; ++e) h[e] = relu(h[e] + bh[e]);
        if (l == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) store_chunk<kH>(a2, tid, c, 64, h + 8 * c);
        } else {
            const float* h2 = reinterpret_cast<const float*>(sh + kSlotHead2);
            float y[3];
            dense_s<3, 64>(h2, h2 + 192, h, y);
            // f_stage: the tile's F rows (128 x 24 contiguous bytes) are staged in the free a2
            // operand buffer and stored as 16-byte chunks — full sectors whether F is device
            // memory or mapped pinned host memory written over PCIe (zero copy)
            double* fs = reinterpret_cast<double*>(a2);
            if (live) {
                for (int c = 0; c < 3; ++c) {
                    float yc = fabsf(y[c]);
                    const int64_t oq = perm ? int64_t(perm[q]) : q;  // the caller's row (locality reordering)
                    if (y_out) y_out[3 * oq + c] = yc;
                    if (F_out) {
                        const double f = pow(cfg8[8 * q + 4 + c], d.gamma) * expm1(double(yc));  // decode_prediction
                        if (f_stage)
                            fs[3 * tid + c] = f;
                        else
                            F_out[3 * oq + c] = f;
                    }
                }
            }
            if (f_stage && F_out) {
                consumer_bar_sync();
                const int64_t rem = n - int64_t(tile) * kUmmaM, rows = rem < kUmmaM ? rem : kUmmaM;
                const int chunks = int(rows * 3 / 2);  // 16-byte chunks; an odd row count leaves 8 bytes
                double* dst = F_out + int64_t(tile) * kUmmaM * 3;
                for (int k = tid; k < chunks; k += kConsumers)
                    reinterpret_cast<double2*>(dst)[k] = reinterpret_cast<const double2*>(fs)[k];
                if ((rows & 1) && tid == 0) dst[rows * 3 - 1] = fs[rows * 3 - 1];
            }
        }
        ++j;
    }
    tc_fence_before();
    consumer_bar_sync();
    if (warp == 0) tmem_dealloc(tmem, kTmemCols);
#ifdef SF_TC_PROFILE
    if (prof) atomicAdd(&g_tc_prof[8], (unsigned long long)(clock64() - t_start));
#endif
#undef PROF
}

// ---- round-robin backbone: a tile's three feature-type chains interleaved ------------
//
// The six stacks of the network (src/predictor.cpp:352-387) are independent until the per-type
// merges, and a stack is a chain of 2 x 12 small GEMMs whose cost is the tcgen05 round trip
// (issue -> commit -> mbarrier -> tcgen05.ld, ~800 cycles measured) rather than the MMA work.
// Here one CTA runs the three chains tau = 0, 1, 2 of its tile round robin — chain tau is the
// diffuse stack of type tau followed by the highlight stack of type tau — so while one chain's
// MMA is in flight the consumer warps do the other two chains' epilogues; every GEMM is the
// same operation on the same operands as in k_backbone_tc (bit-identical results). The
// diffuse output of a chain waits in TMEM (fp32) for its merge. Two CTAs per SM (two tiles,
// six chains), ~106 KB of shared memory each:
//   A[3]    the chains' [128 x 32] 16-bit operands (o_att, then u, then the next o_att)
//   big[3]  FC-1 bundles: W1[:, :32], W1[:, 32:], the tile's sorted-feature block, b1 + W1's
//           mean / max columns (the three chains' FC-1 of one layer in flight together)
//   small[3] FC-2 bundles (W2, b2 + the payload of the chain's next FC-1: the layer's mean/max
//           block, attention parameters, conditioning layer), then merge / cross / head bundles
// TMEM (256 columns): [32 tau, +32) chain accumulators, [96 + 32 tau, +32) the chains' fp32
// residuals o_att, [192 + 16 tau, +16) diffuse outputs as 16-bit pairs (the merge operand, rounded
// as k_backbone_tc rounds it); the cross accumulator [192, 256) once those are read.
namespace rr {
constexpr int NSB = 3, NSS = 3;
constexpr int SBB = 17792, OF = 5120, OB = 17408, KF = 48;  // big slot (FC-1)
constexpr int SBS = 9344;                                   // small slot
constexpr int PMM = 2304, PATT = 6400, PINIT = 6656;        // FC-2 payload offsets
constexpr int kA = kUmmaM * 32 * 2;
constexpr size_t kSmem = 128 + 3 * kA + size_t(NSB) * SBB + size_t(NSS) * SBS;
constexpr int kCols = 256, kColRes = 96, kColOd = 192, kColX = 192;
constexpr int kThreadsRR = kConsumers + 64;  // + producer warp + MMA-issuer warp
static_assert(kSlotW1b + 32 * KF * 2 <= OF && OF + kUmmaM * KF * 2 <= OB && OB + 384 <= SBB, "rr big slot");
static_assert(kSlotB2 + 128 <= PMM && PMM + kUmmaM * 32 <= PATT && PATT + 256 <= PINIT && PINIT + 1024 <= SBS &&
                  kSlotHead2 + 784 <= SBS && SBS % 128 == 0 && SBB % 128 == 0 && kA % 128 == 0,
              "rr small slot");
}  // namespace rr

// One step's copies into `dst` (a ring slot), completing on `bar`.
__device__ __forceinline__ void issue_bundle(uint8_t* dst, uint64_t* bar, const StepRegs& sr, const uint8_t* wpk,
                                             const uint8_t* ops, const uint8_t* mms, int tile, int n_tiles) {
    mbar_expect_tx(bar, uint32_t(sr.w[0].y));
#pragma unroll
    for (int c = 0; c < kMaxCopies; ++c) {
        if (c >= sr.w[0].x) break;
        const int4 c0 = sr.w[1 + 2 * c], c1 = sr.w[2 + 2 * c];
        const int kind = c0.x;
        const uint32_t off = uint32_t(c0.y), bytes = uint32_t(c0.z);
        const int64_t a = (int64_t(uint32_t(c1.y)) << 32) | uint32_t(c1.x);
        const int64_t stride = (int64_t(uint32_t(c1.w)) << 32) | uint32_t(c1.z);
        const uint8_t* src;
        if (kind == 0)
            src = wpk + a;
        else if (kind == 1)
            src = ops + a * n_tiles + int64_t(tile) * stride;
        else
            src = mms + a * int64_t(n_tiles) * 4096 + int64_t(tile) * 4096;
        bulk_g2s(dst + off, src, bytes, bar);
    }
}

template <bool kH>
__global__ void __launch_bounds__(rr::kThreadsRR, 2)
    k_backbone_rr(const TcDesc d, const uint8_t* __restrict__ wpk, const uint8_t* __restrict__ ops,
                  const uint8_t* __restrict__ mms, int n_tiles, int64_t n, const double* __restrict__ cfg8,
                  float* __restrict__ y_out, double* __restrict__ F_out, const int* __restrict__ perm,
                  int f_stage) {
    using namespace rr;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // full / empty of the big and small rings; per chain: MMA done (commit), operand ready
    // (one arrival per consumer warp, awaited by the MMA warp)
    __shared__ uint64_t bars[2 * NSB + 2 * NSS + 6];
    __shared__ uint32_t tmem_slot;
    __shared__ int s_kf[2][16];
    uint64_t* full_b = bars;
    uint64_t* empty_b = bars + NSB;
    uint64_t* full_s = bars + 2 * NSB;
    uint64_t* empty_s = bars + 2 * NSB + NSS;
    uint64_t* mbar = bars + 2 * NSB + 2 * NSS;
    uint64_t* ready = mbar + 3;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
#ifdef SF_TC_PROFILE
    const bool prof = d.prof && blockIdx.x == 0 && tid == 0;
    long long t_last = clock64();
    const long long t_start = t_last;
#define RPROF(k)                                                            \
    if (prof) {                                                             \
        long long t_now = clock64();                                        \
        atomicAdd(&g_tc_prof[k], (unsigned long long)(t_now - t_last));     \
        t_last = t_now;                                                     \
    }
#else
#define RPROF(k)
#endif
    uint8_t* abuf = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint8_t* big = abuf + 3 * kA;
    uint8_t* small = big + NSB * SBB;
    uint8_t* D[3] = {big, big + SBB, big + 2 * SBB};  // merge staging in the idle big slots (tail)
    auto A = [&](int t) { return abuf + t * kA; };

    if (warp == 0) tmem_alloc(&tmem_slot, kCols);
    if (tid == 0) {
        for (int s = 0; s < 2 * NSB + 2 * NSS + 6; ++s) {
            const bool per_warp = (s >= NSB && s < 2 * NSB) || (s >= 2 * NSB + NSS && s < 2 * NSB + 2 * NSS) ||
                                  s >= 2 * NSB + 2 * NSS + 3;
            mbar_init(&bars[s], per_warp ? kConsumers / 32 : 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) s_kf[tid >> 4][tid & 15] = (d.counts[tid >> 4][tid & 15] + 15) / 16 * 16;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const int nl0 = d.nl[0], L = d.nl[0] + d.nl[1];

    if (warp == kConsumers / 32) {  // producer: both rings, in program order
        if ((tid & 31) == 0) {
            StepRegs cur, nxt;
            load_step(d, 0, cur);
            int cnt[2] = {0, 0};
            for (int j = 0; j < d.n_steps; ++j) {
                if (j + 1 < d.n_steps) load_step(d, j + 1, nxt);
                const int cls = cur.w[0].w;  // 0 big (FC-1), 1 small
                const int c = cnt[cls]++;
                const int slot = c % 3;
                if (c >= 3) SF_WAIT(&(cls ? empty_s : empty_b)[slot], uint32_t(c / 3 - 1) & 1u, 2, j);
                issue_bundle(cls ? small + slot * SBS : big + slot * SBB, &(cls ? full_s : full_b)[slot], cur, wpk,
                             ops, mms, tile, n_tiles);
                cur = nxt;
            }
        }
        return;
    }
    if (warp == kConsumers / 32 + 1) {  // MMA issuer: every GEMM of the tile, in consumer order
        if ((tid & 31) == 0) {
            uint32_t rpar = 0;
            auto wready = [&](int t) {
                SF_WAIT(&ready[t], (rpar >> t) & 1u, 5, t);
                rpar ^= 1u << t;
                tc_fence_after();
            };
            int nb = 0, nsm = 3;  // bundles taken (the chain-start payloads are the consumers')
            auto fc1 = [&](int t, int kind, int i) {
                wready(t);
                SF_WAIT(&full_b[t], uint32_t(nb / 3) & 1u, 6, nb);
                ++nb;
                const uint32_t b1s = smem_u32(big + t * SBB);
                issue_gemm<kH>(tmem + 32 * t, 32, smem_u32(A(t)), 32, b1s + kSlotW1a, false);
                issue_gemm<kH>(tmem + 32 * t, 32, b1s + OF, s_kf[kind][i], b1s + kSlotW1b, true);
                umma_commit(&mbar[t]);
            };
            auto small_wait = [&](int t) {
                SF_WAIT(&full_s[t], uint32_t(nsm / 3) & 1u, 7, nsm);
                ++nsm;
            };
            for (int t = 0; t < 3; ++t) fc1(t, 0, 0);
            for (int l = 0; l < L; ++l) {
                for (int t = 0; t < 3; ++t) {
                    wready(t);
                    small_wait(t);
                    issue_gemm<kH>(tmem + 32 * t, 32, smem_u32(A(t)), 32, smem_u32(small + t * SBS), false);
                    umma_commit(&mbar[t]);
                }
                if (l + 1 < L)
                    for (int t = 0; t < 3; ++t) fc1(t, l + 1 < nl0 ? 0 : 1, l + 1 < nl0 ? l + 1 : l + 1 - nl0);
            }
            // merges (ready[0] = the consumers staged od and oh of every chain)
            wready(0);
            for (int t = 0; t < 3; ++t) small_wait(t);
            for (int t = 0; t < 3; ++t) {
                const uint32_t sm = smem_u32(small + t * SBS);
                issue_gemm<kH>(tmem + 64 * t, 64, smem_u32(D[t]), 32, sm, false);
                issue_gemm<kH>(tmem + 64 * t, 64, smem_u32(A(t)), 32, sm + kSlotWmHi, true);
            }
            umma_commit(&mbar[0]);
            // cross
            wready(0);
            for (int t = 0; t < 3; ++t) small_wait(t);
            for (int t = 0; t < 3; ++t) {
                const uint32_t sc = smem_u32(small + t * SBS);
                issue_gemm<kH>(tmem + kColX, 64, smem_u32(D[t]), 32, sc, t > 0);
                issue_gemm<kH>(tmem + kColX, 64, smem_u32(A(t)), 32, sc + kSlotWmHi, true);
            }
            umma_commit(&mbar[0]);
            // heads
            for (int hl = 0; hl < 2; ++hl) {
                wready(0);
                const int sh = nsm % 3;
                small_wait(sh);
                const uint32_t shp = smem_u32(small + sh * SBS);
                issue_gemm<kH>(tmem, 64, smem_u32(D[0]), 32, shp, false);
                issue_gemm<kH>(tmem, 64, smem_u32(A(0)), 32, shp + kSlotWmHi, true);
                umma_commit(&mbar[0]);
            }
        }
        return;
    }

    // ---- consumer warps: thread = query row = TMEM lane
    const int64_t q = int64_t(tile) * kUmmaM + tid;
    const bool live = q < n;
    const uint32_t lane = uint32_t(warp * 32) << 16;

    RowCtx rc;
    for (int i = 0; i < 7; ++i) rc.cfgv[i] = 0.0f;
    rc.g_mean = 0.0f;
    rc.alpha = 0.0f;
    rc.literal = d.literal;
    if (live) {
        const double* c8 = cfg8 + 8 * q;
        int ng = int(c8[0]);
        for (int i = 0; i < ng; ++i) rc.g_mean += float(c8[1 + i]);
        if (ng > 0) rc.g_mean /= float(double(ng));
        rc.alpha = float(c8[7]);
        for (int i = 0; i < ng && i < 3; ++i) rc.cfgv[i] = float(c8[1 + i]);
        for (int i = 0; i < 4; ++i) rc.cfgv[3 + i] = float(c8[4 + i]);
    }

    int nb = 0, nsm = 0;  // bundles taken from each ring (program order); chain t always uses slot t
    auto acq_big = [&]() {
        RPROF(6);
        SF_WAIT(&full_b[nb % NSB], uint32_t(nb / NSB) & 1u, 1, nb);
        RPROF(1);
        ++nb;
    };
    auto acq_small = [&]() {
        RPROF(6);
        SF_WAIT(&full_s[nsm % NSS], uint32_t(nsm / NSS) & 1u, 4, nsm);
        RPROF(2);
        ++nsm;
    };
    auto rel = [&](uint64_t* bar) {
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(bar);
    };
    // operands written by this warp -> visible to the tensor core; one arrival per warp
    auto signal = [&](int t) {
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&ready[t]);
        RPROF(3);
    };
    uint32_t mpar = 0;
    auto wait_mma = [&](int t) {
        RPROF(7);
        SF_WAIT(&mbar[t], (mpar >> t) & 1u, 3, t);
        RPROF(0);
        mpar ^= 1u << t;
        tc_fence_after();
    };

    // each chain's current layer (mean, max) of its type, kept in registers; the chain loops stay
    // rolled (one copy of the code: the unrolled kernel missed in the instruction cache)
    float2 pool0 = make_float2(0.0f, 0.0f), pool1 = pool0, pool2 = pool0;
    auto get_pool = [&](int t) { return t == 0 ? pool0 : (t == 1 ? pool1 : pool2); };
    auto set_pool = [&](int t, float2 v) {
        if (t == 0)
            pool0 = v;
        else if (t == 1)
            pool1 = v;
        else
            pool2 = v;
    };

    // chain starts: the first diffuse layer's conditioning + attention (one payload bundle each)
#pragma unroll 1
    for (int t = 0; t < 3; ++t) {
        acq_small();
        float oa[32];
        float2 pl;
        stack_start<PMM, PATT, PINIT>(small + t * SBS, t, rc, oa, pl);
        set_pool(t, pl);
        rel(&empty_s[t]);
        tmem_st32(tmem + lane + kColRes + 32 * t, oa);
        store_row32<kH>(A(t), oa);
        signal(t);
    }
    for (int l = 0; l < L; ++l) {
        // FC-1 epilogues: u = relu(acc + b1 + mean W1[:, mean] + max W1[:, max])
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
            acq_big();
            wait_mma(t);
            const float* b1 = reinterpret_cast<const float*>(big + t * SBB + OB);
            const float2 pl = get_pool(t);
            float acc[32];
            tmem_ld32(tmem + lane + 32 * t, acc);
#pragma unroll
            for (int e = 0; e < 32; ++e)
                acc[e] = relu(acc[e] + fmaf(pl.x, b1[32 + e], fmaf(pl.y, b1[64 + e], b1[e])));
            rel(&empty_b[t]);
            store_row32<kH>(A(t), acc);
            RPROF(4);
            signal(t);
        }
        // FC-2 epilogues: o = relu(acc + b2) + o_att -> the next layer's o_att
        const bool last = l == L - 1, sw = l + 1 == nl0;
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
            acq_small();
            wait_mma(t);
            const uint8_t* s2 = small + t * SBS;
            float o[32];
            {
                float res[32];
                tmem_ld32(tmem + lane + 32 * t, o);
                tmem_ld32(tmem + lane + kColRes + 32 * t, res);
                const float4* b2 = reinterpret_cast<const float4*>(s2 + kSlotB2);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float4 v = b2[e];
                    o[4 * e] = relu(o[4 * e] + v.x) + res[4 * e];
                    o[4 * e + 1] = relu(o[4 * e + 1] + v.y) + res[4 * e + 1];
                    o[4 * e + 2] = relu(o[4 * e + 2] + v.z) + res[4 * e + 2];
                    o[4 * e + 3] = relu(o[4 * e + 3] + v.w) + res[4 * e + 3];
                }
            }
            if (last) {  // the highlight output: K 32-63 of the merge input
                rel(&empty_s[t]);
                store_row32<kH>(A(t), o);
                continue;
            }
            float2 pn;
            if (sw) {  // diffuse output (16-bit, as the merge reads it) parked in TMEM; highlight stack starts
                uint32_t pk16[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk16[e] = pack16<kH>(o[2 * e], o[2 * e + 1]);
                tmem_st16(tmem + lane + kColOd + 16 * t, pk16);
                stack_start<PMM, PATT, PINIT>(s2, t, rc, o, pn);
            } else {
                const float w = attention<PMM, PATT>(s2, t, rc, pn);
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = o[e] * w;
            }
            set_pool(t, pn);
            rel(&empty_s[t]);
            tmem_st32(tmem + lane + kColRes + 32 * t, o);  // the next layer's o_att
            store_row32<kH>(A(t), o);
            RPROF(5);
            signal(t);
        }
    }
    RPROF(9);

    // merges: merged_tau = relu(W_m [od; oh] + b), od (TMEM, 16-bit) staged in the idle big slots
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        uint32_t od[16];
        tmem_ld16(tmem + lane + kColOd + 16 * t, od);
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(D[t] + canon_off(tid, 8 * c, 32)) =
                make_uint4(od[4 * c], od[4 * c + 1], od[4 * c + 2], od[4 * c + 3]);
    }
    signal(0);
    for (int t = 0; t < 3; ++t) acq_small();
    wait_mma(0);
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const float* bm = reinterpret_cast<const float*>(small + t * SBS + kSlotBias);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float acc[32];
            tmem_ld32(tmem + lane + 64 * t + 32 * half, acc);
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = relu(acc[e] + bm[32 * half + e]);
            store_row32<kH>(half ? A(t) : D[t], acc);
        }
        rel(&empty_s[t]);
    }
    signal(0);
    // cross = sum_tau W_c[:, 64 tau : 64 tau + 64] merged_tau (one accumulator)
    for (int t = 0; t < 3; ++t) acq_small();
    wait_mma(0);
    {
        const float* bc = reinterpret_cast<const float*>(small + 2 * SBS + kSlotBias);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float h[32];
            tmem_ld32(tmem + lane + kColX + 32 * half, h);
#pragma unroll
            for (int e = 0; e < 32; ++e) h[e] = relu(h[e] + bc[32 * half + e]);
            store_row32<kH>(half ? A(0) : D[0], h);
        }
    }
    for (int t = 0; t < 3; ++t) rel(&empty_s[t]);
    signal(0);
    // head 0 / 1 (64 -> 64, relu); head 2 (64 -> 3) SIMT from the head-1 bundle
    for (int hl = 0; hl < 2; ++hl) {
        const int sh = nsm % NSS;
        acq_small();
        const uint8_t* shp = small + sh * SBS;
        wait_mma(0);
        const float* bh = reinterpret_cast<const float*>(shp + kSlotBias);
        float h[64];
        tmem_ld32(tmem + lane, h);
        tmem_ld32(tmem + lane + 32, h + 32);
#pragma unroll
        for (int e = 0; e < 64; ++e) h[e] = relu(h[e] + bh[e]);
        if (hl == 0) {
            store_row32<kH>(D[0], h);
            store_row32<kH>(A(0), h + 32);
            rel(&empty_s[sh]);
            signal(0);
            continue;
        }
        const float* h2 = reinterpret_cast<const float*>(shp + kSlotHead2);
        float y[3];
        dense_s<3, 64>(h2, h2 + 192, h, y);
        double* fs = reinterpret_cast<double*>(D[1]);  // F staging (see k_backbone_tc)
        if (live) {
            for (int c = 0; c < 3; ++c) {
                const float yc = fabsf(y[c]);
                const int64_t oq = perm ? int64_t(perm[q]) : q;
                if (y_out) y_out[3 * oq + c] = yc;
                if (F_out) {
                    const double f = pow(cfg8[8 * q + 4 + c], d.gamma) * expm1(double(yc));  // decode_prediction
                    if (f_stage)
                        fs[3 * tid + c] = f;
                    else
                        F_out[3 * oq + c] = f;
                }
            }
        }
        if (f_stage && F_out) {
            consumer_bar_sync();
            const int64_t rem = n - int64_t(tile) * kUmmaM, rows = rem < kUmmaM ? rem : kUmmaM;
            const int chunks = int(rows * 3 / 2);
            double* dst = F_out + int64_t(tile) * kUmmaM * 3;
            for (int k = tid; k < chunks; k += kConsumers)
                reinterpret_cast<double2*>(dst)[k] = reinterpret_cast<const double2*>(fs)[k];
            if ((rows & 1) && tid == 0) dst[rows * 3 - 1] = fs[rows * 3 - 1];
        }
        rel(&empty_s[sh]);
    }
    RPROF(10);
    tc_fence_before();
    consumer_bar_sync();
    if (warp == 0) tmem_dealloc(tmem, kCols);
#ifdef SF_TC_PROFILE
    if (prof) atomicAdd(&g_tc_prof[8], (unsigned long long)(clock64() - t_start));
#endif
#undef RPROF
}

// ---- host-side packing ------------------------------------------------------------

// B operand of one GEMM: rows = N outputs, cols [col0, col0+cols) of W (leading dim ld), zero padded to Kp.
uint32_t pack_blob(std::vector<uint8_t>& buf, const float* W, int rows, int cols, int ld, int col0, int Kp,
                   bool f16) {
    size_t off = (buf.size() + 127) & ~size_t(127);
    size_t bytes = size_t(rows) * Kp * 2;
    buf.resize(off + bytes, 0);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < Kp; ++k) {
            float v = k < cols ? W[size_t(r) * ld + col0 + k] : 0.0f;
            if (f16) {
                __half h = __float2half_rn(v);
                std::memcpy(&buf[off + canon_off(r, k, Kp)], &h, 2);
            } else {
                __nv_bfloat16 h = __float2bfloat16_rn(v);
                std::memcpy(&buf[off + canon_off(r, k, Kp)], &h, 2);
            }
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
    if (c.n_diffuse_layers * 6 + c.n_highlight_layers * 6 + 3 * 2 + 2 + 1 > kMaxSteps) return false;
    for (int i = 0; i < c.n_diffuse_layers; ++i)
        if (c.diffuse_counts[i] > 64) return false;
    for (int i = 0; i < c.n_highlight_layers; ++i)
        if (c.highlight_counts[i] > 64) return false;
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
            L.kf[k][i] = (counts[i] + 15) / 16 * 16;  // sorted values only (mean / max: fp32 in the epilogue)
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

// The packed operands of one backbone: [0] bf16, [1] fp16 (each made on first use).
struct TcPacks {
    std::unique_ptr<TcPack> p[2];
};

void tc_prepare(sf_backbone& b, cudaStream_t s, bool f16) {
    if (!b.tc) b.tc = new TcPacks;
    auto* packs = static_cast<TcPacks*>(b.tc);
    if (packs->p[f16 ? 1 : 0]) return;
    auto pack_blob_ = [&](std::vector<uint8_t>& bf, const float* W, int rows, int cols, int ld, int col0, int Kp) {
        return pack_blob(bf, W, rows, cols, ld, col0, Kp, f16);
    };
    const sf_backbone_config& c = b.cfg;
    const BackboneLayout& L = b.layout;
    const SortLayout S = sort_layout(c);
    int kf_max = 0;
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < S.nl[k]; ++i) kf_max = std::max(kf_max, S.kf[k][i]);
    static const bool force_wide = std::getenv("SF_TC_WIDE") != nullptr;  // A/B
    const bool narrow = kf_max <= RingNarrow::KF && !force_wide;
    std::vector<float> P(size_t(L.total));
    SFB_CUDA(cudaMemcpyAsync(P.data(), b.d_params, P.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
    SFB_CUDA(cudaStreamSynchronize(s));
    auto pk = std::make_unique<TcPack>();
    pk->narrow = narrow;
    pk->tri = narrow;  // RingNarrow and RingTri share the bundle layout: chosen per launch
    std::vector<uint8_t> buf;
    std::vector<Step> steps;
    const int W = 32;
    auto push = [&](Step st) {
        st.total = 0;
        for (int k = 0; k < st.ncopy; ++k) st.total += st.c[k].bytes;
        steps.push_back(st);
    };
    // Attention payload of an FC-1 step: appended to the bundle of the step before it.
    auto add_payload = [&](int kind, int tau, int i, int64_t att_off, int64_t init_off) {
        Step& prev = steps.back();
        prev.c[prev.ncopy++] = Copy{2, uint32_t(kPayMM), uint32_t(kUmmaM * 8 * 4), 0, S.mm_layer[kind][i], 4096};
        std::vector<float> att(52, 0.0f);  // [W1 32, b1 4, W2 12, b2 3, pad]
        if (!c.literal_attention)
            for (int k = 0; k < 51; ++k) att[size_t(k)] = P[size_t(att_off + k)];
        prev.c[prev.ncopy++] = pcopy(pack_f32(buf, att), f32_bytes(att.size()), kPayAtt);
        if (i == 0) {  // conditioning layer of the stack
            std::vector<float> ini = slice(P, init_off, size_t(W * 7 + W));
            prev.c[prev.ncopy++] = pcopy(pack_f32(buf, ini), f32_bytes(ini.size()), kPayInit);
        }
        (void)tau;
    };
    steps.push_back(Step{});  // step 0: payload of the first FC-1 step only
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            const int64_t init_off = L.stack_off[kind][tau];
            int64_t off = init_off + W * 7 + W;
            for (int i = 0; i < S.nl[kind]; ++i) {
                const int64_t att_off = off;
                if (!c.literal_attention) off += 51;
                add_payload(kind, tau, i, att_off, init_off);
                const int cnt = S.counts[kind][i];
                const int K = W + cnt + 2, kf = S.kf[kind][i];
                Step st{};
                st.k2 = kf;
                st.c[0] = pcopy(pack_blob_(buf, P.data() + off, W, W, K, 0, W), W * W * 2, kSlotW1a);
                st.c[1] = pcopy(pack_blob_(buf, P.data() + off, W, cnt, K, W, kf), uint32_t(W * kf * 2), kSlotW1b);
                st.c[2] = Copy{1, uint32_t(narrow ? RingNarrow::OF : RingWide::OF), uint32_t(kUmmaM * kf * 2), 0, S.seg_prefix[kind][i][tau],
                               int64_t(kUmmaM) * kf * 2};
                // b1 [32], then the mean and max columns of W1 [32] + [32] (fp32 rank-2 update)
                std::vector<float> bmx = slice(P, off + int64_t(W) * K, W);
                for (int r = 0; r < W; ++r) bmx.push_back(P[size_t(off + int64_t(r) * K + W + cnt)]);
                for (int r = 0; r < W; ++r) bmx.push_back(P[size_t(off + int64_t(r) * K + W + cnt + 1)]);
                st.c[3] = pcopy(pack_f32(buf, bmx), f32_bytes(bmx.size()), narrow ? RingNarrow::OB : RingWide::OB);
                st.ncopy = 4;
                push(st);
                off += int64_t(W) * K + W;
                Step s2{};
                s2.k2 = W;
                s2.c[0] = pcopy(pack_blob_(buf, P.data() + off, W, W, W, 0, W), W * W * 2, 0);
                s2.c[1] = pcopy(pack_f32(buf, slice(P, off + W * W, W)), f32_bytes(W), kSlotB2);
                s2.ncopy = 2;
                push(s2);
                off += W * W + W;
            }
        }
        const int64_t mo = L.merge_off + int64_t(tau) * (64 * 64 + 64);
        Step sm{};
        sm.k2 = 64;
        sm.c[0] = pcopy(pack_blob_(buf, P.data() + mo, 64, 32, 64, 0, 32), 4096, 0);
        sm.c[1] = pcopy(pack_blob_(buf, P.data() + mo, 64, 32, 64, 32, 32), 4096, kSlotWmHi);
        sm.c[2] = pcopy(pack_f32(buf, slice(P, mo + 64 * 64, 64)), f32_bytes(64), kSlotBias);
        sm.ncopy = 3;
        push(sm);
        Step sc{};
        sc.k2 = 64;
        sc.c[0] = pcopy(pack_blob_(buf, P.data() + L.cross_off, 64, 64, 192, 64 * tau, 64), 8192, 0);
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
        sh.c[0] = pcopy(pack_blob_(buf, P.data() + L.head_off[l], 64, 64, 64, 0, 64), 8192, 0);
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
    for (Step& st : steps) {
        st.total = 0;
        for (int k = 0; k < st.ncopy; ++k) st.total += st.c[k].bytes;
    }
    // k_backbone_rr's program: the three chains' steps interleaved in the order the consumers
    // take them (chain starts; per layer three FC-1 (big ring) then three FC-2 (small ring, each
    // carrying the payload of its chain's next FC-1); merges, cross chunks, heads).
    std::vector<Step> rsteps;
    const int Lr = S.nl[0] + S.nl[1];
    pk->rr = narrow && S.nl[0] >= 1 && S.nl[1] >= 1 && 3 + 6 * Lr + 8 <= kMaxSteps;
    if (pk->rr) {
        int64_t att_o[2][3][16], w1_o[2][3][16], w2_o[2][3][16];
        for (int kind = 0; kind < 2; ++kind)
            for (int tau = 0; tau < 3; ++tau) {
                int64_t off = L.stack_off[kind][tau] + W * 7 + W;
                for (int i = 0; i < S.nl[kind]; ++i) {
                    att_o[kind][tau][i] = off;
                    if (!c.literal_attention) off += 51;
                    w1_o[kind][tau][i] = off;
                    off += int64_t(W) * (W + S.counts[kind][i] + 2) + W;
                    w2_o[kind][tau][i] = off;
                    off += W * W + W;
                }
            }
        auto payload = [&](Step& st, int kind, int tau, int i) {
            st.c[st.ncopy++] = Copy{2, uint32_t(rr::PMM), uint32_t(kUmmaM * 8 * 4), 0, S.mm_layer[kind][i], 4096};
            std::vector<float> att(52, 0.0f);
            if (!c.literal_attention)
                for (int k = 0; k < 51; ++k) att[size_t(k)] = P[size_t(att_o[kind][tau][i] + k)];
            st.c[st.ncopy++] = pcopy(pack_f32(buf, att), f32_bytes(att.size()), rr::PATT);
            if (i == 0) {
                std::vector<float> ini = slice(P, L.stack_off[kind][tau], size_t(W * 7 + W));
                st.c[st.ncopy++] = pcopy(pack_f32(buf, ini), f32_bytes(ini.size()), rr::PINIT);
            }
        };
        for (int tau = 0; tau < 3; ++tau) {
            Step st{};
            st.cls = 1;
            payload(st, 0, tau, 0);
            rsteps.push_back(st);
        }
        for (int l = 0; l < Lr; ++l) {
            const int kind = l < S.nl[0] ? 0 : 1, i = kind ? l - S.nl[0] : l;
            const int cnt = S.counts[kind][i], K = W + cnt + 2, kf = S.kf[kind][i];
            for (int tau = 0; tau < 3; ++tau) {
                const int64_t off = w1_o[kind][tau][i];
                Step st{};
                st.cls = 0;
                st.k2 = kf;
                st.c[0] = pcopy(pack_blob_(buf, P.data() + off, W, W, K, 0, W), W * W * 2, kSlotW1a);
                st.c[1] = pcopy(pack_blob_(buf, P.data() + off, W, cnt, K, W, kf), uint32_t(W * kf * 2), kSlotW1b);
                st.c[2] = Copy{1, uint32_t(rr::OF), uint32_t(kUmmaM * kf * 2), 0, S.seg_prefix[kind][i][tau],
                               int64_t(kUmmaM) * kf * 2};
                std::vector<float> bmx = slice(P, off + int64_t(W) * K, W);
                for (int r = 0; r < W; ++r) bmx.push_back(P[size_t(off + int64_t(r) * K + W + cnt)]);
                for (int r = 0; r < W; ++r) bmx.push_back(P[size_t(off + int64_t(r) * K + W + cnt + 1)]);
                st.c[3] = pcopy(pack_f32(buf, bmx), f32_bytes(bmx.size()), rr::OB);
                st.ncopy = 4;
                rsteps.push_back(st);
            }
            for (int tau = 0; tau < 3; ++tau) {
                const int64_t off = w2_o[kind][tau][i];
                Step st{};
                st.cls = 1;
                st.k2 = W;
                st.c[0] = pcopy(pack_blob_(buf, P.data() + off, W, W, W, 0, W), W * W * 2, 0);
                st.c[1] = pcopy(pack_f32(buf, slice(P, off + W * W, W)), f32_bytes(W), kSlotB2);
                st.ncopy = 2;
                if (l + 1 < Lr) {
                    const int kn = l + 1 < S.nl[0] ? 0 : 1, inx = kn ? l + 1 - S.nl[0] : l + 1;
                    payload(st, kn, tau, inx);
                }
                rsteps.push_back(st);
            }
        }
        // 64-wide bundles: W[:, 0:32] at 0, W[:, 32:64] at kSlotWmHi, bias at kSlotBias
        auto wide = [&](int64_t w_off, int ld, int col0, int64_t b_off) {
            Step st{};
            st.cls = 1;
            st.k2 = 64;
            st.c[0] = pcopy(pack_blob_(buf, P.data() + w_off, 64, 32, ld, col0, 32), 4096, 0);
            st.c[1] = pcopy(pack_blob_(buf, P.data() + w_off, 64, 32, ld, col0 + 32, 32), 4096, kSlotWmHi);
            st.ncopy = 2;
            if (b_off >= 0) st.c[st.ncopy++] = pcopy(pack_f32(buf, slice(P, b_off, 64)), f32_bytes(64), kSlotBias);
            return st;
        };
        for (int tau = 0; tau < 3; ++tau) {
            const int64_t mo = L.merge_off + int64_t(tau) * (64 * 64 + 64);
            rsteps.push_back(wide(mo, 64, 0, mo + 64 * 64));
        }
        for (int tau = 0; tau < 3; ++tau)
            rsteps.push_back(wide(L.cross_off, 192, 64 * tau, tau == 2 ? L.cross_off + 64 * 192 : -1));
        for (int l = 0; l < 2; ++l) {
            Step st = wide(L.head_off[l], 64, 0, L.head_off[l] + 64 * 64);
            if (l == 1) {
                std::vector<float> h2 = slice(P, L.head_off[2], 3 * 64 + 3);
                st.c[st.ncopy++] = pcopy(pack_f32(buf, h2), f32_bytes(h2.size()), kSlotHead2);
            }
            rsteps.push_back(st);
        }
        for (Step& st : rsteps) {
            st.total = 0;
            for (int k = 0; k < st.ncopy; ++k) st.total += st.c[k].bytes;
        }
    }
    TcDesc& d = pk->desc;
    d.nl[0] = S.nl[0];
    d.nl[1] = S.nl[1];
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < S.nl[k]; ++i) d.counts[k][i] = S.counts[k][i];
    d.literal = c.literal_attention;
    d.gamma = c.gamma;
    d.n_steps = int(steps.size());
    d.prof = std::getenv("SF_DEBUG_TC") != nullptr;
    const size_t blob_bytes = (buf.size() + 255) & ~size_t(255);
    buf.resize(blob_bytes + (steps.size() + rsteps.size()) * sizeof(Step));
    std::memcpy(buf.data() + blob_bytes, steps.data(), steps.size() * sizeof(Step));
    if (!rsteps.empty())
        std::memcpy(buf.data() + blob_bytes + steps.size() * sizeof(Step), rsteps.data(), rsteps.size() * sizeof(Step));
    SFB_CUDA(cudaMalloc(&pk->d_blobs, buf.size()));
    SFB_CUDA(cudaMemcpy(pk->d_blobs, buf.data(), buf.size(), cudaMemcpyHostToDevice));
    d.steps = reinterpret_cast<const Step*>(pk->d_blobs + blob_bytes);
    pk->desc_rr = d;
    pk->desc_rr.n_steps = int(rsteps.size());
    pk->desc_rr.steps = d.steps + steps.size();
    packs->p[f16 ? 1 : 0] = std::move(pk);
}

void tc_release(sf_backbone& b) {
    auto packs = static_cast<TcPacks*>(b.tc);
    if (!packs) return;
    for (auto& pk : packs->p)
        if (pk) cudaFree(pk->d_blobs);
    delete packs;
    b.tc = nullptr;
}

void launch_backbone_tc(const sf_backbone& b, int64_t n, const uint8_t* ops, const float* mms, const double* cfg8,
                        float* y, double* F, cudaStream_t s, const int* perm, bool f16) {
    if (n <= 0) return;
    auto packs = static_cast<const TcPacks*>(b.tc);
    const TcPack* pk = packs ? packs->p[f16 ? 1 : 0].get() : nullptr;
    if (!pk) fail(SF_ERR_INVALID_ARGUMENT, "tc backbone: operands not prepared for this precision");
    // RingTri (three chains per SM, each ~1.3x slower under the heavier sharing) or RingNarrow (two)
    // by whole waves: at C5 (7,200 tiles) RingTri measured 1.71 vs 1.97 ms (bit-identical), while a
    // 512-tile C2 batch is two waves either way and RingNarrow's faster chains win.
    // SF_TC_RING=tri|narrow forces one (A/B).
    const int64_t n_tiles64 = (n + kUmmaM - 1) / kUmmaM;
    // k_backbone_rr (the three chains of a tile interleaved, two CTAs per SM) with SF_TC_RR=1:
    // bit-identical, measured slower at C5 (2.05 vs 1.53 ms: its consumer warps are latency-bound
    // and two CTAs per SM give 8 of them where the one-chain kernel's three give 12)
    static const char* rr_env = std::getenv("SF_TC_RR");
    if (pk->rr && rr_env && rr_env[0] == '1') {
        auto kern = f16 ? k_backbone_rr<true> : k_backbone_rr<false>;
        static std::mutex rr_mu;
        static std::unordered_map<int, bool> rr_set;
        int dev = 0;
        SFB_CUDA(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lk(rr_mu);
            const int key = 2 * dev + (f16 ? 1 : 0);
            if (!rr_set[key]) {
                SFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rr::kSmem)));
                SFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                              int(cudaSharedmemCarveoutMaxShared)));
                rr_set[key] = true;
            }
        }
        const int n_tiles = int(n_tiles64);
        const int f_stage = F && !perm && (reinterpret_cast<uintptr_t>(F) & 15) == 0 ? 1 : 0;
        kern<<<n_tiles, rr::kThreadsRR, rr::kSmem, s>>>(pk->desc_rr, pk->d_blobs, ops, reinterpret_cast<const uint8_t*>(mms),
                                                 n_tiles, n, cfg8, y, F, perm, f_stage);
        SFB_CUDA(cudaGetLastError());
        count_launch();
        return;
    }
    bool tri = false;
    if (pk->tri) {
        static const char* force = std::getenv("SF_TC_RING");
        const int64_t S = sm_count();
        const double t_tri = 1.3 * double((n_tiles64 + 3 * S - 1) / (3 * S));
        const double t_nar = double((n_tiles64 + 2 * S - 1) / (2 * S));
        tri = force ? std::string(force) == "tri" : t_tri < t_nar;
    }
    size_t smem = tri ? ring_smem<RingTri>() : pk->narrow ? ring_smem<RingNarrow>() : ring_smem<RingWide>();
    static const bool solo = std::getenv("SF_DEBUG_TC") && std::atoi(std::getenv("SF_DEBUG_TC")) == 2;
    if (solo) smem = 200 * 1024;  // one CTA per SM: uncontended chain latency
    auto kern = tri          ? (f16 ? k_backbone_tc<true, RingTri> : k_backbone_tc<false, RingTri>)
                : pk->narrow ? (f16 ? k_backbone_tc<true, RingNarrow> : k_backbone_tc<false, RingNarrow>)
                             : (f16 ? k_backbone_tc<true, RingWide> : k_backbone_tc<false, RingWide>);
    // function attributes are per device: remember the size set on each device and variant (a
    // process may drive several GPUs, from several threads)
    static std::mutex attr_mu;
    static std::unordered_map<int, size_t> attr_set;
    int dev = 0;
    SFB_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(attr_mu);
        const int key = 8 * dev + (f16 ? 1 : 0) + (pk->narrow ? 2 : 0) + (tri ? 4 : 0);
        if (attr_set[key] != smem) {
            SFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            SFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          int(cudaSharedmemCarveoutMaxShared)));
            attr_set[key] = smem;
            // co-resident tiles per SM by design (RingTri: 3 x (128 registers x 160 threads,
            // ~70 KB smem, 128 TMEM columns); RingWide: 2); the occupancy API does not model
            // TMEM, so no runtime check here.
        }
    }
    const int n_tiles = int((n + kUmmaM - 1) / kUmmaM);
    const int f_stage = F && !perm && (reinterpret_cast<uintptr_t>(F) & 15) == 0 ? 1 : 0;
    kern<<<n_tiles, kThreads, smem, s>>>(pk->desc, pk->d_blobs, ops, reinterpret_cast<const uint8_t*>(mms), n_tiles, n,
                                        cfg8, y, F, perm, f_stage);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void tc_read_prof(unsigned long long* out) {
    SFB_CUDA(cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(unsigned long long) * 16));
    unsigned long long z[16] = {};
    SFB_CUDA(cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z)));
}

}  // namespace sfb
