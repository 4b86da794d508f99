// sf_tc.cu — the backbone forward on 5th-generation tensor cores (tcgen05).
//
// One CTA = one tile of 128 shading points = UMMA_M. Thread t owns query row t,
// which is also TMEM lane t, so every epilogue is a private tcgen05.ld of the
// thread's own accumulator row. Every dense layer of the reference network
// (src/predictor.cpp:206-235, 352-387) whose K is large enough becomes one
// tcgen05.mma chain D[128 x N] (fp32, TMEM) = A[128 x K] (bf16, SMEM) * W^T:
//
//   FC-1 (N=32, K = 32 + n_i + 2 -> padded to 16), FC-2 (N=32, K=32),
//   per-type merge (N=64, K=64), cross merge (N=64, K=192 as 3 x 64),
//   head 0/1 (N=64, K=64)
//
// The reference's W[out][in] row-major is exactly UMMA's K-major B operand, so
// weights are pre-packed once (tc_prepare) into the no-swizzle canonical layout
// and streamed per layer with cp.async.bulk (TMA bulk copy) into a 2-deep SMEM
// ring, the copy of layer j+1 overlapping layer j. The tiny SIMT parts (the 7->32
// conditioning layer, the 8->4->3 channel attention and the 64->3 output layer)
// stay FP32 on the CUDA cores, as does the residual stream o.
//
// Precision: bf16 operands (weights, o_att, features, u, merges), fp32
// accumulation and fp32 residual/bias/activation; see tests/test_gpu_parity.py
// test_bf16_* for the stated tolerance.
#include <cuda_bf16.h>

#include <cstring>
#include <vector>

#include "sf_internal.h"

namespace sfb {

namespace {

constexpr int kTile = 128;        // queries per CTA (UMMA_M)
constexpr int kThreads = 128;     // one thread per query row / TMEM lane
constexpr int kTmemCols = 128;    // fc1 [0,32), fc2 [32,64), merge/cross/head [64,128)
constexpr int kBlobMax = 8192;    // largest weight blob (64 x 64 bf16)
constexpr int kMaxBlobs = 128;

// --- UMMA descriptors (no swizzle, K-major canonical layout) -------------------------
// element (r, k) of an R x K operand lives at byte (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2
// with LBO = 128 (adjacent 8-element K chunks) and SBO = K*16 (adjacent 8-row groups).
__host__ __device__ constexpr uint32_t canon_off(int r, int k, int K) {
    return uint32_t((r >> 3) * (K * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;  // descriptor version for tcgen05
    return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kTile >> 4) << 24);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "SF_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra SF_DONE_%=;\n\t"
        "bra SF_WAIT_%=;\n"
        "SF_DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 consecutive fp32 TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Row `row` of a K-wide canonical operand: 8 elements (16 B) per chunk.
__device__ __forceinline__ void store_chunk(uint8_t* base, int row, int kchunk, int K, const float* v8) {
    uint4 u;
    u.x = pack_bf16(v8[0], v8[1]);
    u.y = pack_bf16(v8[2], v8[3]);
    u.z = pack_bf16(v8[4], v8[5]);
    u.w = pack_bf16(v8[6], v8[7]);
    *reinterpret_cast<uint4*>(base + canon_off(row, kchunk * 8, K)) = u;
}

struct Blob {
    uint32_t off;    // byte offset into the packed weight buffer
    uint16_t bytes;  // blob size
    uint16_t K;      // operand K (multiple of 16)
};

struct TcDesc {
    int nl[2];
    int counts[2][16];
    int slice_off[2][16];
    int W, M, H;
    int literal;
    double gamma;
    int64_t stack_off[2][3];
    int64_t merge_off, cross_off, head_off[3];
    int n_blobs;
    int kp1_max;
    Blob blobs[kMaxBlobs];
};

struct TcState {
    uint8_t* smem_a1;  // fc1 A [128 x kp1_max]
    uint8_t* smem_a2;  // fc2/merge/head A [128 x 64]
    uint8_t* smem_ac;  // cross A [128 x 192]
    uint8_t* smem_w[2];
    uint64_t* wbar;    // [2]
    uint64_t* mbar;
    uint32_t tmem;
    uint32_t wpar[2];
    uint32_t mpar;
    int next_blob;     // next blob index to be loaded
    int cur_blob;      // blob index consumed by the next MMA
};

// Thread 0: start the bulk copy of blob `j` into ring slot j % 2.
__device__ __forceinline__ void issue_blob(TcState& s, const TcDesc& d, const uint8_t* wpk, int j) {
    if (j >= d.n_blobs) return;
    const Blob& b = d.blobs[j];
    uint64_t* bar = &s.wbar[j & 1];
    mbar_expect_tx(bar, b.bytes);
    bulk_g2s(s.smem_w[j & 1], wpk + b.off, b.bytes, bar);
}

// One synchronous GEMM step: D[tmem_col, +N) (+)= A * Wblob^T, then wait.
// Called by all threads after their SMEM operand rows are written.
__device__ __forceinline__ void gemm_step(TcState& s, const TcDesc& d, const uint8_t* wpk,
                                          uint32_t a_saddr, uint32_t a_sbo, int n, uint32_t tmem_col,
                                          bool accumulate) {
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    const int j = s.cur_blob;
    const int slot = j & 1;
    if (threadIdx.x == 0) {
        mbar_wait(&s.wbar[slot], s.wpar[slot]);
        tc_fence_after();
        const Blob& b = d.blobs[j];
        const uint32_t w_saddr = smem_u32(s.smem_w[slot]);
        const uint32_t b_sbo = uint32_t(b.K) * 16;
        const uint32_t id = idesc_bf16(n);
        for (int k = 0; k < b.K / 16; ++k) {
            uint64_t da = smem_desc(a_saddr + k * 256, 128, a_sbo);
            uint64_t db = smem_desc(w_saddr + k * 256, 128, b_sbo);
            umma_bf16(s.tmem + tmem_col, da, db, id, (accumulate || k > 0) ? 1u : 0u);
        }
        umma_commit(s.mbar);
        // ring slot (j+1)&1 was read by MMA j-1, which completed before this step
        issue_blob(s, d, wpk, j + 1);
    }
    s.wpar[slot] ^= 1;
    s.cur_blob = j + 1;
    mbar_wait(s.mbar, s.mpar);
    s.mpar ^= 1;
    tc_fence_after();
}

__device__ __forceinline__ float relu(float v) { return v > 0.0f ? v : 0.0f; }

// dense y = W x + b (FP32 SIMT, sequential accumulation with FMA)
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
    k_backbone_tc(TcDesc d, const float* __restrict__ P, const uint8_t* __restrict__ wpk, int64_t n,
                  const float* __restrict__ slices, const double* __restrict__ cfg8, float* __restrict__ y_out,
                  double* __restrict__ F_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[3];
    __shared__ uint32_t tmem_slot;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int64_t q = int64_t(blockIdx.x) * kTile + tid;
    const bool live = q < n;
    const int W = d.W;  // == 32 (tc_supported)

    TcState s;
    uintptr_t base = (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023);
    s.smem_a1 = reinterpret_cast<uint8_t*>(base);
    s.smem_a2 = s.smem_a1 + kTile * d.kp1_max * 2;
    s.smem_ac = s.smem_a2 + kTile * 64 * 2;
    s.smem_w[0] = s.smem_ac + kTile * 192 * 2;
    s.smem_w[1] = s.smem_w[0] + kBlobMax;
    s.wbar = bars;
    s.mbar = bars + 2;
    s.wpar[0] = s.wpar[1] = 0;
    s.mpar = 0;
    s.cur_blob = 0;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    s.tmem = tmem_slot;
    if (tid == 0) issue_blob(s, d, wpk, 0);
    const uint32_t lane_base = uint32_t(warp * 32) << 16;

    // ---- conditioning (make_config / cfg_vector, src/predictor.cpp:193-202)
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
        cfgv[3] = float(c8[4]);
        cfgv[4] = float(c8[5]);
        cfgv[5] = float(c8[6]);
        cfgv[6] = float(c8[7]);
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
                const float* sl = slices + int64_t(d.slice_off[kind][i]) * n + q;
                // channel attention (src/neural.cpp:473-491), FP32
                float v[8] = {0, 0, 0, 0, 0, 0, g_mean, alpha};
                if (live)
                    for (int t = 0; t < 3; ++t) {
                        v[t] = __ldg(sl + int64_t(t * (cnt + 2) + cnt) * n);
                        v[3 + t] = __ldg(sl + int64_t(t * (cnt + 2) + cnt + 1) * n);
                    }
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
                // FC-1 operand row: [o_att | sorted_tau | mean | max | 0...]
                const int K1 = d.blobs[s.cur_blob].K;
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk(s.smem_a1, tid, c, K1, oa + 8 * c);
                const float* st = sl + int64_t(tau * (cnt + 2)) * n;
                for (int c = 4; c < K1 / 8; ++c) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        int k = c * 8 + e - 32;
                        v8[e] = (live && k < cnt + 2) ? __ldg(st + int64_t(k) * n) : 0.0f;
                    }
                    store_chunk(s.smem_a1, tid, c, K1, v8);
                }
                gemm_step(s, d, wpk, smem_u32(s.smem_a1), uint32_t(K1) * 16, 32, 0, false);
                // FC-1 epilogue: u = relu(acc + b1) -> bf16 operand of FC-2
                const float* b1 = P + off + int64_t(W) * (W + cnt + 2);
                float acc[32];
                tmem_ld32(s.tmem + lane_base + 0, acc);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float v8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + __ldg(b1 + 8 * c + e));
                    store_chunk(s.smem_a2, tid, c, 32, v8);
                }
                off += int64_t(W) * (W + cnt + 2) + W;
                gemm_step(s, d, wpk, smem_u32(s.smem_a2), 32 * 16, 32, 32, false);
                // FC-2 epilogue + residual: o = relu(acc + b2) + o_att (fp32)
                const float* b2 = P + off + W * W;
                tmem_ld32(s.tmem + lane_base + 32, acc);
#pragma unroll
                for (int j = 0; j < 32; ++j) o[j] = relu(acc[j] + __ldg(b2 + j)) + oa[j];
                off += W * W + W;
            }
            if (kind == 0) {
#pragma unroll
                for (int j = 0; j < 16; ++j) od_pk[j] = pack_bf16(o[2 * j], o[2 * j + 1]);
            } else {
                // merge operand row [od | oh] (K = 64)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(s.smem_a2 + canon_off(tid, 8 * c, 64)) =
                        make_uint4(od_pk[4 * c], od_pk[4 * c + 1], od_pk[4 * c + 2], od_pk[4 * c + 3]);
#pragma unroll
                for (int c = 0; c < 4; ++c) store_chunk(s.smem_a2, tid, 4 + c, 64, o + 8 * c);
            }
        }
        // merged_tau = relu(W_m [od; oh] + b) -> columns [64 tau, 64 tau + 64) of the cross operand
        gemm_step(s, d, wpk, smem_u32(s.smem_a2), 64 * 16, 64, 64, false);
        const float* bm = P + d.merge_off + int64_t(tau) * (64 * 64 + 64) + 64 * 64;
        for (int half = 0; half < 2; ++half) {
            float acc[32];
            tmem_ld32(s.tmem + lane_base + 64 + 32 * half, acc);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v8[e] = relu(acc[8 * c + e] + __ldg(bm + 32 * half + 8 * c + e));
                store_chunk(s.smem_ac, tid, tau * 8 + half * 4 + c, 192, v8);
            }
        }
    }
    // cross = relu(W_c [m0; m1; m2] + b): K = 192 streamed as three 64-wide blobs
    for (int c = 0; c < 3; ++c)
        gemm_step(s, d, wpk, smem_u32(s.smem_ac) + c * 8 * 128, 192 * 16, 64, 64, c > 0);
    float h[64];
    {
        const float* bc = P + d.cross_off + 64 * 192;
        tmem_ld32(s.tmem + lane_base + 64, h);
        tmem_ld32(s.tmem + lane_base + 96, h + 32);
#pragma unroll
        for (int j = 0; j < 64; ++j) h[j] = relu(h[j] + __ldg(bc + j));
    }
    for (int l = 0; l < 2; ++l) {
#pragma unroll
        for (int c = 0; c < 8; ++c) store_chunk(s.smem_a2, tid, c, 64, h + 8 * c);
        gemm_step(s, d, wpk, smem_u32(s.smem_a2), 64 * 16, 64, 64, false);
        const float* bh = P + d.head_off[l] + 64 * 64;
        tmem_ld32(s.tmem + lane_base + 64, h);
        tmem_ld32(s.tmem + lane_base + 96, h + 32);
#pragma unroll
        for (int j = 0; j < 64; ++j) h[j] = relu(h[j] + __ldg(bh + j));
    }
    // output layer 64 -> 3 (FP32 SIMT), |x|, decode_prediction
    float y[3];
    dense_simt(P + d.head_off[2], P + d.head_off[2] + 3 * 64, 3, 64, h, y);
    if (live) {
        for (int c = 0; c < 3; ++c) {
            float yc = fabsf(y[c]);
            if (y_out) y_out[3 * q + c] = yc;
            if (F_out) F_out[3 * q + c] = pow(alb[c], d.gamma) * expm1(double(yc));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s.tmem), "r"(kTmemCols));
}

// ---- host-side packing -----------------------------------------------------------------

struct TcPack {
    uint8_t* d_blobs = nullptr;
    size_t bytes = 0;
    TcDesc desc{};
};

void pack_blob(std::vector<uint8_t>& buf, std::vector<Blob>& blobs, const float* W, int rows, int cols, int ld,
               int col0, int Kp) {
    // B operand of one GEMM: rows = N outputs, K = Kp (cols [col0, col0+cols) of W, zero padded)
    size_t off = (buf.size() + 127) & ~size_t(127);
    size_t bytes = size_t(rows) * Kp * 2;
    buf.resize(off + bytes, 0);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < Kp; ++k) {
            float v = k < cols ? W[size_t(r) * ld + col0 + k] : 0.0f;
            __nv_bfloat16 h = __float2bfloat16_rn(v);
            std::memcpy(&buf[off + canon_off(r, k, Kp)], &h, 2);
        }
    blobs.push_back(Blob{uint32_t(off), uint16_t(bytes), uint16_t(Kp)});
}

}  // namespace

bool tc_supported(const sf_backbone_config& c) {
    if (c.width != 32 || c.merge_width != 64 || c.head_width != 64) return false;
    for (int i = 0; i < c.n_diffuse_layers; ++i)
        if (c.diffuse_counts[i] + 2 + 32 > 96) return false;
    for (int i = 0; i < c.n_highlight_layers; ++i)
        if (c.highlight_counts[i] + 2 + 32 > 96) return false;
    return true;
}

void tc_prepare(sf_backbone& b, cudaStream_t s) {
    if (b.tc) return;
    const sf_backbone_config& c = b.cfg;
    const BackboneLayout& L = b.layout;
    std::vector<float> P(size_t(L.total));
    SFB_CUDA(cudaMemcpyAsync(P.data(), b.d_params, P.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
    SFB_CUDA(cudaStreamSynchronize(s));
    auto pk = new TcPack();
    TcDesc& d = pk->desc;
    std::vector<uint8_t> buf;
    std::vector<Blob> blobs;
    const int W = 32;
    d.kp1_max = 0;
    for (int tau = 0; tau < 3; ++tau) {
        for (int kind = 0; kind < 2; ++kind) {
            int nl = kind == 0 ? c.n_diffuse_layers : c.n_highlight_layers;
            const int* counts = kind == 0 ? c.diffuse_counts : c.highlight_counts;
            int64_t off = L.stack_off[kind][tau] + W * 7 + W;
            for (int i = 0; i < nl; ++i) {
                if (!c.literal_attention) off += 51;
                int K = W + counts[i] + 2;
                int Kp = (K + 15) / 16 * 16;
                d.kp1_max = std::max(d.kp1_max, Kp);
                pack_blob(buf, blobs, P.data() + off, W, K, K, 0, Kp);
                off += int64_t(W) * K + W;
                pack_blob(buf, blobs, P.data() + off, W, W, W, 0, W);
                off += W * W + W;
            }
        }
        pack_blob(buf, blobs, P.data() + L.merge_off + int64_t(tau) * (64 * 64 + 64), 64, 64, 64, 0, 64);
    }
    for (int k = 0; k < 3; ++k) pack_blob(buf, blobs, P.data() + L.cross_off, 64, 64, 192, 64 * k, 64);
    for (int l = 0; l < 2; ++l) pack_blob(buf, blobs, P.data() + L.head_off[l], 64, 64, 64, 0, 64);
    if (blobs.size() > size_t(kMaxBlobs)) fail(SF_ERR_INVALID_ARGUMENT, "tc backbone: too many layers");
    d.n_blobs = int(blobs.size());
    for (size_t i = 0; i < blobs.size(); ++i) d.blobs[i] = blobs[i];
    pk->bytes = buf.size();
    SFB_CUDA(cudaMalloc(&pk->d_blobs, buf.size()));
    SFB_CUDA(cudaMemcpy(pk->d_blobs, buf.data(), buf.size(), cudaMemcpyHostToDevice));
    // network description (shared with the fp32 kernel's slice layout)
    d.nl[0] = c.n_diffuse_layers;
    d.nl[1] = c.n_highlight_layers;
    int so = 0;
    for (int kind = 0; kind < 2; ++kind) {
        int nl = d.nl[kind];
        const int* counts = kind == 0 ? c.diffuse_counts : c.highlight_counts;
        for (int i = 0; i < nl; ++i) {
            d.counts[kind][i] = counts[i];
            d.slice_off[kind][i] = so;
            so += 3 * (counts[i] + 2);
        }
    }
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
    b.tc = pk;
}

void tc_release(sf_backbone& b) {
    auto pk = static_cast<TcPack*>(b.tc);
    if (!pk) return;
    cudaFree(pk->d_blobs);
    delete pk;
    b.tc = nullptr;
}

static size_t tc_smem_bytes(const TcDesc& d) {
    return 1024 + size_t(kTile) * d.kp1_max * 2 + kTile * 64 * 2 + kTile * 192 * 2 + 2 * kBlobMax;
}

void launch_backbone_tc(const sf_backbone& b, int64_t n, const float* slices, const double* cfg8, float* y,
                        double* F, cudaStream_t s) {
    if (n <= 0) return;
    auto pk = static_cast<const TcPack*>(b.tc);
    size_t smem = tc_smem_bytes(pk->desc);
    static bool attr_set = false;
    if (!attr_set) {
        SFB_CUDA(cudaFuncSetAttribute(k_backbone_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_set = true;
    }
    unsigned grid = unsigned((n + kTile - 1) / kTile);
    k_backbone_tc<<<grid, kThreads, smem, s>>>(pk->desc, b.d_params, pk->d_blobs, n, slices, cfg8, y, F);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
