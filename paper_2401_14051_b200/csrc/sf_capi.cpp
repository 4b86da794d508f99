// sf_capi.cpp — the C ABI (include/scatterfield_b200.h) and the native host
// runtime behind it: handle ownership, host<->device staging, parameter layout
// and initialisation, Gauss-Legendre nodes, stream-ordered scratch memory and
// query chunking. Every entry point converts exceptions to a status code plus a
// thread-local message (reference Errc semantics, inc/error.h:11-32).
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <unordered_map>
#include <string>
#include <vector>

#include "sf_internal.h"
#include "sf_umma.cuh"

using sfb::fail;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& fn) {
    try {
        fn();
        return SF_OK;
    } catch (const sfb::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return SF_ERR_NUMERIC;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SF_ERR_INVALID_ARGUMENT;
    }
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear: unregistered host memory
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device alias of pinned (page-locked, mapped) host memory, else nullptr. The backbone writes
// F into such a buffer in place (16-byte chunks over PCIe, overlapped with the tiles still
// computing) instead of a copy after the last tile (SF_NO_ZERO_COPY=1: copy).
void* mapped_alias(const void* p) {
    static const bool off = std::getenv("SF_NO_ZERO_COPY") != nullptr;
    if (!p || off) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Stream-ordered scratch buffer.
template <typename T>
struct Scratch {
    T* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(size_t n, cudaStream_t st) { alloc(n, st); }
    void alloc(size_t n, cudaStream_t st) {
        s = st;
        keep_pool();
        if (n) SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st));
    }
    // Per-call scratch comes from the device's stream-ordered pool; keep its memory mapped
    // between calls (the default release threshold of 0 unmaps it at every synchronise,
    // and re-mapping ~100 MB of operand blocks per query batch costs more than the batch).
    static void keep_pool() {
        static thread_local int done_dev = -1;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        done_dev = dev;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

// Input array: device pointer passed through, host array staged to the device.
template <typename T>
struct In {
    const T* d = nullptr;
    Scratch<T> buf;
    In(const T* src, size_t n, cudaStream_t s) {
        if (!src || n == 0) return;
        if (is_device_ptr(src)) {
            d = src;
            return;
        }
        buf.alloc(n, s);
        SFB_CUDA(cudaMemcpyAsync(buf.p, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
        d = buf.p;
    }
};

// Output array: device pointer written directly, host array copied back by finish().
template <typename T>
struct Out {
    T* host = nullptr;
    T* d = nullptr;
    size_t n = 0;
    Scratch<T> buf;
    cudaStream_t s;
    Out(T* dst, size_t count, cudaStream_t st) : n(count), s(st) {
        if (!dst || n == 0) return;
        if (is_device_ptr(dst)) {
            d = dst;
            return;
        }
        host = dst;
        buf.alloc(n, s);
        d = buf.p;
    }
    void finish() {
        if (host) SFB_CUDA(cudaMemcpyAsync(host, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
};

void sync(cudaStream_t s) { SFB_CUDA(cudaStreamSynchronize(s)); }

sf_grid* new_grid(int nx, int ny, int nz, double vs, const double o[3]) {
    if (nx <= 0 || ny <= 0 || nz <= 0) fail(SF_ERR_BAD_DIMS, "density grid: dims must be positive");
    if (!(vs > 0.0)) fail(SF_ERR_BAD_VALUE, "density grid: voxel_size must be positive");
    // the kernels index voxels with 32-bit integers
    if (int64_t(nx) * ny * nz >= (int64_t(1) << 31)) fail(SF_ERR_BAD_DIMS, "density grid: more than 2^31 - 1 voxels");
    auto g = std::make_unique<sf_grid>();
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    g->vs = vs;
    for (int i = 0; i < 3; ++i) g->origin[i] = o[i];
    // DensityGrid::bounds: origin + Vec3{nx*vs, ny*vs, nz*vs} (src/volume_grid.cpp:35-38)
    g->hi[0] = o[0] + nx * vs;
    g->hi[1] = o[1] + ny * vs;
    g->hi[2] = o[2] + nz * vs;
    SFB_CUDA(cudaMalloc(&g->d, g->count() * sizeof(float)));
    return g.release();
}

void free_grid(sf_grid* g) {
    if (!g) return;
    if (g->owned && g->d) {
        if (g->pooled)
            cudaFreeAsync(g->d, g->pool_stream);
        else
            cudaFree(g->d);
    }
    delete g;
}

// Intermediate grid of a build (graded fields, conv outputs): stream-ordered pool memory,
// so allocating and freeing it never synchronises the device.
sf_grid* new_scratch_grid(int nx, int ny, int nz, double vs, const double o[3], cudaStream_t s) {
    auto g = std::make_unique<sf_grid>();
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    g->vs = vs;
    for (int i = 0; i < 3; ++i) {
        g->origin[i] = o[i];
        g->hi[i] = o[i] + (i == 0 ? nx : i == 1 ? ny : nz) * vs;
    }
    Scratch<float>::keep_pool();
    SFB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&g->d), g->count() * sizeof(float), s));
    g->pooled = true;
    g->pool_stream = s;
    return g.release();
}

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// ---- reference RNG + init (inc/rng.h:12-66, src/neural.cpp:444-452) ----------------
uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Pcg32 {
    uint64_t state = 0, inc = 0;
    Pcg32(uint64_t seed, uint64_t seq) {
        inc = (splitmix64(seq) << 1u) | 1u;
        next();
        state += splitmix64(seed);
        next();
    }
    uint32_t next() {
        uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        uint32_t xs = uint32_t(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = uint32_t(old >> 59u);
        return (xs >> rot) | (xs << ((~rot + 1u) & 31));
    }
    double next_double() {
        uint64_t hi = next();
        uint64_t lo = next();
        return double((hi << 21) ^ (lo >> 11)) * 0x1p-53;
    }
};

// walk_params (src/predictor.cpp:62-109): fn(rows, cols, fan_in), cols = 0 for biases.
template <typename F>
void walk_params(const sf_backbone_config& c, F&& fn) {
    const int W = c.width;
    for (int k = 0; k < 2; ++k) {
        int nl = k == 0 ? c.n_diffuse_layers : c.n_highlight_layers;
        const int* counts = k == 0 ? c.diffuse_counts : c.highlight_counts;
        for (int t = 0; t < 3; ++t) {
            fn(W, 7, 7);
            fn(W, 0, 0);
            for (int i = 0; i < nl; ++i) {
                if (!c.literal_attention) {
                    fn(4, 8, 8);
                    fn(4, 0, 0);
                    fn(3, 4, 4);
                    fn(3, 0, 0);
                }
                int ld = counts[i] + 2;
                fn(W, W + ld, W + ld);
                fn(W, 0, 0);
                fn(W, W, W);
                fn(W, 0, 0);
            }
        }
    }
    const int M = c.merge_width;
    for (int t = 0; t < 3; ++t) {
        fn(M, 2 * W, 2 * W);
        fn(M, 0, 0);
    }
    fn(M, 3 * M, 3 * M);
    fn(M, 0, 0);
    const int H = c.head_width;
    const int outs[3] = {H, H, 3}, ins[3] = {M, H, H};
    for (int l = 0; l < 3; ++l) {
        fn(outs[l], ins[l], ins[l]);
        fn(outs[l], 0, 0);
    }
}

BackboneLayout make_layout(const sf_backbone_config& c) {
    BackboneLayout L{};
    int64_t off = 0;
    int idx = 0;
    // per-stack tensor counts: 2 + nl*(4 or 8)
    const int per_blk = c.literal_attention ? 4 : 8;
    const int n_d = 2 + c.n_diffuse_layers * per_blk, n_h = 2 + c.n_highlight_layers * per_blk;
    walk_params(c, [&](int rows, int cols, int) {
        // record the start of each stack / merge / cross / head tensor group
        int i = idx;
        if (i < 3 * n_d) {
            if (i % n_d == 0) L.stack_off[0][i / n_d] = off;
        } else if (i < 3 * n_d + 3 * n_h) {
            int j = i - 3 * n_d;
            if (j % n_h == 0) L.stack_off[1][j / n_h] = off;
        } else {
            int j = i - 3 * n_d - 3 * n_h;
            if (j == 0) L.merge_off = off;
            if (j == 6) L.cross_off = off;
            if (j == 8) L.head_off[0] = off;
            if (j == 10) L.head_off[1] = off;
            if (j == 12) L.head_off[2] = off;
        }
        off += int64_t(rows) * (cols > 0 ? cols : 1);
        ++idx;
    });
    L.total = off;
    return L;
}

std::vector<float> he_init(const sf_backbone_config& c) {
    std::vector<float> out;
    uint64_t ordinal = 0;
    walk_params(c, [&](int rows, int cols, int fan_in) {
        size_t n = size_t(rows) * size_t(cols > 0 ? cols : 1);
        uint64_t seed = splitmix64(c.seed + 0x5eedu * (ordinal + 1));
        if (fan_in > 0) {
            double bound = std::sqrt(6.0 / double(fan_in));
            Pcg32 rng(seed, 0xfeedu);
            for (size_t i = 0; i < n; ++i) out.push_back(float((2.0 * rng.next_double() - 1.0) * bound));
        } else {
            out.insert(out.end(), n, 0.0f);
        }
        ++ordinal;
    });
    return out;
}

// Gauss-Legendre nodes (src/quadrature.cpp:16-44), same Newton iteration.
void gauss_legendre(int n, std::vector<double>& x_out, std::vector<double>& w_out) {
    x_out.assign(size_t(n), 0.0);
    w_out.assign(size_t(n), 0.0);
    const int m = (n + 1) / 2;
    for (int i = 0; i < m; ++i) {
        double x = std::cos(3.14159265358979323846 * (i + 0.75) / (n + 0.5));
        double pp = 0.0;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1.0, p1 = 0.0;
            for (int j = 0; j < n; ++j) {
                double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j + 1.0) * x * p1 - j * p2) / (j + 1.0);
            }
            pp = n * (x * p0 - p1) / (x * x - 1.0);
            double dx = p0 / pp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        x_out[size_t(i)] = -x;
        x_out[size_t(n - 1 - i)] = x;
        double w = 2.0 / ((1.0 - x * x) * pp * pp);
        w_out[size_t(i)] = w;
        w_out[size_t(n - 1 - i)] = w;
    }
}

void validate_backbone_config(const sf_backbone_config& c) {
    if (c.n_diffuse_layers < 1 || c.n_highlight_layers < 1 || c.n_diffuse_layers > 16 ||
        c.n_highlight_layers > 16)
        fail(SF_ERR_INVALID_ARGUMENT, "backbone needs 1..16 layers per template kind");
    if (c.width < 1 || c.merge_width < 1 || c.head_width < 1)
        fail(SF_ERR_INVALID_ARGUMENT, "backbone widths must be positive");
    for (int i = 0; i < c.n_diffuse_layers; ++i)
        if (c.diffuse_counts[i] < 1) fail(SF_ERR_INVALID_ARGUMENT, "layer counts must be positive");
    for (int i = 0; i < c.n_highlight_layers; ++i)
        if (c.highlight_counts[i] < 1) fail(SF_ERR_INVALID_ARGUMENT, "layer counts must be positive");
}

void validate_albedo(const double a[3]) {
    for (int i = 0; i < 3; ++i)
        if (!(a[i] > 0.0 && a[i] < 1.0)) fail(SF_ERR_BAD_VALUE, "albedo components must lie in (0,1)");
}

void validate_phase_model(const sf_phase_model& m) {
    if (m.kind < 0 || m.kind > 2) fail(SF_ERR_BAD_VALUE, "phase: unknown kind");
    if (m.kind == SF_PHASE_ISOTROPIC) return;
    if (m.n_lobes < 1 || m.n_lobes > 3) fail(SF_ERR_BAD_VALUE, "phase: model has no lobes");
    double sum = 0.0;
    for (int k = 0; k < m.n_lobes; ++k) {
        if (!(m.weight[k] >= 0.0)) fail(SF_ERR_BAD_VALUE, "phase: lobe weight must be nonnegative");
        if (!(m.g[k] > -1.0 && m.g[k] < 1.0)) fail(SF_ERR_BAD_VALUE, "phase: asymmetry must lie in (-1, 1)");
        sum += m.weight[k];
    }
    if (std::abs(sum - 1.0) > 1e-9) fail(SF_ERR_BAD_VALUE, "phase: lobe weights must sum to 1");
}

int nd_total(const sf_template* t) { return t ? t->total : 0; }

}  // namespace

namespace {
std::atomic<int64_t> g_launches{0};

// Per-stage CUDA-event profiling (sf_profile_enable / sf_profile_read).
struct StageRec {
    int stage;
    cudaEvent_t a, b;
    int64_t launches;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<StageRec> g_recs;

struct StageScope {
    int stage;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    int64_t l0 = 0;
    StageScope(int st, cudaStream_t str) : stage(st), s(str) {
        if (!g_prof_on.load()) return;
        cudaEventCreate(&a);
        cudaEventRecord(a, s);
        l0 = g_launches.load();
    }
    ~StageScope() {
        if (!a) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_recs.push_back({stage, a, b, g_launches.load() - l0});
    }
};
}  // namespace

namespace sfb {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}
}  // namespace sfb

extern "C" {

const char* sf_last_error(void) { return g_last_error.c_str(); }
const char* sf_version(void) { return "scatterfield-b200 0.1 (sm_100a)"; }
int sf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ---- DensityGrid -------------------------------------------------------------------
int sf_grid_create(int nx, int ny, int nz, double vs, const double origin[3], const float* values,
                   sf_grid** out) {
    return guard([&] {
        std::unique_ptr<sf_grid, void (*)(sf_grid*)> g(new_grid(nx, ny, nz, vs, origin), free_grid);
        size_t bytes = g->count() * sizeof(float);
        if (values)
            SFB_CUDA(cudaMemcpy(g->d, values, bytes, cudaMemcpyDefault));
        else
            SFB_CUDA(cudaMemset(g->d, 0, bytes));
        *out = g.release();
    });
}

int sf_grid_info(const sf_grid* g, int dims[3], double* vs, double origin[3]) {
    return guard([&] {
        if (!g) fail(SF_ERR_INVALID_ARGUMENT, "null grid");
        dims[0] = g->nx;
        dims[1] = g->ny;
        dims[2] = g->nz;
        if (vs) *vs = g->vs;
        if (origin)
            for (int i = 0; i < 3; ++i) origin[i] = g->origin[i];
    });
}

const float* sf_grid_device_ptr(const sf_grid* g) { return g ? g->d : nullptr; }

int sf_grid_download(const sf_grid* g, float* dst, sf_stream stream) {
    return guard([&] {
        SFB_CUDA(cudaMemcpyAsync(dst, g->d, g->count() * sizeof(float), cudaMemcpyDefault, stream));
        sync(stream);
    });
}

void sf_grid_destroy(sf_grid* g) { free_grid(g); }

int sf_grid_sample_trilinear(const sf_grid* g, int64_t n, const double* pts, double* out,
                             sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        In<double> ip(pts, size_t(n) * 3, stream);
        Out<double> op(out, size_t(n), stream);
        sfb::launch_sample_trilinear(*g, n, ip.d, op.d, stream);
        op.finish();
        sync(stream);
    });
}

// ---- DensityPyramid ------------------------------------------------------------------
int sf_pyramid_build(const sf_grid* finest, sf_pyramid** out, sf_stream stream) {
    return guard([&] {
        if (!is_pow2(finest->nx) || !is_pow2(finest->ny) || !is_pow2(finest->nz))
            fail(SF_ERR_BAD_DIMS, "pyramid: dims must be powers of two");
        auto p = std::make_unique<sf_pyramid>();
        auto cleanup = [&] {
            for (sf_grid* l : p->levels) free_grid(l);
            p->levels.clear();
            if (p->block) cudaFree(p->block);
            p->block = nullptr;
        };
        try {
            // level dims (build_pyramid, src/volume_grid.cpp:91-130: halve until max dim 1)
            std::vector<int> dims{finest->nx, finest->ny, finest->nz};
            size_t total = 0;
            for (int nx = finest->nx, ny = finest->ny, nz = finest->nz;;) {
                total += size_t(nx) * ny * nz;
                if (std::max({nx, ny, nz}) <= 1) break;
                nx = std::max(1, nx / 2);
                ny = std::max(1, ny / 2);
                nz = std::max(1, nz / 2);
                dims.insert(dims.end(), {nx, ny, nz});
            }
            SFB_CUDA(cudaMalloc(&p->block, total * sizeof(float)));
            size_t off = 0;
            double vs = finest->vs;
            for (size_t l = 0; l < dims.size() / 3; ++l, vs *= 2.0) {
                auto g = std::make_unique<sf_grid>();
                g->nx = dims[3 * l];
                g->ny = dims[3 * l + 1];
                g->nz = dims[3 * l + 2];
                g->vs = vs;
                for (int i = 0; i < 3; ++i) {
                    g->origin[i] = finest->origin[i];
                    g->hi[i] = finest->origin[i] + (i == 0 ? g->nx : i == 1 ? g->ny : g->nz) * vs;
                }
                g->d = p->block + off;
                g->owned = false;
                off += g->count();
                p->levels.push_back(g.release());
                p->pads.push_back(std::make_unique<sfb::PadCache>());
            }
            SFB_CUDA(cudaMemcpyAsync(p->levels[0]->d, finest->d, finest->count() * sizeof(float),
                                     cudaMemcpyDeviceToDevice, stream));
            for (size_t l = 1; l < p->levels.size(); ++l)
                sfb::launch_pyramid_down(*p->levels[l - 1], *p->levels[l], stream);
            sync(stream);
        } catch (...) {
            cleanup();
            throw;
        }
        *out = p.release();
    });
}

int sf_pyramid_level_count(const sf_pyramid* p) { return p ? int(p->levels.size()) : 0; }

const sf_grid* sf_pyramid_level(const sf_pyramid* p, int level) {
    if (!p || level < 0 || level >= int(p->levels.size())) return nullptr;
    return p->levels[size_t(level)];
}

void sf_pyramid_destroy(sf_pyramid* p) {
    if (!p) return;
    for (sf_grid* l : p->levels) free_grid(l);
    if (p->block) cudaFree(p->block);
    delete p;
}

// ---- transmittance ---------------------------------------------------------------------
namespace {
void normalize3(const double l[3], double o[3]) {
    double len = std::sqrt(l[0] * l[0] + l[1] * l[1] + l[2] * l[2]);
    o[0] = l[0] / len;
    o[1] = l[1] / len;
    o[2] = l[2] / len;
}

sf_grid* graded_level(const sf_pyramid* p, int level, const double light[3], double lambda,
                      double step, cudaStream_t s, bool scratch = false, int zlo = 0, int zhi = -1,
                      bool fast = false) {
    if (level < 0 || level >= int(p->levels.size()))
        fail(SF_ERR_INVALID_ARGUMENT, "graded_transmittance: invalid level");
    if (!(lambda > 0.0 && lambda < 1.0))
        fail(SF_ERR_INVALID_ARGUMENT, "graded_transmittance: lambda outside (0,1)");
    if (!(step > 0.0)) fail(SF_ERR_INVALID_ARGUMENT, "optical_depth: step must be positive");
    const sf_grid* rho = p->levels[size_t(level)];
    double ld[3];
    normalize3(light, ld);
    double ts[3] = {-ld[0], -ld[1], -ld[2]};
    double coeff = std::pow(lambda, level + 1);
    sf_grid* out = scratch ? new_scratch_grid(rho->nx, rho->ny, rho->nz, rho->vs, rho->origin, s)
                           : new_grid(rho->nx, rho->ny, rho->nz, rho->vs, rho->origin);
    try {
        sfb::launch_graded(*rho, ts, coeff, step, zlo, zhi < 0 ? rho->nz : zhi, out->d, s, fast,
                           p->pads.size() > size_t(level) ? p->pads[size_t(level)].get() : nullptr);
    } catch (...) {
        free_grid(out);
        throw;
    }
    return out;
}

void combiner_weights(int L, const float* kernels, const float* scales, std::vector<float>& K, std::vector<float>& S) {
    K.assign(size_t(L) * 27, 0.0f);
    S.assign(size_t(L), 0.0f);
    if (kernels) {
        std::memcpy(K.data(), kernels, K.size() * sizeof(float));
        std::memcpy(S.data(), scales, S.size() * sizeof(float));
    } else {  // CombinerWeights::identity (src/feature_pipeline.cpp:29-35)
        for (int l = 0; l < L; ++l) {
            K[size_t(l) * 27 + 13] = 1.0f;
            S[size_t(l)] = float(1.0 / L);
        }
    }
}

// conv3 of every level (level 0 over rows [c0, c1) only) then the combine of level-0 rows
// [z0, z1) into out.
void conv_combine(const std::vector<const sf_grid*>& fields, const std::vector<float>& K,
                  const std::vector<float>& S, int c0, int c1, int z0, int z1, float* out, cudaStream_t s,
                  bool fast = false, bool sync_end = true) {
    const sf_grid& base = *fields[0];
    std::vector<sf_grid*> conv;
    try {
        for (size_t l = 0; l < fields.size(); ++l) {
            const sf_grid& f = *fields[l];
            sf_grid* c = new_scratch_grid(f.nx, f.ny, f.nz, f.vs, f.origin, s);
            conv.push_back(c);
            sfb::launch_conv3(f, &K[l * 27], l == 0 ? c0 : 0, l == 0 ? c1 : f.nz, c->d, s, fast);
        }
        std::vector<const sf_grid*> cv(conv.begin(), conv.end());
        sfb::launch_combine(cv, S, base, z0, z1, out, s, fast);
        if (sync_end) sync(s);  // scratch grids are stream-ordered pool memory: no sync needed to free them
    } catch (...) {
        for (sf_grid* c : conv) free_grid(c);
        throw;
    }
    for (sf_grid* c : conv) free_grid(c);
}

sf_tvol* combine(const std::vector<const sf_grid*>& fields, const float* kernels,
                 const float* scales, const double light[3], cudaStream_t s, bool fast = false) {
    if (fields.empty()) fail(SF_ERR_INVALID_ARGUMENT, "combine_transmittance: no fields");
    const sf_grid& base = *fields[0];
    const int L = int(fields.size());
    auto t = std::make_unique<sf_tvol>();
    normalize3(light, t->light);
    combiner_weights(L, kernels, scales, t->kernels, t->scales);
    t->values = new_grid(base.nx, base.ny, base.nz, base.vs, base.origin);
    try {
        conv_combine(fields, t->kernels, t->scales, 0, base.nz, 0, base.nz, t->values->d, s, fast);
    } catch (...) {
        free_grid(t->values);
        throw;
    }
    return t.release();
}
}  // namespace

int sf_graded_transmittance(const sf_pyramid* p, int level, const double light[3], double lambda,
                            double step, sf_grid** out, sf_stream stream) {
    return guard([&] {
        sf_grid* g = graded_level(p, level, light, lambda, step, stream);
        try {
            sync(stream);
        } catch (...) {
            free_grid(g);
            throw;
        }
        *out = g;
    });
}

int sf_conv3_replicate(const sf_grid* in, const float kernel[27], sf_grid** out,
                       sf_stream stream) {
    return guard([&] {
        sf_grid* g = new_grid(in->nx, in->ny, in->nz, in->vs, in->origin);
        try {
            sfb::launch_conv3(*in, kernel, 0, in->nz, g->d, stream);
            sync(stream);
        } catch (...) {
            free_grid(g);
            throw;
        }
        *out = g;
    });
}

int sf_combine_transmittance(const sf_grid* const* fields, int n, const float* kernels,
                             const float* scales, const double light[3], sf_tvol** out,
                             sf_stream stream) {
    return guard([&] {
        if (n <= 0) fail(SF_ERR_INVALID_ARGUMENT, "combine_transmittance: no fields");
        if (!kernels || !scales) fail(SF_ERR_SHAPE_MISMATCH, "combine_transmittance: weight/level mismatch");
        std::vector<const sf_grid*> f(fields, fields + n);
        *out = combine(f, kernels, scales, light, stream);
    });
}

namespace {
// Per device: a second stream and a fork / join event pair for the per-light build, whose coarse
// mip levels (a tail of small launches that cannot fill the GPU) run beside level 0's passes.
struct BuildSide {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
BuildSide& build_side() {
    static auto* m = new std::unordered_map<int, BuildSide>;
    int dev = 0;
    SFB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_side_mu);
    BuildSide& b = (*m)[dev];
    if (!b.side) {
        // High priority: the block scheduler then dispatches the coarse levels' blocks into the
        // slots level 0's large grids free, instead of after those grids' last blocks are issued
        // (SF_SIDE_PRIO=0: default priority)
        static const bool high = !std::getenv("SF_SIDE_PRIO") || std::atoi(std::getenv("SF_SIDE_PRIO")) != 0;
        int least = 0, greatest = 0;
        SFB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SFB_CUDA(cudaStreamCreateWithPriority(&b.side, cudaStreamNonBlocking, high ? greatest : least));
        SFB_CUDA(cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreateWithFlags(&b.join, cudaEventDisableTiming));
    }
    return b;
}

// Graded fields of every level (level 0 over rows [m0, m1), m1 < 0: all). With `fork`, levels 1..
// run on the side stream beside level 0 (bit-identical) and are joined before returning; all
// scratch is then freed on `stream`. The per-frame builds fork (relight, z-slab); the one-shot
// build_transmittance_volume, which allocates its output volume per call, does not (no gain there).
std::vector<sf_grid*> graded_fields(const sf_pyramid* p, const double light[3], double lambda, double step_scale,
                                    bool fast, cudaStream_t stream, int m0 = 0, int m1 = -1, bool fork = false) {
    static const bool side_on = !std::getenv("SF_BUILD_SERIAL");
    const int L = int(p->levels.size());
    BuildSide* bs = fork && side_on && L > 1 ? &build_side() : nullptr;
    if (bs) {
        SFB_CUDA(cudaEventRecord(bs->fork, stream));
        SFB_CUDA(cudaStreamWaitEvent(bs->side, bs->fork, 0));
    }
    std::vector<sf_grid*> fields;
    try {
        for (int i = 0; i < L; ++i) {
            const double step = step_scale * p->levels[size_t(i)]->vs;
            fields.push_back(graded_level(p, i, light, lambda, step, bs && i > 0 ? bs->side : stream, true,
                                          i == 0 ? m0 : 0, i == 0 ? m1 : -1, fast));
        }
    } catch (...) {
        for (sf_grid* g : fields) free_grid(g);
        throw;
    }
    if (bs) {
        SFB_CUDA(cudaEventRecord(bs->join, bs->side));
        SFB_CUDA(cudaStreamWaitEvent(stream, bs->join, 0));
        for (sf_grid* g : fields) g->pool_stream = stream;
    }
    return fields;
}
}  // namespace

int sf_build_transmittance_volume_ex(const sf_pyramid* p, const double light[3], const float* kernels,
                                     const float* scales, double lambda, double step_scale, int flags,
                                     sf_tvol** out, sf_stream stream) {
    return guard([&] {
        const bool fast = (flags & SF_BUILD_FP32_MARCH) != 0;
        std::vector<sf_grid*> fields;
        try {
            fields = graded_fields(p, light, lambda, step_scale, fast, stream);
            std::vector<const sf_grid*> f(fields.begin(), fields.end());
            *out = combine(f, kernels, scales, light, stream, fast);
        } catch (...) {
            for (sf_grid* g : fields) free_grid(g);
            throw;
        }
        for (sf_grid* g : fields) free_grid(g);
    });
}

int sf_build_transmittance_volume(const sf_pyramid* p, const double light[3], const float* kernels,
                                  const float* scales, double lambda, double step_scale,
                                  sf_tvol** out, sf_stream stream) {
    return sf_build_transmittance_volume_ex(p, light, kernels, scales, lambda, step_scale, 0, out, stream);
}

int sf_build_transmittance_slab(const sf_pyramid* p, const double light[3], const float* kernels,
                                const float* scales, double lambda, double step_scale, int flags, int z0, int z1,
                                float* out, sf_stream stream) {
    return guard([&] {
        const bool fast = (flags & SF_BUILD_FP32_MARCH) != 0;
        const sf_grid& g0 = *p->levels[0];
        if (z0 < 0 || z1 > g0.nz || z0 > z1) fail(SF_ERR_INVALID_ARGUMENT, "transmittance slab: z range outside the grid");
        Out<float> o(out, size_t(g0.nx) * g0.ny * size_t(z1 - z0), stream);
        if (z1 == z0) return;
        std::vector<sf_grid*> fields;
        try {
            // level 0 marched only for the rows the slab's conv and combine read (a 2-row halo:
            // the combine's trilinear at a level-0 centre may round into the next row), coarser
            // levels whole (<= 1/8 of the work, computed by every shard)
            const int c0 = std::max(z0 - 1, 0), c1 = std::min(z1 + 1, g0.nz);
            const int m0 = std::max(z0 - 2, 0), m1 = std::min(z1 + 2, g0.nz);
            fields = graded_fields(p, light, lambda, step_scale, fast, stream, m0, m1, true);
            std::vector<float> K, S;
            combiner_weights(int(fields.size()), kernels, scales, K, S);
            std::vector<const sf_grid*> f(fields.begin(), fields.end());
            conv_combine(f, K, S, c0, c1, z0, z1, o.d, stream, fast, o.host != nullptr);
        } catch (...) {
            for (sf_grid* g : fields) free_grid(g);
            throw;
        }
        for (sf_grid* g : fields) free_grid(g);
        o.finish();
        if (o.host) sync(stream);  // device output: asynchronous on `stream`
    });
}

int sf_tvol_from_values(int nx, int ny, int nz, double vs, const double origin[3],
                        const float* values, const double light[3], sf_tvol** out) {
    return guard([&] {
        auto t = std::make_unique<sf_tvol>();
        normalize3(light, t->light);
        t->values = new_grid(nx, ny, nz, vs, origin);
        cudaError_t e = cudaMemcpy(t->values->d, values, t->values->count() * sizeof(float),
                                   cudaMemcpyDefault);
        if (e != cudaSuccess) {
            free_grid(t->values);
            sfb::cuda_check(e, "tvol upload");
        }
        *out = t.release();
    });
}

const sf_grid* sf_tvol_values(const sf_tvol* t) { return t ? t->values : nullptr; }

void sf_tvol_destroy(sf_tvol* t) {
    if (!t) return;
    free_grid(t->values);
    delete t;
}

int sf_light_entry_point(const double lo[3], const double hi[3], const double p[3],
                         const double light[3], double out[3]) {
    return guard([&] {
        double ld[3];
        normalize3(light, ld);
        double ts[3] = {-ld[0], -ld[1], -ld[2]};
        double t0 = -1e300, t1 = 1e300;
        bool hit = true;
        for (int i = 0; i < 3 && hit; ++i) {
            if (ts[i] == 0.0) {
                if (p[i] < lo[i] || p[i] > hi[i]) hit = false;
                continue;
            }
            double inv = 1.0 / ts[i];
            double ta = (lo[i] - p[i]) * inv, tb = (hi[i] - p[i]) * inv;
            if (ta > tb) std::swap(ta, tb);
            t0 = std::max(t0, ta);
            t1 = std::min(t1, tb);
            if (t0 > t1) hit = false;
        }
        if (!hit) {
            for (int i = 0; i < 3; ++i) out[i] = p[i] - ld[i] * 1e-9;
            return;
        }
        double t = std::max(t1, 1e-9);
        for (int i = 0; i < 3; ++i) out[i] = p[i] + ts[i] * t;
    });
}

// ---- PhaseTable ------------------------------------------------------------------------
int sf_phase_table_build(int gr, int ar, int hr, int nodes, sf_phase_table** out, sf_stream stream) {
    return guard([&] {
        if (gr < 2 || ar < 2 || hr < 2) fail(SF_ERR_INVALID_ARGUMENT, "phase table: resolutions must be >= 2");
        if (nodes < 1) fail(SF_ERR_INVALID_ARGUMENT, "gauss_legendre: n must be positive");
        std::vector<double> x, w;
        gauss_legendre(nodes, x, w);
        auto t = std::make_unique<sf_phase_table>();
        t->g = gr;
        t->a = ar;
        t->h = hr;
        SFB_CUDA(cudaMalloc(&t->d, size_t(gr) * ar * hr * sizeof(float)));
        try {
            sfb::launch_phase_table(gr, ar, hr, x, w, t->d, stream);
            sync(stream);
        } catch (...) {
            cudaFree(t->d);
            throw;
        }
        *out = t.release();
    });
}

int sf_phase_table_from_values(int gr, int ar, int hr, const float* values, sf_phase_table** out) {
    return guard([&] {
        if (gr < 2 || ar < 2 || hr < 2) fail(SF_ERR_SHAPE_MISMATCH, "phase table: value count mismatch");
        auto t = std::make_unique<sf_phase_table>();
        t->g = gr;
        t->a = ar;
        t->h = hr;
        size_t bytes = size_t(gr) * ar * hr * sizeof(float);
        SFB_CUDA(cudaMalloc(&t->d, bytes));
        cudaError_t e = cudaMemcpy(t->d, values, bytes, cudaMemcpyDefault);
        if (e != cudaSuccess) {
            cudaFree(t->d);
            sfb::cuda_check(e, "phase table upload");
        }
        *out = t.release();
    });
}

int sf_phase_table_info(const sf_phase_table* t, int dims[3]) {
    return guard([&] {
        dims[0] = t->g;
        dims[1] = t->a;
        dims[2] = t->h;
    });
}

int sf_phase_table_download(const sf_phase_table* t, float* dst, sf_stream stream) {
    return guard([&] {
        SFB_CUDA(cudaMemcpyAsync(dst, t->d, size_t(t->g) * t->a * t->h * sizeof(float),
                                 cudaMemcpyDefault, stream));
        sync(stream);
    });
}

int sf_phase_table_lookup_hg(const sf_phase_table* t, int64_t n, const double* g,
                             const double* angle, const double* half, double* out,
                             sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        In<double> a(g, size_t(n), stream), b(angle, size_t(n), stream), c(half, size_t(n), stream);
        Out<double> o(out, size_t(n), stream);
        sfb::launch_lookup_hg(*t, n, a.d, b.d, c.d, o.d, stream);
        o.finish();
        sync(stream);
    });
}

void sf_phase_table_destroy(sf_phase_table* t) {
    if (!t) return;
    cudaFree(t->d);
    cudaFree(t->d_quad);
    delete t;
}

// ---- SamplingTemplate ------------------------------------------------------------------
int sf_template_create(int kind, int n_layers, const int* counts, const double* points,
                       const double* caps, double gen_distance, double cone_half_angle,
                       sf_template** out) {
    return guard([&] {
        if (kind != SF_TEMPLATE_DIFFUSE && kind != SF_TEMPLATE_HIGHLIGHT)
            fail(SF_ERR_BAD_VALUE, "template: unknown kind");
        if (n_layers < 1) fail(SF_ERR_INVALID_ARGUMENT, "template: no layers");
        if (kind == SF_TEMPLATE_HIGHLIGHT && !(gen_distance > 0.0))
            fail(SF_ERR_INVALID_ARGUMENT, "highlight template: zero entry distance");
        auto t = std::make_unique<sf_template>();
        t->kind = kind;
        t->n_layers = n_layers;
        t->counts.assign(counts, counts + n_layers);
        for (int c : t->counts)
            if (c < 0) fail(SF_ERR_INVALID_ARGUMENT, "template: negative layer count");
        for (int c : t->counts) t->total += c;
        t->points.assign(points, points + size_t(t->total) * 3);
        t->caps.assign(caps, caps + n_layers);
        t->gen_distance = gen_distance;
        t->cone_half_angle = cone_half_angle;
        std::vector<double> pc;
        for (int l = 0; l < n_layers; ++l) pc.insert(pc.end(), size_t(t->counts[size_t(l)]), caps[l]);
        size_t np = std::max<size_t>(1, size_t(t->total));
        SFB_CUDA(cudaMalloc(&t->d_points, np * 3 * sizeof(double)));
        SFB_CUDA(cudaMalloc(&t->d_caps, np * sizeof(double)));
        SFB_CUDA(cudaMalloc(&t->d_pts4, np * sizeof(float4)));
        if (t->total) {
            std::vector<float4> p4(size_t(t->total));
            for (int i = 0; i < t->total; ++i)
                p4[size_t(i)] = make_float4(float(t->points[3 * size_t(i)]), float(t->points[3 * size_t(i) + 1]),
                                            float(t->points[3 * size_t(i) + 2]), float(pc[size_t(i)]));
            SFB_CUDA(cudaMemcpy(t->d_pts4, p4.data(), p4.size() * sizeof(float4), cudaMemcpyHostToDevice));
            SFB_CUDA(cudaMemcpy(t->d_points, t->points.data(), t->points.size() * sizeof(double),
                                cudaMemcpyHostToDevice));
            SFB_CUDA(cudaMemcpy(t->d_caps, pc.data(), pc.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        *out = t.release();
    });
}

int sf_template_total_points(const sf_template* t) { return t ? t->total : 0; }

int sf_place_template(const sf_template* t, int64_t n, const double* p, const double* omega,
                      const double* entry, double ts, double* out_pts, double* out_caps,
                      sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        In<double> ip(p, size_t(n) * 3, stream), iw(omega, size_t(n) * 3, stream),
            ie(entry, size_t(n) * 3, stream);
        Out<double> op(out_pts, size_t(n) * t->total * 3, stream), oc(out_caps, size_t(n) * t->total, stream);
        Scratch<int> err(1, stream);
        SFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
        sfb::launch_place_template(*t, n, ip.d, iw.d, ie.d, ts, op.d, oc.d, err.p, stream);
        int herr = 0;
        SFB_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        op.finish();
        oc.finish();
        sync(stream);
        if (herr) fail(SF_ERR_INVALID_ARGUMENT, "place_template: entry coincides with p");
    });
}

void sf_template_destroy(sf_template* t) {
    if (!t) return;
    cudaFree(t->d_points);
    cudaFree(t->d_caps);
    cudaFree(t->d_pts4);
    delete t;
}

// ---- sample_features --------------------------------------------------------------------
int sf_sample_features(const sf_grid* density, const sf_tvol* tvol, const sf_template* tmpl,
                       const sf_phase_model* model, const sf_phase_table* table, double ts,
                       int64_t n, const double* queries, float* out, sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        validate_phase_model(*model);
        const sf_grid& tv = *tvol->values;
        if (tv.nx != density->nx || tv.ny != density->ny || tv.nz != density->nz)
            fail(SF_ERR_SHAPE_MISMATCH, "sample_features: transmittance volume geometry differs");
        In<double> iq(queries, size_t(n) * 9, stream);
        Out<float> of(out, size_t(n) * 3 * tmpl->total, stream);
        Scratch<int> err(1, stream);
        SFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
        sfb::SceneDev sc = sfb::scene_dev(*density, tv, nullptr, *model, *table, ts);
        sfb::launch_sample_features(sc, sfb::template_dev(*tmpl), n, iq.d, nullptr, of.d, 3 * tmpl->total, 0,
                                    err.p, stream);
        int herr = 0;
        SFB_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        of.finish();
        sync(stream);
        if (herr) fail(SF_ERR_INVALID_ARGUMENT, "place_template: entry coincides with p");
    });
}

// ---- Backbone ------------------------------------------------------------------------------
int sf_backbone_create(const sf_backbone_config* config, const float* params, sf_backbone** out) {
    return guard([&] {
        validate_backbone_config(*config);
        auto b = std::make_unique<sf_backbone>();
        b->cfg = *config;
        b->layout = make_layout(*config);
        size_t bytes = size_t(b->layout.total) * sizeof(float);
        SFB_CUDA(cudaMalloc(&b->d_params, bytes));
        cudaError_t e;
        if (params) {
            e = cudaMemcpy(b->d_params, params, bytes, cudaMemcpyDefault);
        } else {
            std::vector<float> init = he_init(*config);
            e = cudaMemcpy(b->d_params, init.data(), bytes, cudaMemcpyHostToDevice);
        }
        if (e != cudaSuccess) {
            cudaFree(b->d_params);
            sfb::cuda_check(e, "backbone upload");
        }
        *out = b.release();
    });
}

int64_t sf_backbone_param_count(const sf_backbone* b) { return b ? b->layout.total : 0; }

int sf_backbone_download_params(const sf_backbone* b, float* dst, sf_stream stream) {
    return guard([&] {
        SFB_CUDA(cudaMemcpyAsync(dst, b->d_params, size_t(b->layout.total) * sizeof(float),
                                 cudaMemcpyDefault, stream));
        sync(stream);
    });
}

void sf_backbone_destroy(sf_backbone* b);

namespace {
std::mutex g_tc_mu;

void check_precision(const sf_backbone& b, int precision, cudaStream_t s) {
    if (precision == SF_PRECISION_FP32) return;
    if (precision != SF_PRECISION_BF16 && precision != SF_PRECISION_FP16)
        fail(SF_ERR_INVALID_ARGUMENT, "unknown precision");
    if (!sfb::tc_supported(b.cfg))
        fail(SF_ERR_INVALID_ARGUMENT,
             "bf16 tensor-core backbone needs widths 32/64/64 and layers of at most 62 points");
    std::lock_guard<std::mutex> lk(g_tc_mu);
    sfb::tc_prepare(const_cast<sf_backbone&>(b), s, precision == SF_PRECISION_FP16);
}


// Event recorded on `from` and waited on by `to`; `ev` a reusable event (a wait captures the
// event's state when it is enqueued, so re-recording it later is safe).
void stream_wait(cudaStream_t to, cudaStream_t from, cudaEvent_t ev = nullptr) {
    cudaEvent_t e = ev;
    if (!e) SFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SFB_CUDA(cudaEventRecord(e, from));
    SFB_CUDA(cudaStreamWaitEvent(to, e, 0));
    if (!ev) SFB_CUDA(cudaEventDestroy(e));  // released once the wait completes
}

// Per-device workspace of the bf16 query path: one block carved into the call's buffers and
// kept between calls (instead of ~10 stream-ordered allocations per call). Calls on one device
// are enqueued under a mutex; a call on a different stream than the previous user first waits
// for the previous call's completion event, so the block is never used by two calls at once.
// Growing synchronises the device.
struct Workspace {
    uint8_t* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev[8] = {};
    int next_ev = 0;
    cudaEvent_t done = nullptr;        // recorded at the end of the last call's work
    cudaStream_t last = nullptr;
    bool used = false;
    cudaStream_t copy = nullptr;       // this device's copy stream for the host-I/O overlap
};
std::mutex g_ws_mu;
std::unordered_map<int, Workspace>& workspaces() {
    static auto* m = new std::unordered_map<int, Workspace>;
    return *m;
}

extern "C++" {
struct Carve {
    uint8_t* base;
    size_t off = 0;
    template <typename T>
    T* take(size_t count) {
        T* r = count && base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += (count * sizeof(T) + 255) & ~size_t(255);
        return r;
    }
};
}

// bf16 path over one chunk: fused sample+sort (or sort of given features) -> tcgen05 backbone.
void run_bf16_chunk(const sf_backbone& b, const sfb::SortLayout& L, const sfb::SceneDev* sc,
                    const sfb::TemplateDev* dt, const sfb::TemplateDev* ht, const float* planes, int n_planes,
                    const float4* pre, int64_t m, const void* recs, const float* feats, const double* cfg8,
                    uint8_t* ops, float* mms, int* err, float* y, double* F, cudaStream_t s, bool f16) {
    {
        StageScope st(SF_STAGE_SAMPLE_SORT, s);
        sfb::launch_sample_sort(sc, dt, ht, planes, n_planes, pre, L, m, recs, feats, ops, mms, err, s, false, 0, 0,
                                f16);
    }
    {
        StageScope st(SF_STAGE_BACKBONE, s);
        sfb::launch_backbone_tc(b, m, ops, mms, cfg8, y, F, s, nullptr, f16);
    }
}
}  // namespace

int sf_predict(const sf_backbone* b, int64_t n, const float* features, const double* config8,
               int precision, float* y_out, double* F_out, sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        const sf_backbone_config& c = b->cfg;
        int64_t feat = 0;
        for (int i = 0; i < c.n_diffuse_layers; ++i) feat += 3 * c.diffuse_counts[i];
        for (int i = 0; i < c.n_highlight_layers; ++i) feat += 3 * c.highlight_counts[i];
        if (!is_device_ptr(config8))
            for (int64_t i = 0; i < n; ++i) validate_albedo(config8 + 8 * i + 4);
        check_precision(*b, precision, stream);
        In<float> f(features, size_t(n) * feat, stream);
        In<double> cf(config8, size_t(n) * 8, stream);
        Out<float> oy(y_out, size_t(n) * 3, stream);
        Out<double> oF(F_out, size_t(n) * 3, stream);
        if (precision == SF_PRECISION_FP32) {
            Scratch<float> slices(size_t(n) * sfb::slices_per_query(c), stream);
            {
                StageScope st(SF_STAGE_SLICE, stream);
                sfb::launch_slice(c, n, f.d, slices.p, stream);
            }
            {
                StageScope st(SF_STAGE_BACKBONE, stream);
                sfb::launch_backbone_fp32(*b, n, slices.p, cf.d, oy.d, oF.d, stream);
            }
        } else {
            const sfb::SortLayout L = sfb::sort_layout(c);
            const int64_t tiles = (n + sfb::kUmmaM - 1) / sfb::kUmmaM;
            Scratch<uint8_t> ops(size_t(tiles) * L.tile_bytes, stream);
            Scratch<float> mms(size_t(L.n_layers) * tiles * sfb::kUmmaM * 8, stream);
            run_bf16_chunk(*b, L, nullptr, nullptr, nullptr, nullptr, 0, nullptr, n, nullptr, f.d, cf.d, ops.p,
                           mms.p, nullptr, oy.d, oF.d, stream, precision == SF_PRECISION_FP16);
        }
        oy.finish();
        oF.finish();
        sync(stream);
    });
}

// ---- fused query -----------------------------------------------------------------------------
int sf_scene_create(const sf_grid* density, const sf_tvol* tvol, const sf_template* dt,
                    const sf_template* ht, const sf_phase_model* model, const sf_phase_table* table,
                    double ts, sf_scene** out) {
    return guard([&] {
        validate_phase_model(*model);
        if (dt->kind != SF_TEMPLATE_DIFFUSE || ht->kind != SF_TEMPLATE_HIGHLIGHT)
            fail(SF_ERR_INVALID_ARGUMENT, "scene: need a diffuse and a highlight template");
        const sf_grid& tv = *tvol->values;
        if (tv.nx != density->nx || tv.ny != density->ny || tv.nz != density->nz)
            fail(SF_ERR_SHAPE_MISMATCH, "scene: transmittance volume geometry differs");
        // the production sampler addresses 32-byte xy-quad records with unsigned 32-bit indices
        if (sfb::xpair_records(density->nx, density->ny, density->nz) / 2 >= (size_t(1) << 32))
            fail(SF_ERR_BAD_DIMS, "scene: volume too large for the query records (2^32 records)");
        auto s = std::make_unique<sf_scene>();
        s->density = density;
        s->tvol = tvol;
        s->dt = dt;
        s->ht = ht;
        s->model = *model;
        s->table = table;
        s->template_scale = ts;
        s->n_planes = model->kind == SF_PHASE_ISOTROPIC ? 1 : model->n_lobes;
        try {
            SFB_CUDA(cudaMalloc(&s->d_dt, density->count() * sizeof(float2)));
            SFB_CUDA(cudaMalloc(&s->d_dt4, sfb::xpair_records(density->nx, density->ny, density->nz) *
                                                sizeof(float4)));
            SFB_CUDA(cudaMalloc(&s->d_planes, size_t(s->n_planes) * table->a * (table->h + 1) * sizeof(float2)));
            SFB_CUDA(cudaMalloc(&s->d_pre, std::max<size_t>(1, size_t(dt->total)) * 2 * sizeof(float4)));
            sfb::launch_interleave(density->d, tv.d, s->d_dt, density->count(), nullptr);
            sfb::launch_xpair(density->d, tv.d, density->nx, density->ny, density->nz, s->d_dt4, nullptr);
            sfb::launch_blend_planes(*table, *model, s->d_planes, nullptr);
            SFB_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            cudaFree(s->d_dt);
            cudaFree(s->d_dt4);
            cudaFree(s->d_planes);
            cudaFree(s->d_pre);
            throw;
        }
        *out = s.release();
    });
}

// the scene's own transmittance volume (one allocation on first use, kept)
static sf_tvol* scene_own_tvol(sf_scene* s) {
    if (!s->own_tvol) {
        const sf_grid& d = *s->density;
        auto t = std::make_unique<sf_tvol>();
        t->values = new_grid(d.nx, d.ny, d.nz, d.vs, d.origin);
        s->own_tvol = t.release();
    }
    return s->own_tvol;
}


int sf_scene_relight(sf_scene* s, const sf_pyramid* p, const double light[3], const float* kernels,
                     const float* scales, double lambda, double step_scale, int flags, sf_stream stream) {
    return guard([&] {
        if (!s || !p || p->levels.empty()) fail(SF_ERR_INVALID_ARGUMENT, "scene_relight: null scene or pyramid");
        const sf_grid& g0 = *p->levels[0];
        const sf_grid& d = *s->density;
        if (g0.nx != d.nx || g0.ny != d.ny || g0.nz != d.nz || g0.vs != d.vs || g0.origin[0] != d.origin[0] ||
            g0.origin[1] != d.origin[1] || g0.origin[2] != d.origin[2])
            fail(SF_ERR_SHAPE_MISMATCH, "scene_relight: pyramid geometry differs from the scene's density");
        const bool fast = (flags & SF_BUILD_FP32_MARCH) != 0;
        const int L = int(p->levels.size());
        sf_tvol* t = scene_own_tvol(s);  // first relight: the scene's own volume (one allocation, kept)
        normalize3(light, t->light);
        combiner_weights(L, kernels, scales, t->kernels, t->scales);
        std::vector<sf_grid*> fields, conv;
        try {
            // levels 1.. (graded field and 3D-CNN convolution) on the side stream while level 0 runs
            // on `stream` (the same kernels and operands: bit-identical); the combine waits for both.
            // Side-stream scratch is freed on `stream` after the join.
            static const bool side_on = !std::getenv("SF_BUILD_SERIAL");
            BuildSide* bs = side_on && L > 1 ? &build_side() : nullptr;
            if (bs) {
                SFB_CUDA(cudaEventRecord(bs->fork, stream));
                SFB_CUDA(cudaStreamWaitEvent(bs->side, bs->fork, 0));
            }
            auto level_stream = [&](int i) { return bs && i > 0 ? bs->side : stream; };
            {
                StageScope st(SF_STAGE_MARCH, stream);
                for (int i = 0; i < L; ++i) {
                    const double step = step_scale * p->levels[size_t(i)]->vs;
                    fields.push_back(graded_level(p, i, light, lambda, step, level_stream(i), true, 0, -1, fast));
                }
            }
            StageScope st(SF_STAGE_COMBINER, stream);
            for (int i = L - 1; i >= 0; --i) {  // the side stream's convolutions are queued first
                const sf_grid& f = *fields[size_t(i)];
                sf_grid* c = new_scratch_grid(f.nx, f.ny, f.nz, f.vs, f.origin, level_stream(i));
                conv.insert(conv.begin(), c);
                sfb::launch_conv3(f, &t->kernels[size_t(i) * 27], 0, f.nz, c->d, level_stream(i), fast);
            }
            if (bs) {
                SFB_CUDA(cudaEventRecord(bs->join, bs->side));
                SFB_CUDA(cudaStreamWaitEvent(stream, bs->join, 0));
                for (sf_grid* g : fields) g->pool_stream = stream;
                for (sf_grid* g : conv) g->pool_stream = stream;
            }
            std::vector<const sf_grid*> cv(conv.begin(), conv.end());
            sfb::launch_combine(cv, t->scales, *fields[0], 0, d.nz, t->values->d, stream, fast);
        } catch (...) {
            for (sf_grid* g : fields) free_grid(g);
            for (sf_grid* g : conv) free_grid(g);
            throw;
        }
        for (sf_grid* g : conv) free_grid(g);
        for (sf_grid* g : fields) free_grid(g);
        s->tvol = t;
        StageScope st(SF_STAGE_RECORDS, stream);
        sfb::launch_xpair(d.d, t->values->d, d.nx, d.ny, d.nz, s->d_dt4, stream);
        s->dt_stale = true;
    });
}

int sf_scene_tvol_storage(sf_scene* s, float** out) {
    return guard([&] {
        if (!s || !out) fail(SF_ERR_INVALID_ARGUMENT, "scene_tvol_storage: null argument");
        *out = scene_own_tvol(s)->values->d;
    });
}

int sf_scene_commit_tvol(sf_scene* s, const double light[3], sf_stream stream) {
    return guard([&] {
        if (!s) fail(SF_ERR_INVALID_ARGUMENT, "scene_commit_tvol: null scene");
        sf_tvol* t = scene_own_tvol(s);
        normalize3(light, t->light);
        s->tvol = t;
        const sf_grid& d = *s->density;
        StageScope st(SF_STAGE_RECORDS, stream);
        sfb::launch_xpair(d.d, t->values->d, d.nx, d.ny, d.nz, s->d_dt4, stream);
        s->dt_stale = true;
    });
}

void sf_scene_destroy(sf_scene* s) {
    if (!s) return;
    sf_tvol_destroy(s->own_tvol);
    cudaFree(s->d_dt);
    cudaFree(s->d_dt4);
    cudaFree(s->d_planes);
    cudaFree(s->d_pre);
    delete s;
}

namespace {
// The interleaved {density, transmittance} volume of the exact (FP32) path after a relight.
void refresh_dt(const sf_scene* s, cudaStream_t stream) {
    if (!s->dt_stale) return;
    sf_scene* m = const_cast<sf_scene*>(s);
    sfb::launch_interleave(s->density->d, s->tvol->values->d, m->d_dt, s->density->count(), stream);
    m->dt_stale = false;
}

// sf_query / sf_query_media: medium is the scene-wide medium, media (nullable) per-query
// {g, albedo rgb} rows that override it (single-lobe HG per query).
void query_impl(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium, const double* media_in,
                int64_t n, const double* queries, int precision, double* F_out, float* y_out, cudaStream_t stream,
                float* dbg_pools = nullptr) {
        if (n <= 0) return;
        sf_medium_params uniform{};
        if (media_in) {
            if (!is_device_ptr(media_in))
                for (int64_t i = 0; i < n; ++i) {
                    validate_albedo(media_in + 4 * i + 1);
                    if (!(media_in[4 * i] > -1.0 && media_in[4 * i] < 1.0))
                        fail(SF_ERR_INVALID_ARGUMENT, "PhaseModel::hg: g outside (-1, 1)");
                }
            medium = &uniform;
        } else {
            validate_albedo(medium->albedo);
        }
        In<double> imedia(media_in, media_in ? size_t(n) * 4 : 0, stream);
        const double* media = media_in ? imedia.d : nullptr;
        const sf_backbone_config& c = b->cfg;
        int nd = 0, nh = 0;
        for (int i = 0; i < c.n_diffuse_layers; ++i) nd += c.diffuse_counts[i];
        for (int i = 0; i < c.n_highlight_layers; ++i) nh += c.highlight_counts[i];
        if (nd != s->dt->total || nh != s->ht->total)
            fail(SF_ERR_SHAPE_MISMATCH, "feature block does not match template counts");
        check_precision(*b, precision, stream);
        if (precision == SF_PRECISION_BF16 || precision == SF_PRECISION_FP16) {
            const bool f16 = precision == SF_PRECISION_FP16;
            // production path: query_prep -> fused sample+sort -> tcgen05 backbone per chunk of
            // up to 4096 tiles, all on the caller's stream. With host query rows the chunk's rows
            // arrive on a copy stream in two windows: the first (~1/5 of the rows, a whole number
            // of the sampling grid's rounds) is prepared and sampled while the rest lands; both
            // windows fill one operand layout, so the backbone still runs once per chunk (no
            // extra wave tail).
            const sfb::SortLayout L = sfb::sort_layout(c);
            const int64_t n_tiles = (n + sfb::kUmmaM - 1) / sfb::kUmmaM;
            const bool h_in = !is_device_ptr(queries);
            // pinned host F (not on the Morton path, whose rows are scattered): written in place
            double* z_F = nullptr;
            const bool hF0 = F_out && !is_device_ptr(F_out);
            bool zero_copy = false;
            static const bool overlap_on = !std::getenv("SF_NO_HOST_OVERLAP");
            // Volumes beyond L2 (x-pair records of a 256^3 grid are 268 MB): process the queries
            // grouped by the Morton order of their 64^3 cell (a counting sort, launch_cell_order) so
            // concurrently sampled queries share the volume's cache lines; results are written back
            // to the caller's rows.
            static const int morton_env = std::getenv("SF_MORTON") ? std::atoi(std::getenv("SF_MORTON")) : -1;
            const size_t vol_bytes = sfb::xpair_records(s->density->nx, s->density->ny, s->density->nz) *
                                     sizeof(float4);
            const bool reorder = !dbg_pools && (morton_env >= 0 ? morton_env > 0 && n > 1
                                                                : (vol_bytes > (size_t(96) << 20) && n >= 4096));
            if (hF0 && !reorder && (reinterpret_cast<uintptr_t>(F_out) & 15) == 0) {
                z_F = static_cast<double*>(mapped_alias(F_out));
                zero_copy = z_F != nullptr;
            }
            const bool h_out = (hF0 && !zero_copy) || (y_out && !is_device_ptr(y_out));
            const bool overlap = overlap_on && !reorder && h_in && n_tiles >= 64;
            // SF_CHUNK_TILES (A/B): chunks small enough that the sampler's operand blocks are still
            // in L2 when the backbone reads them (plain stores instead of evict-first)
            static const int64_t chunk_env = std::getenv("SF_CHUNK_TILES") ? std::atoll(std::getenv("SF_CHUNK_TILES")) : 0;
            // Queries go through the sampler and the backbone in chunks of up to 2^14 tiles (2,097,152
            // queries; ~0.28 MB of operands per tile, so <= ~4.7 GB of workspace operands): one chunk
            // for a C5 frame, two for C4 -- every backbone launch ends in a tail of partly idle SMs,
            // so fewer, larger chunks are faster (C5 query 5.86 -> 5.79 ms, C4 22.8 -> 22.4 ms against
            // 2^12-tile chunks, bit-identical). SF_CHUNK_CAP overrides the cap (A/B, small-memory runs).
            // (read per call, not cached: tests switch it within one process)
            const char* cap_s = std::getenv("SF_CHUNK_CAP");
            const int64_t cap_env = cap_s ? std::atoll(cap_s) : 0;
            const int64_t chunk_tiles =
                std::min<int64_t>(n_tiles, chunk_env > 0 ? chunk_env : (cap_env > 0 ? cap_env : 1 << 14));
            const bool l2_keep = chunk_env > 0;
            const int64_t chunk = chunk_tiles * sfb::kUmmaM;
            // sampling windows {first row, rows, chunk's first row}
            struct Win {
                int64_t r0, m, c0;
            };
            std::vector<Win> wins;
            {
                const int64_t rq = sfb::sample_sort_round_queries();
                const int64_t unit = rq / std::gcd(rq, int64_t(sfb::kUmmaM));  // tiles per whole number of rounds
                static const double first = std::getenv("SF_FIRST_WINDOW") ? std::atof(std::getenv("SF_FIRST_WINDOW"))
                                                                           : 0.2;
                for (int64_t c0 = 0; c0 < n; c0 += chunk) {
                    const int64_t m = std::min(chunk, n - c0), tiles = (m + sfb::kUmmaM - 1) / sfb::kUmmaM;
                    int64_t w0 = overlap ? std::max<int64_t>(1, std::llround(first * double(tiles) / double(unit))) * unit
                                         : 0;
                    if (w0 >= tiles || first <= 0.0) w0 = 0;
                    if (w0) {
                        wins.push_back({c0, w0 * sfb::kUmmaM, c0});
                        wins.push_back({c0 + w0 * sfb::kUmmaM, m - w0 * sfb::kUmmaM, c0});
                    } else {
                        wins.push_back({c0, m, c0});
                    }
                }
            }
            // the call's device buffers, carved from the stream's workspace
            const bool hF = hF0 && !zero_copy, hy = y_out && !is_device_ptr(y_out);
            auto carve_all = [&](uint8_t* base, Carve& cv) {
                cv = Carve{base};
                struct {
                    uint8_t *ops, *recs;
                    float* mms;
                    double *cfg8, *rows, *F;
                    int *err, *perm;
                    float* y;
                    uint32_t* keys;
                    int* idx;
                } b{};
                b.ops = cv.take<uint8_t>(size_t(chunk_tiles) * L.tile_bytes);
                b.mms = cv.take<float>(size_t(L.n_layers) * chunk * 8);
                b.cfg8 = cv.take<double>(size_t(chunk) * 8);
                b.recs = cv.take<uint8_t>(size_t(chunk) * sfb::query_rec_bytes());
                b.err = cv.take<int>(1);
                b.rows = cv.take<double>(h_in ? size_t(n) * 9 : 0);
                b.F = cv.take<double>(hF ? size_t(n) * 3 : 0);
                b.y = cv.take<float>(hy ? size_t(n) * 3 : 0);
                b.perm = cv.take<int>(reorder ? size_t(n) : 0);
                b.keys = cv.take<uint32_t>(reorder ? size_t(n) : 0);  // cell keys (launch_cell_order)
                b.idx = nullptr;
                return b;
            };
            Carve probe{nullptr};
            carve_all(nullptr, probe);
            const size_t sort_tmp = reorder ? size_t(sfb::kOrderCells + 1024) * sizeof(int) : 0;  // cell counts
            const size_t need = probe.off + sort_tmp + 256;
            std::unique_lock<std::mutex> wlk(g_ws_mu);
            int dev = 0;
            SFB_CUDA(cudaGetDevice(&dev));
            Workspace& ws = workspaces()[dev];
            if (!ws.done) {
                SFB_CUDA(cudaEventCreateWithFlags(&ws.done, cudaEventDisableTiming));
                for (auto& e : ws.ev) SFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            if (ws.cap < need) {
                if (ws.p) {
                    SFB_CUDA(cudaDeviceSynchronize());
                    cudaFree(ws.p);
                    ws.p = nullptr;
                    ws.cap = 0;
                }
                SFB_CUDA(cudaMalloc(&ws.p, need));
                ws.cap = need;
            } else if (ws.used && ws.last != stream) {
                SFB_CUDA(cudaStreamWaitEvent(stream, ws.done, 0));  // the previous call, other stream
            }
            const bool had_prev = ws.used;
            ws.used = true;
            ws.last = stream;
            struct DoneGuard {  // on every exit path: later calls order after this one
                Workspace& w;
                cudaStream_t s;
                ~DoneGuard() { cudaEventRecord(w.done, s); }
            } done_guard{ws, stream};
            Carve cv{nullptr};
            auto bufs = carve_all(ws.p, cv);
            uint8_t* sort_tmp_p = ws.p + cv.off;
            auto next_event = [&]() {
                cudaEvent_t e = ws.ev[ws.next_ev];
                ws.next_ev = (ws.next_ev + 1) % 8;
                return e;
            };
            struct {
                uint8_t* p;
            } ops{bufs.ops}, recs{bufs.recs};
            struct {
                float* p;
            } mms{bufs.mms}, y_buf{bufs.y};
            struct {
                double* p;
            } cfg8{bufs.cfg8}, rows_buf{bufs.rows}, F_buf{bufs.F};
            struct {
                int* p;
            } err{bufs.err}, perm{bufs.perm};
            SFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
            const double* rows = h_in ? rows_buf.p : queries;
            double* Fd = F_out ? (zero_copy ? z_F : (F_buf.p ? F_buf.p : F_out)) : nullptr;
            float* yd = y_out ? (y_buf.p ? y_buf.p : y_out) : nullptr;
            sfb::SceneDev sc = sfb::scene_dev(*s->density, *s->tvol->values, s->d_dt, s->model, *s->table,
                                              s->template_scale);
            sc.dt4 = s->d_dt4;
            if (media) sc.phase.quad = sfb::phase_quad(*s->table, stream);
            sfb::TemplateDev dt = sfb::template_dev(*s->dt), ht = sfb::template_dev(*s->ht);
            cudaStream_t cs = stream;
            if (h_in || h_out) {  // the device's copy stream (calls on one device hold g_ws_mu)
                if (!ws.copy) SFB_CUDA(cudaStreamCreateWithFlags(&ws.copy, cudaStreamNonBlocking));
                cs = ws.copy;
                // the rows may land as soon as the previous call is done with the workspace, so the
                // copy overlaps whatever the caller queued on `stream` since (e.g. a relight)
                if (had_prev) SFB_CUDA(cudaStreamWaitEvent(cs, ws.done, 0));
            }
            // every chunk's rows are queued at once, each followed by its own event
            std::vector<cudaEvent_t> rows_ready;
            struct EvGuard {
                std::vector<cudaEvent_t>& v;
                ~EvGuard() {
                    for (cudaEvent_t e : v) cudaEventDestroy(e);
                }
            } ev_guard{rows_ready};
            if (h_in)
                for (const Win& w : wins) {
                    SFB_CUDA(cudaMemcpyAsync(rows_buf.p + 9 * w.r0, queries + 9 * w.r0, size_t(w.m) * 9 * sizeof(double),
                                             cudaMemcpyHostToDevice, cs));
                    cudaEvent_t e;
                    SFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    rows_ready.push_back(e);
                    SFB_CUDA(cudaEventRecord(e, cs));
                }
            if (reorder) {
                for (cudaEvent_t e : rows_ready) SFB_CUDA(cudaStreamWaitEvent(stream, e, 0));  // every row
                sfb::launch_cell_order(s->density->dev(), n, rows, bufs.keys, reinterpret_cast<int*>(sort_tmp_p), perm.p,
                                       stream);
            }
            size_t wi = 0;
            for (int64_t c0 = 0; c0 < n; c0 += chunk) {
                const int64_t m = std::min(chunk, n - c0), layout_tiles = (m + sfb::kUmmaM - 1) / sfb::kUmmaM;
                for (; wi < wins.size() && wins[wi].c0 == c0; ++wi) {
                    const Win& w = wins[wi];
                    if (h_in && !reorder) SFB_CUDA(cudaStreamWaitEvent(stream, rows_ready[wi], 0));  // window's rows
                    {  // the first window's launch also makes the diffuse constants (light of row 0)
                        StageScope st(SF_STAGE_CONFIG, stream);
                        const sfb::TemplateDev* dtp = wi == 0 ? &dt : nullptr;
                        if (reorder)
                            sfb::launch_query_prep(sc, ht, *medium, w.m, rows, media, cfg8.p + 8 * (w.r0 - c0), recs.p,
                                                   stream, perm.p + w.r0, rows, dtp, s->d_planes, s->n_planes, s->d_pre);
                        else
                            sfb::launch_query_prep(sc, ht, *medium, w.m, rows + 9 * w.r0, media ? media + 4 * w.r0 : nullptr,
                                                   cfg8.p + 8 * (w.r0 - c0), recs.p, stream, nullptr, rows, dtp,
                                                   s->d_planes, s->n_planes, s->d_pre);
                    }
                    {
                        StageScope st(SF_STAGE_SAMPLE_SORT, stream);
                        sfb::launch_sample_sort(&sc, &dt, &ht, s->d_planes, s->n_planes, s->d_pre, L, w.m, recs.p,
                                                nullptr, ops.p, mms.p, err.p, stream, media != nullptr,
                                                (w.r0 - c0) / sfb::kUmmaM, layout_tiles, f16, l2_keep);
                    }
                }
                {
                    StageScope st(SF_STAGE_BACKBONE, stream);
                    if (reorder)
                        sfb::launch_backbone_tc(*b, m, ops.p, mms.p, cfg8.p, yd, Fd, stream, perm.p + c0, f16);
                    else
                        sfb::launch_backbone_tc(*b, m, ops.p, mms.p, cfg8.p, yd ? yd + 3 * c0 : nullptr,
                                                Fd ? Fd + 3 * c0 : nullptr, stream, nullptr, f16);
                }
                if (dbg_pools)  // the chunk's fp32 pools, [layer][row][8] -> [layer][n][8]
                    SFB_CUDA(cudaMemcpy2DAsync(dbg_pools + 8 * c0, size_t(n) * 8 * sizeof(float), mms.p,
                                               size_t(chunk) * 8 * sizeof(float), size_t(m) * 8 * sizeof(float),
                                               size_t(L.n_layers), cudaMemcpyDeviceToDevice, stream));
                if (h_out && !reorder) {  // results home: on the copy stream while a next chunk computes
                    const bool last = c0 + chunk >= n;
                    cudaStream_t ds = last ? stream : cs;
                    if (!last) stream_wait(cs, stream, next_event());
                    if (F_buf.p)
                        SFB_CUDA(cudaMemcpyAsync(F_out + 3 * c0, F_buf.p + 3 * c0, size_t(m) * 3 * sizeof(double),
                                                 cudaMemcpyDeviceToHost, ds));
                    if (y_buf.p)
                        SFB_CUDA(cudaMemcpyAsync(y_out + 3 * c0, y_buf.p + 3 * c0, size_t(m) * 3 * sizeof(float),
                                                 cudaMemcpyDeviceToHost, ds));
                }
            }
            if (h_out && reorder) {  // scattered rows: one copy home after the last chunk
                if (F_buf.p)
                    SFB_CUDA(cudaMemcpyAsync(F_out, F_buf.p, size_t(n) * 3 * sizeof(double), cudaMemcpyDeviceToHost,
                                             stream));
                if (y_buf.p)
                    SFB_CUDA(cudaMemcpyAsync(y_out, y_buf.p, size_t(n) * 3 * sizeof(float), cudaMemcpyDeviceToHost,
                                             stream));
            }
            if (cs != stream) stream_wait(stream, cs, next_event());  // the caller sees the copies
            if (!h_out && !h_in && !zero_copy) return;  // device in/out: asynchronous (see below)
            int herr = 0;
            SFB_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
            sync(stream);
            if (herr) fail(SF_ERR_INVALID_ARGUMENT, "place_template: entry coincides with p");
            return;
        }
        refresh_dt(s, stream);
        In<double> iq(queries, size_t(n) * 9, stream);
        Out<double> oF(F_out, size_t(n) * 3, stream);
        Out<float> oy(y_out, size_t(n) * 3, stream);
        const int64_t chunk = std::min<int64_t>(n, 1 << 17);
        const int64_t feat = 3 * int64_t(nd + nh);
        Scratch<float> feats(size_t(chunk) * feat, stream);
        Scratch<float> slices(size_t(chunk) * sfb::slices_per_query(c), stream);
        Scratch<double> cfg8(size_t(chunk) * 8, stream);
        Scratch<int> err(1, stream);
        SFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
        sfb::SceneDev sc = sfb::scene_dev(*s->density, *s->tvol->values, s->d_dt, s->model, *s->table,
                                          s->template_scale);
        for (int64_t q0 = 0; q0 < n; q0 += chunk) {
            int64_t m = std::min(chunk, n - q0);
            const double* qd = iq.d + 9 * q0;
            {
                StageScope st(SF_STAGE_CONFIG, stream);
                sfb::launch_make_cfg8(*medium, m, qd, media ? media + 4 * q0 : nullptr, cfg8.p, stream);
            }
            const double* mq = media ? media + 4 * q0 : nullptr;
            {
                StageScope st(SF_STAGE_FEATURES_DIFFUSE, stream);
                sfb::launch_sample_features(sc, sfb::template_dev(*s->dt), m, qd, mq, feats.p, feat, 0,
                                            err.p, stream);
            }
            {
                StageScope st(SF_STAGE_FEATURES_HIGHLIGHT, stream);
                sfb::launch_sample_features(sc, sfb::template_dev(*s->ht), m, qd, mq, feats.p, feat,
                                            3 * nd, err.p, stream);
            }
            {
                StageScope st(SF_STAGE_SLICE, stream);
                sfb::launch_slice(c, m, feats.p, slices.p, stream);
            }
            {
                StageScope st(SF_STAGE_BACKBONE, stream);
                sfb::launch_backbone_fp32(*b, m, slices.p, cfg8.p, oy.d ? oy.d + 3 * q0 : nullptr,
                                          oF.d ? oF.d + 3 * q0 : nullptr, stream);
            }
        }
        if (!oF.host && !oy.host && !iq.buf.p) {
            // Device in, device out: stay asynchronous (no host round trip). A
            // highlight placement failure (entry == p, where the reference throws)
            // shows up as NaN rows in the outputs instead of an error status.
            return;
        }
        int herr = 0;
        SFB_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        oF.finish();
        oy.finish();
        sync(stream);
        if (herr) fail(SF_ERR_INVALID_ARGUMENT, "place_template: entry coincides with p");
}
}  // namespace

int sf_debug_query_pools(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium, int64_t n,
                         const double* queries, float* pools, sf_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        const sfb::SortLayout L = sfb::sort_layout(b->cfg);
        Out<float> o(pools, size_t(L.n_layers) * size_t(n) * 8, stream);
        Scratch<double> Fd(size_t(n) * 3, stream);
        query_impl(s, b, medium, nullptr, n, queries, SF_PRECISION_BF16, Fd.p, nullptr, stream, o.d);
        o.finish();
        sync(stream);
    });
}

int sf_query(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium, int64_t n,
             const double* queries, int precision, double* F_out, float* y_out, sf_stream stream) {
    return guard([&] { query_impl(s, b, medium, nullptr, n, queries, precision, F_out, y_out, stream); });
}

// ---- image entry point: bake_field + render_volume ------------------------------------------
int sf_bake_field(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium,
                  const double camera_pos[3], int precision, float* out, sf_stream stream) {
    return guard([&] {
        const sf_grid& g = *s->density;
        const size_t nvox = g.count();
        Out<float> o(out, 3 * nvox, stream);
        SFB_CUDA(cudaMemsetAsync(o.d, 0, 3 * nvox * sizeof(float), stream));
        Scratch<int> idx(nvox, stream), cnt(1, stream);
        size_t tmp_bytes = 0;
        sfb::launch_occupied(g, idx.p, cnt.p, nullptr, tmp_bytes, stream);
        Scratch<uint8_t> tmp(tmp_bytes, stream);
        sfb::launch_occupied(g, idx.p, cnt.p, tmp.p, tmp_bytes, stream);
        int m = 0;
        SFB_CUDA(cudaMemcpyAsync(&m, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        sync(stream);
        if (m > 0) {
            Scratch<double> rows(size_t(m) * 9, stream), F(size_t(m) * 3, stream);
            sfb::launch_bake_rows(g, idx.p, cnt.p, m, camera_pos, s->tvol->light, rows.p, stream);
            query_impl(s, b, medium, nullptr, m, rows.p, precision, F.p, nullptr, stream);
            sfb::launch_scatter_field(g, idx.p, cnt.p, m, F.p, o.d, stream);
        }
        o.finish();
        sync(stream);
    });
}

int sf_render_volume(const sf_grid* density, const double sigma_t[3], const double albedo[3], int material_class,
                     const double camera_pos[3], const double look_at[3], const double up[3], double vfov_deg,
                     int width, int height, const float* field, double step_scale, const double background[3],
                     float* img, sf_stream stream) {
    return guard([&] {
        // Camera::Camera (src/camera.cpp:15-18), MediumProperties::validate (src/volume_grid.cpp:132-154)
        if (width <= 0 || height <= 0) fail(SF_ERR_INVALID_ARGUMENT, "camera: resolution must be positive");
        if (vfov_deg <= 0.0 || vfov_deg >= 180.0) fail(SF_ERR_INVALID_ARGUMENT, "camera: vfov out of range");
        validate_albedo(albedo);
        const double lo = (material_class <= 1) ? 0.0 : 0.5, hi = (material_class <= 1) ? 0.5 : 1.0;
        for (int c = 0; c < 3; ++c)
            if (albedo[c] < lo || albedo[c] > hi)
                fail(SF_ERR_BAD_VALUE, "medium: albedo outside the material class range");
        for (int c = 0; c < 3; ++c)
            if (!(sigma_t[c] > 0.0) || !std::isfinite(sigma_t[c]))
                fail(SF_ERR_BAD_VALUE, "medium: sigma_t scale must be positive");
        if (!(step_scale > 0.0)) fail(SF_ERR_INVALID_ARGUMENT, "render: step_scale must be positive");
        In<float> f(field, field ? 3 * density->count() : 0, stream);
        Out<float> o(img, size_t(width) * height * 3, stream);
        sfb::launch_render(*density, f.d, sigma_t, albedo, camera_pos, look_at, up, vfov_deg, width, height,
                           step_scale, background, o.d, stream);
        o.finish();
        sync(stream);
    });
}

int sf_query_media(const sf_scene* s, const sf_backbone* b, int64_t n, const double* queries, const double* media,
                   int precision, double* F_out, float* y_out, sf_stream stream) {
    return guard([&] {
        if (!media) fail(SF_ERR_INVALID_ARGUMENT, "query_media: media rows required");
        query_impl(s, b, nullptr, media, n, queries, precision, F_out, y_out, stream);
    });
}

int sf_profile_enable(int on) {
    g_prof_on.store(on != 0);
    return SF_OK;
}

int sf_profile_read(double stage_ms[SF_STAGE_COUNT], int64_t stage_launches[SF_STAGE_COUNT]) {
    return guard([&] {
        std::vector<StageRec> recs;
        {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            recs.swap(g_recs);
        }
        for (int i = 0; i < SF_STAGE_COUNT; ++i) {
            stage_ms[i] = 0.0;
            if (stage_launches) stage_launches[i] = 0;
        }
        cudaError_t first = cudaSuccess;
        for (StageRec& r : recs) {
            float ms = 0.0f;
            cudaError_t e = cudaEventSynchronize(r.b);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
            if (e != cudaSuccess && first == cudaSuccess) first = e;
            stage_ms[r.stage] += ms;
            if (stage_launches) stage_launches[r.stage] += r.launches;
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        sfb::cuda_check(first, "profile events");
    });
}

int sf_host_alloc(size_t bytes, void** out) {
    return guard([&] {
        if (!out) fail(SF_ERR_INVALID_ARGUMENT, "sf_host_alloc: null output");
        *out = nullptr;
        if (bytes == 0) return;
        constexpr size_t kHuge = size_t(2) << 20;
        const size_t size = (bytes + kHuge - 1) / kHuge * kHuge;
        void* p = nullptr;
        if (posix_memalign(&p, kHuge, size) != 0 || !p) fail(SF_ERR_CUDA, "sf_host_alloc: out of host memory");
        madvise(p, size, MADV_HUGEPAGE);  // best effort (THP may be off)
        std::memset(p, 0, size);          // fault the pages in before pinning
        const cudaError_t e = cudaHostRegister(p, size, cudaHostRegisterPortable);
        if (e != cudaSuccess) {
            free(p);
            sfb::cuda_check(e, "cudaHostRegister");
        }
        *out = p;
    });
}

int sf_host_free(void* p) {
    return guard([&] {
        if (!p) return;
        sfb::cuda_check(cudaHostUnregister(p), "cudaHostUnregister");
        free(p);
    });
}

int64_t sf_launch_count(void) { return g_launches.load(); }

int sf_probe_l2_read(size_t bytes, int reps, double* gbs) {
    return guard([&] {
        if (!gbs || bytes < 4096 || reps < 1) fail(SF_ERR_INVALID_ARGUMENT, "sf_probe_l2_read: bad arguments");
        *gbs = sfb::probe_l2_read_gbs(bytes, reps);
    });
}

int sf_debug_tc_profile(uint64_t out[16]) {
    return guard([&] {
        unsigned long long v[16];
        sfb::tc_read_prof(v);
        for (int i = 0; i < 16; ++i) out[i] = v[i];
    });
}

}  // extern "C"

extern "C" void sf_backbone_destroy(sf_backbone* b) {
    if (!b) return;
    cudaFree(b->d_params);
    if (b->d_paramsT) cudaFree(b->d_paramsT);
    sfb::tc_release(*b);
    delete b;
}
