// sf_internal.h — handle layouts and launcher declarations shared by the
// translation units of libsf_b200.so (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/scatterfield_b200.h"
#include "sf_device.cuh"

// ---- error plumbing ---------------------------------------------------------
namespace sfb {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(SF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define SFB_CUDA(x) ::sfb::cuda_check((x), #x)

// ---- launch configuration helpers --------------------------------------------
int sm_count();
void count_launch();  // every kernel launch of the library increments sf_launch_count()

// Image entry point (sf_render.cu): occupied-voxel compaction, bake rows, field scatter, march.
int64_t launch_occupied(const sf_grid& g, int* idx, int* count, void* tmp, size_t& tmp_bytes, cudaStream_t s);
void launch_bake_rows(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double cam[3],
                      const double light[3], double* rows, cudaStream_t s);
void launch_scatter_field(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double* F,
                          float* out, cudaStream_t s);
void launch_render(const sf_grid& density, const float* field, const double mu[3], const double albedo[3],
                   const double pos[3], const double look_at[3], const double up[3], double vfov_deg, int width,
                   int height, double step_scale, const double bg[3], float* img, cudaStream_t s);

}  // namespace sfb

// ---- handle layouts ----------------------------------------------------------
struct sf_grid {
    int nx = 0, ny = 0, nz = 0;
    double vs = 1.0;
    double origin[3] = {0, 0, 0};
    double hi[3] = {0, 0, 0};  // origin + n*vs (DensityGrid::bounds)
    float* d = nullptr;
    bool owned = true;
    cudaStream_t pool_stream = nullptr;  // set: stream-ordered scratch, freed with cudaFreeAsync
    bool pooled = false;
    size_t count() const { return size_t(nx) * ny * nz; }
    sfb::GridDev dev() const {
        int e;
        double ivs = std::frexp(vs, &e) == 0.5 ? 1.0 / vs : 0.0;
        return sfb::GridDev{d,         nx,        ny,    nz,    vs,    origin[0],
                            origin[1], origin[2], hi[0], hi[1], hi[2], ivs,
                            uint32_t((nx + 2) >> 1) << 2, uint32_t(ny + 1) * (uint32_t((nx + 2) >> 1) << 2)};
    }
};

namespace sfb {
// Padded pair records of one pyramid level (the input of the graded-transmittance tap kernels),
// made on first use and kept with the pyramid (the density is immutable): [FP32, FP64] x
// [x-fastest, z-fastest]. `ready` orders later users on other streams after the fill.
struct PadCache {
    std::mutex mu;
    void* rec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    cudaEvent_t ready[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    ~PadCache() {
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                if (rec[a][b]) cudaFree(rec[a][b]);
                if (ready[a][b]) cudaEventDestroy(ready[a][b]);
            }
    }
};
}  // namespace sfb

struct sf_pyramid {
    std::vector<sf_grid*> levels;  // level 0 is a copy of the finest grid
    float* block = nullptr;        // one allocation holding every level (levels are views)
    std::vector<std::unique_ptr<sfb::PadCache>> pads;  // one per level
};

struct sf_tvol {
    double light[3] = {0, 0, 0};
    sf_grid* values = nullptr;
    std::vector<float> kernels, scales;
};

struct sf_phase_table {
    int g = 0, a = 0, h = 0;
    float* d = nullptr;
    // [G][A][H] float4 {P(g, a, h), P(g, a, h + 1), P(g + 1, a, h), P(g + 1, a, h + 1)}: the per-query-g
    // lookup's two bilinear cells as 16-byte records (made on the first mixed-media query)
    mutable float4* d_quad = nullptr;
    mutable std::mutex quad_mu;
};

struct sf_template {
    int kind = 0;
    int n_layers = 0;
    int total = 0;
    std::vector<int> counts;
    std::vector<double> points;  // [total][3]
    std::vector<double> caps;    // [n_layers] layer cap_radius
    double gen_distance = 0.0, cone_half_angle = 0.0;
    double* d_points = nullptr;  // [total][3]
    double* d_caps = nullptr;    // [total] per-point layer cap radius (unscaled)
    float4* d_pts4 = nullptr;    // [total] {x, y, z, cap} as float
};

// Parameter layout of one stack and of the whole net, in walk_params order
// (src/predictor.cpp:62-109).
struct BackboneLayout {
    int64_t total = 0;
    int64_t stack_off[2][3];  // [kind][tau]
    int64_t merge_off;        // 3 x (W [M][2W], b [M])
    int64_t cross_off;        // W [M][3M], b [M]
    int64_t head_off[3];      // W, b
};

struct sf_backbone {
    sf_backbone_config cfg{};
    BackboneLayout layout{};
    float* d_params = nullptr;  // canonical f32 params
    float* d_paramsT = nullptr; // the same with every dense W [out][in] stored [in][out] (FP32 path, lazy)
    void* tc = nullptr;         // packed bf16 operands for the tensor-core path (lazy)
};

struct sf_scene {
    const sf_grid* density = nullptr;
    const sf_tvol* tvol = nullptr;
    const sf_template* dt = nullptr;
    const sf_template* ht = nullptr;
    sf_phase_model model{};
    const sf_phase_table* table = nullptr;
    double template_scale = 1.0;
    float2* d_dt = nullptr;  // interleaved {density, transmittance} level-0 volume
    float* d_planes = nullptr;  // phase table pre-blended at each lobe's g, [n_planes][A][H + 1] floats
    int n_planes = 0;
    float4* d_dt4 = nullptr;    // xy-quad records of the {density, transmittance} volume (k_xpair)
    float4* d_pre = nullptr;    // per diffuse point {offset (voxels), half angle}, {unit axis, light side}
    sf_tvol* own_tvol = nullptr;  // the volume sf_scene_relight builds into (owned)
    bool dt_stale = false;        // d_dt not yet refreshed after a relight (the FP32 path refreshes it)
};

// ---- launchers (defined in the .cu files) --------------------------------------
namespace sfb {

void launch_pyramid_down(const sf_grid& src, sf_grid& dst, cudaStream_t s);
// Per-light build kernels over voxel rows z in [zlo, zhi) (the whole grid, or a z-slab of a
// build sharded over GPUs). launch_combine writes rows [zlo, zhi) to out[0...].
// fast: FP32 march (production bf16 path; ~1e-6 relative optical depth) instead of the FP64 reference march
// cache (optional): the level's padded records, kept between calls
void launch_graded(const sf_grid& level, const double to_source[3], double coeff, double step, int zlo, int zhi,
                   float* out, cudaStream_t s, bool fast = false, PadCache* cache = nullptr);
// fast: FP32 accumulation / interpolation (production build), else the reference's FP64.
void launch_conv3(const sf_grid& in, const float k27[27], int zlo, int zhi, float* out, cudaStream_t s,
                  bool fast = false);
void launch_combine(const std::vector<const sf_grid*>& conv, const std::vector<float>& scales,
                    const sf_grid& base, int zlo, int zhi, float* out, cudaStream_t s, bool fast = false);
void launch_interleave(const float* density, const float* tvol, float2* out, size_t n,
                       cudaStream_t s);
void launch_phase_table(int gr, int ar, int hr, const std::vector<double>& nodes,
                        const std::vector<double>& weights, float* out, cudaStream_t s);
// The table's quad records (sf_phase_table::d_quad), made once.
const float4* phase_quad(const sf_phase_table& t, cudaStream_t s);
void launch_lookup_hg(const sf_phase_table& t, int64_t n, const double* g, const double* a,
                      const double* h, double* out, cudaStream_t s);
void launch_sample_trilinear(const sf_grid& g, int64_t n, const double* pts, double* out,
                             cudaStream_t s);
void launch_place_template(const sf_template& t, int64_t n, const double* p,
                           const double* omega, const double* entry, double ts, double* pts,
                           double* caps, int* err, cudaStream_t s);

// Query-side scene view (sampling).
struct SceneDev {
    GridDev grid;          // density geometry (v = density)
    const float2* dt;      // interleaved {density, tvol}
    const float4* dt4;     // xy-quad records, two float4 each (k_xpair; fused path)
    const float* tvol;     // plain tvol (when dt == nullptr)
    PhaseDev phase;
    double template_scale;
};
struct TemplateDev {
    int kind;
    int total;
    const double* pts;
    const double* caps;
    double gen_distance;
    const float4* pts4;  // {x, y, z, layer cap radius} in float (fused path)
};
SceneDev scene_dev(const sf_grid& density, const sf_grid& tvol, const float2* dt,
                   const sf_phase_model& m, const sf_phase_table& t, double ts);
TemplateDev template_dev(const sf_template& t);

// media: NULL, or per-query {g, albedo rgb} [n][4] (single-lobe HG per query, config C4)
void launch_sample_features(const SceneDev& sc, const TemplateDev& td, int64_t n,
                            const double* queries, const double* media, float* out, int64_t row_stride,
                            int64_t col_offset, int* err, cudaStream_t s);
int64_t slices_per_query(const sf_backbone_config& c);
void launch_slice(const sf_backbone_config& c, int64_t n, const float* feats, float* slices,
                  cudaStream_t s);
void launch_backbone_fp32(const sf_backbone& b, int64_t n, const float* slices,
                          const double* cfg8, float* y, double* F, cudaStream_t s);
void launch_make_cfg8(const sf_medium_params& m, int64_t n, const double* queries, const double* media,
                      double* cfg8, cudaStream_t s);

// Layout of the sorted-feature operand blocks produced by k_sample_sort and
// consumed by the tensor-core backbone: for every (kind, layer, tau) segment a
// [n_tiles][128 x kf] bf16 block in UMMA canonical layout (kf = pad16(n):
// sorted values, zeros; the pools enter FC-1 in fp32 from the block below), and for every (kind, layer) a
// [n_tiles*128][8] fp32 block {mean d,p,t, max d,p,t, 0, 0} for the attention.
struct SortLayout {
    int nl[2];
    int npts[2];
    int counts[2][16];
    int start[2][16];
    int kf[2][16];
    int mm_layer[2][16];
    int64_t seg_prefix[2][16][3];  // bytes per tile preceding the segment
    int64_t tile_bytes;            // all segments of one tile
    int n_layers;
};
SortLayout sort_layout(const sf_backbone_config& c);

// Tensor-core (tcgen05, bf16 operands / fp32 accumulation) backbone.
bool tc_supported(const sf_backbone_config& c);
// f16: pack the weights as fp16 (SF_PRECISION_FP16), else bf16; both packs are kept
void tc_prepare(sf_backbone& b, cudaStream_t s, bool f16 = false);
void tc_release(sf_backbone& b);
void tc_read_prof(unsigned long long* out);
// perm (optional): processing row q writes the caller's row perm[q] of y / F
void launch_backbone_tc(const sf_backbone& b, int64_t n, const uint8_t* ops, const float* mms,
                        const double* cfg8, float* y, double* F, cudaStream_t s, const int* perm = nullptr,
                        bool f16 = false);

// Fused feature sampling + per-layer sort/pool + bf16 operand packing (K5+K6).
// Samples the scene when `feats` is null, else sorts the given feature rows.
void launch_sample_sort(const SceneDev* sc, const TemplateDev* dt, const TemplateDev* ht,
                        const float* planes, int n_planes, const float4* pre, const SortLayout& L,
                        int64_t n, const void* recs, const float* feats, uint8_t* ops, float* mms,
                        int* err, cudaStream_t s, bool mixed = false, int64_t tile0 = 0,
                        int64_t layout_tiles = 0, bool f16 = false, bool l2_keep = false);
// layout_tiles > 0: this launch fills tiles [tile0, tile0 + ceil(n / 128)) of an operand /
// pool layout of layout_tiles tiles (one backbone launch over several sampling launches).
// Queries the persistent sampling grid processes per round (one per warp, every SM full):
// a window of a multiple of this many queries has no partial last round.
int64_t sample_sort_round_queries();
// Per-query context records (sampling bases, highlight frame) + make_config rows.
size_t query_rec_bytes();
// perm (optional): processing row q reads the caller's row perm[q] (locality reordering)
// row0: the batch's first row (its light is the one the diffuse constants hold; default:
// queries). dt (optional): also make those diffuse constants (launch_diffuse_light's work)
// in the same launch.
void launch_query_prep(const SceneDev& sc, const TemplateDev& ht, const sf_medium_params& m, int64_t n,
                       const double* queries, const double* media, double* cfg8, void* recs, cudaStream_t s,
                       const int* perm = nullptr, const double* row0 = nullptr, const TemplateDev* dt = nullptr,
                       const float* planes = nullptr, int n_planes = 0, float4* pre = nullptr);
// Processing order for locality: perm = the query rows grouped by the Morton code of their cell in a
// 64^3 partition of the box (a counting sort: histogram, scan, scatter; order within a cell is
// arbitrary, which no result depends on). cells: n keys of scratch; counts: kOrderCells + 1024 ints.
constexpr int kOrderCells = 1 << 18;
void launch_cell_order(const GridDev& g, int64_t n, const double* queries, uint32_t* cells, int* counts, int* perm,
                       cudaStream_t s);
void launch_xpair(const float* rho, const float* tr, int nx, int ny, int nz, float4* out, cudaStream_t s);
double probe_l2_read_gbs(size_t bytes, int reps);  // k_l2_probe: 32-byte reads of an L2-resident buffer
size_t xpair_records(int nx, int ny, int nz);  // float4 units of the padded xy-quad record layout
// Pre-blended phase planes: for each lobe, the table interpolated at that lobe's g
// (PhaseTable::lookup_hg's g axis, src/phase.cpp:191-219), [n_lobes][angle][aperture].
void launch_blend_planes(const sf_phase_table& t, const sf_phase_model& m, float* planes,
                         cudaStream_t s);

// Image entry point (sf_render.cu): occupied-voxel compaction, bake rows, field scatter, march.
int64_t launch_occupied(const sf_grid& g, int* idx, int* count, void* tmp, size_t& tmp_bytes, cudaStream_t s);
void launch_bake_rows(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double cam[3],
                      const double light[3], double* rows, cudaStream_t s);
void launch_scatter_field(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double* F,
                          float* out, cudaStream_t s);
void launch_render(const sf_grid& density, const float* field, const double mu[3], const double albedo[3],
                   const double pos[3], const double look_at[3], const double up[3], double vfov_deg, int width,
                   int height, double step_scale, const double bg[3], float* img, cudaStream_t s);

}  // namespace sfb
