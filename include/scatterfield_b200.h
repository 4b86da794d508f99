/* include/scatterfield_b200.h — the drop-in C ABI of the B200 hot path.
 *
 * Replaces the per-shading-point path of the reference's `scatterfield::core`
 * library (arxiv/paper_2401_14051; /root/reference/proj/core). Each entry point
 * cites the reference interface it stands in for (header file:line, all under
 * proj/core/include/scatterfield/). The C++ shim include/scatterfield_b200.hpp
 * re-exposes these with the reference's C++ signatures and exceptions.
 *
 * Conventions
 *  - Plain C types only. Status: 0 = OK, else (Errc ordinal + 1) as in
 *    error.h:11-21, or SF_ERR_CUDA for a device failure; sf_last_error() returns
 *    the thread-local message of the last failing call on this thread.
 *  - Handles own device-resident (HBM) data. Array arguments marked "h/d" may be
 *    host or device pointers (detected with cudaPointerGetAttributes); host
 *    arrays are staged through the given stream. Pinned host memory keeps the
 *    copies asynchronous.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls that write
 *    host memory synchronize that stream before returning.
 *  - Grids are x-fastest float32 (volume_grid.h:28-33). Query rows are 9
 *    doubles: p, omega, light (feature_pipeline.h:57-60 CenterSpec). Feature rows
 *    are float32 diffuse{density[nd], transmittance[nd], phase[nd]} followed by
 *    highlight{...[nh]} (feature_pipeline.h:50-55 SampleFeatureBlock x 2).
 *    Config rows are 8 doubles: n_g, g0, g1, g2, albedo.xyz, alpha
 *    (predictor.h:20-27 ConfigParams).
 *  - Results do not depend on the launch configuration or on the number of GPUs.
 */
#ifndef SCATTERFIELD_B200_H
#define SCATTERFIELD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sf_stream; /* == cudaStream_t */

enum sf_status {
    SF_OK = 0,
    SF_ERR_IO = 1,
    SF_ERR_MALFORMED_HEADER = 2,
    SF_ERR_BAD_DIMS = 3,
    SF_ERR_BAD_VALUE = 4,
    SF_ERR_TRUNCATED = 5,
    SF_ERR_INVALID_ARGUMENT = 6,
    SF_ERR_SHAPE_MISMATCH = 7,
    SF_ERR_PROVENANCE_MISMATCH = 8,
    SF_ERR_NUMERIC = 9,
    SF_ERR_CUDA = 100
};

/* FP32: the reference's arithmetic (parity path). BF16 / FP16: the production path — tcgen05
 * tensor-core network with 16-bit operands (bfloat16 or IEEE half) and fp32 accumulation, same
 * rate; fp16 rounds 8x finer (10-bit mantissa) for the feature and activation ranges here. */
enum sf_precision { SF_PRECISION_FP32 = 0, SF_PRECISION_BF16 = 1, SF_PRECISION_FP16 = 2 };
enum sf_template_kind { SF_TEMPLATE_DIFFUSE = 0, SF_TEMPLATE_HIGHLIGHT = 1 };
enum sf_phase_kind { SF_PHASE_ISOTROPIC = 0, SF_PHASE_HG = 1, SF_PHASE_MULTI_HG = 2 };

typedef struct sf_grid sf_grid;               /* DensityGrid (volume_grid.h:17-58) */
typedef struct sf_pyramid sf_pyramid;         /* DensityPyramid (volume_grid.h:62-72) */
typedef struct sf_tvol sf_tvol;               /* TransmittanceFeatureVolume (feature_pipeline.h:38-47) */
typedef struct sf_phase_table sf_phase_table; /* PhaseTable (phase.h:72-99) */
typedef struct sf_template sf_template;       /* SamplingTemplate (templates.h:18-34) */
typedef struct sf_backbone sf_backbone;       /* Backbone<float> (predictor.h:53-56) */
typedef struct sf_scene sf_scene;             /* bound query inputs, see sf_scene_create */

/* PhaseModel (phase.h:13-41); at most 3 lobes (Skin). */
typedef struct {
    int kind; /* sf_phase_kind */
    int n_lobes;
    double weight[3];
    double g[3];
} sf_phase_model;

/* BackboneConfig (predictor.h:33-46). */
typedef struct {
    int n_diffuse_layers;
    int diffuse_counts[16];
    int n_highlight_layers;
    int highlight_counts[16];
    int width, merge_width, head_width;
    double gamma;
    uint64_t seed;
    int literal_attention;
} sf_backbone_config;

/* The medium part of ConfigParams; alpha = angle(omega, l) is per query
 * (make_config, predictor.h:30-31). */
typedef struct {
    int n_g;
    double g[3];
    double albedo[3];
} sf_medium_params;

const char* sf_last_error(void);
const char* sf_version(void);
int sf_device_count(void);

/* ---- DensityGrid ----------------------------------------------------------- */
/* DensityGrid(nx,ny,nz,voxel_size,origin) + values (volume_grid.h:20-21).
 * values: h/d, may be NULL (zeros). */
int sf_grid_create(int nx, int ny, int nz, double voxel_size, const double origin[3],
                   const float* values, sf_grid** out);
int sf_grid_info(const sf_grid* g, int dims[3], double* voxel_size, double origin[3]);
const float* sf_grid_device_ptr(const sf_grid* g);
int sf_grid_download(const sf_grid* g, float* dst /* h/d */, sf_stream stream);
void sf_grid_destroy(sf_grid* g);
/* sample_trilinear for n points (volume_grid.h:40-42); pts h/d [n][3], out h/d [n]. */
int sf_grid_sample_trilinear(const sf_grid* g, int64_t n, const double* pts, double* out,
                             sf_stream stream);

/* ---- DensityPyramid -------------------------------------------------------- */
/* DensityPyramid(const DensityGrid&) / build_pyramid (volume_grid.h:65,100). */
int sf_pyramid_build(const sf_grid* finest, sf_pyramid** out, sf_stream stream);
int sf_pyramid_level_count(const sf_pyramid* p);
/* Borrowed view of level i, valid while the pyramid lives (volume_grid.h:68). */
const sf_grid* sf_pyramid_level(const sf_pyramid* p, int level);
void sf_pyramid_destroy(sf_pyramid* p);

/* ---- transmittance (feature_pipeline.h:82-122) ------------------------------- */
/* graded_transmittance(pyramid, level, light, lambda, step) (feature_pipeline.h:82-84). */
int sf_graded_transmittance(const sf_pyramid* p, int level, const double light[3],
                            double lambda, double step, sf_grid** out, sf_stream stream);
/* conv3_replicate(grid, kernel) (feature_pipeline.h:87). */
int sf_conv3_replicate(const sf_grid* in, const float kernel[27], sf_grid** out,
                       sf_stream stream);
/* combine_transmittance(fields, weights) (feature_pipeline.h:91-93); kernels
 * [n][27] and scales [n] are host arrays; light is the fields' light direction. */
int sf_combine_transmittance(const sf_grid* const* fields, int n, const float* kernels,
                             const float* scales, const double light[3], sf_tvol** out,
                             sf_stream stream);
/* build_transmittance_volume(pyramid, light, weights, cfg) (feature_pipeline.h:119-122).
 * kernels == NULL selects CombinerWeights::identity (feature_pipeline.h:34). */
int sf_build_transmittance_volume(const sf_pyramid* p, const double light[3],
                                  const float* kernels, const float* scales, double lambda,
                                  double step_scale, sf_tvol** out, sf_stream stream);
/* Build flags. SF_BUILD_FP32_MARCH: the graded transmittance summed in FP32 (ray setup, plane
 * tap weights and sample positions FP64) — the production build feeding the bf16 query path:
 * |dT| ~3e-7 against the FP64 reference march, ~2x faster. 0 = FP64 sums, bit-identical to the
 * reference's march in practice. Both evaluate the midpoint sum of every voxel through the
 * shared per-plane tap lists (sf_build.cu, k_tap_build / k_graded_cols). */
enum { SF_BUILD_FP32_MARCH = 1 };
int sf_build_transmittance_volume_ex(const sf_pyramid* p, const double light[3],
                                     const float* kernels, const float* scales, double lambda,
                                     double step_scale, int flags, sf_tvol** out, sf_stream stream);
/* Rows z in [z0, z1) of build_transmittance_volume's level-0 values, bit-identical to the
 * same rows of the full build: the per-light build sharded by z-slab over GPUs (SURVEY.md
 * §8e). Level 0 is marched only for the slab plus a 2-row halo, coarser levels whole.
 * out h/d [(z1-z0)][ny][nx] (device: asynchronous on `stream`); gather the slabs into
 * sf_scene_tvol_storage, or wrap them with sf_tvol_from_values. */
int sf_build_transmittance_slab(const sf_pyramid* p, const double light[3], const float* kernels,
                                const float* scales, double lambda, double step_scale, int flags, int z0,
                                int z1, float* out, sf_stream stream);
/* TransmittanceFeatureVolume{light_dir, values} from explicit values (the struct's
 * public members, feature_pipeline.h:38-41); values h/d [nz][ny][nx]. */
int sf_tvol_from_values(int nx, int ny, int nz, double voxel_size, const double origin[3],
                        const float* values, const double light[3], sf_tvol** out);
/* Borrowed level-0 grid of the volume (TransmittanceFeatureVolume::values). */
const sf_grid* sf_tvol_values(const sf_tvol* t);
void sf_tvol_destroy(sf_tvol* t);
/* light_entry_point(bounds, p, light) (feature_pipeline.h:98); host-side. */
int sf_light_entry_point(const double lo[3], const double hi[3], const double p[3],
                         const double light[3], double out[3]);

/* ---- PhaseTable (phase.h:72-99) ---------------------------------------------- */
/* PhaseTable(g_res, angle_res, aperture_res, quad_nodes), built on the GPU. */
int sf_phase_table_build(int g_res, int angle_res, int aperture_res, int quad_nodes,
                         sf_phase_table** out, sf_stream stream);
/* PhaseTable::from_values (phase.h:88-89); values h/d. */
int sf_phase_table_from_values(int g_res, int angle_res, int aperture_res,
                               const float* values, sf_phase_table** out);
int sf_phase_table_info(const sf_phase_table* t, int dims[3]);
int sf_phase_table_download(const sf_phase_table* t, float* dst, sf_stream stream);
/* lookup_hg for n triples (phase.h:79-80); all arrays h/d. */
int sf_phase_table_lookup_hg(const sf_phase_table* t, int64_t n, const double* g,
                             const double* angle, const double* half_angle, double* out,
                             sf_stream stream);
void sf_phase_table_destroy(sf_phase_table* t);

/* ---- SamplingTemplate (templates.h:18-76) ------------------------------------ */
/* points: host [total][3] template-local f64; cap_radii: host [n_layers]. */
int sf_template_create(int kind, int n_layers, const int* counts, const double* points,
                       const double* cap_radii, double gen_distance, double cone_half_angle,
                       sf_template** out);
int sf_template_total_points(const sf_template* t);
/* place_template + placed_cap_radii (templates.h:69-76) for n queries:
 * p/omega/entry h/d [n][3]; out_pts h/d [n][total][3]; out_caps h/d [n][total]. */
int sf_place_template(const sf_template* t, int64_t n, const double* p, const double* omega,
                      const double* entry, double template_scale, double* out_pts,
                      double* out_caps, sf_stream stream);
void sf_template_destroy(sf_template* t);

/* ---- sample_features (feature_pipeline.h:105-110) ---------------------------- */
/* Batched sample_features for one template: queries h/d [n][9];
 * out h/d [n][3][npts] = {density, transmittance, phase} per query. */
int sf_sample_features(const sf_grid* density, const sf_tvol* tvol, const sf_template* tmpl,
                       const sf_phase_model* model, const sf_phase_table* table,
                       double template_scale, int64_t n, const double* queries, float* out,
                       sf_stream stream);

/* ---- Backbone (predictor.h:33-139) ------------------------------------------- */
/* make_backbone<float> (predictor.h:59); params NULL = the reference He-uniform
 * init seeded by config->seed (neural.h:109-111), else host/device f32 values in
 * canonical parameter order (src/predictor.cpp:62-109). */
int sf_backbone_create(const sf_backbone_config* config, const float* params,
                       sf_backbone** out);
int64_t sf_backbone_param_count(const sf_backbone* b);
int sf_backbone_download_params(const sf_backbone* b, float* dst, sf_stream stream);
void sf_backbone_destroy(sf_backbone* b);
/* predict_y + decode_prediction over a batch (predictor.h:94-99; predict_field
 * :138-139): features h/d [n][3(nd+nh)], config8 h/d [n][8]; y_out h/d [n][3]
 * (may be NULL), F_out h/d [n][3] (may be NULL). */
int sf_predict(const sf_backbone* b, int64_t n, const float* features, const double* config8,
               int precision, float* y_out, double* F_out, sf_stream stream);

/* ---- fused per-shading-point query (render_neural's bake loop,
 *      src/predictor.cpp:598-609) ------------------------------------------------ */
/* Binds density + transmittance volume + both templates + phase model + table.
 * The handles must outlive the scene. */
int sf_scene_create(const sf_grid* density, const sf_tvol* tvol, const sf_template* diffuse,
                    const sf_template* highlight, const sf_phase_model* model,
                    const sf_phase_table* table, double template_scale, sf_scene** out);
void sf_scene_destroy(sf_scene* s);
/* Per-light / per-frame rebuild of a scene's transmittance feature volume:
 * build_transmittance_volume(pyramid, light, weights, cfg) (feature_pipeline.h:119-122) into the
 * scene's own volume, then the query records, asynchronously on `stream` (no host sync; one
 * allocation on the first call). This is render_neural's per-call build
 * (src/predictor.cpp:593-599) for a renderer that keeps the scene across lights (config C3) or
 * frames (config C5). `p` must be the pyramid of the scene's density grid; kernels == NULL
 * selects the identity combiner; flags as sf_build_transmittance_volume_ex. */
int sf_scene_relight(sf_scene* s, const sf_pyramid* p, const double light[3], const float* kernels,
                     const float* scales, double lambda, double step_scale, int flags, sf_stream stream);
/* The scene's own transmittance storage (device, [nz][ny][nx] f32, allocated on first use) for a
 * volume assembled outside the library — the per-light build sharded by z-slab over GPUs
 * (sf_build_transmittance_slab on every rank, then an all-gather into this storage);
 * sf_scene_commit_tvol then makes it the scene's volume (light = its light direction) and
 * refreshes the query records on `stream`. */
int sf_scene_tvol_storage(sf_scene* s, float** out);
int sf_scene_commit_tvol(sf_scene* s, const double light[3], sf_stream stream);
/* For each query row (p, omega, l): sample_features for both templates,
 * make_config (alpha = angle(omega, l)), backbone forward, decode. queries h/d
 * [n][9]; F_out h/d [n][3] f64; y_out optional h/d [n][3] f32.
 * Errors: a row whose highlight placement is undefined (light entry == p, where the
 * reference's place_template throws, src/templates.cpp:219-220) makes the call return
 * SF_ERR_INVALID_ARGUMENT when any argument is host memory (the call synchronizes); with
 * device queries and outputs the call stays asynchronous and such rows come out as NaN
 * (y and F, both precisions). */
int sf_query(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium,
             int64_t n, const double* queries, int precision, double* F_out, float* y_out,
             sf_stream stream);
/* sf_query with a per-query medium (config C4: per-voxel albedo and g sampled at p by the
 * caller): media h/d [n][4] = {g, albedo r, g, b}; each query uses PhaseModel::hg(g) for its
 * phase features (sample_features(.., model, ..), feature_pipeline.h:105-110) and
 * ConfigParams{g = {g}, albedo} for make_config / decode_prediction (predictor.h:20-31, 99). */
int sf_query_media(const sf_scene* s, const sf_backbone* b, int64_t n, const double* queries,
                   const double* media, int precision, double* F_out, float* y_out, sf_stream stream);

/* bake_field (src/predictor.cpp:559-581) as render_neural runs it (:598-609): the query at
 * every occupied voxel centre (density > 0) of the scene's density grid, omega =
 * normalize(p - camera_pos), l = the scene tvol's light; out h/d [3][nz][ny][nx] f32 =
 * float(F) per channel, 0 at empty voxels. */
int sf_bake_field(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium,
                  const double camera_pos[3], int precision, float* out, sf_stream stream);
/* render_volume (src/rte.cpp:407-447) with the camera of camera.h:19-23 (Camera(position,
 * look_at, up, vfov_degrees, width, height), centre-of-pixel primary rays) and the baked
 * field as the in-scatter provider (BakedField::sample, trilinear, 0 outside; field NULL
 * = F 0). material_class: 0 air, 1 gas, 2 solid/liquid, 3 skin (MediumProperties::validate
 * ranges). img h/d [height][width][3] f32 (ImageF::rgb). */
int sf_render_volume(const sf_grid* density, const double sigma_t[3], const double albedo[3],
                     int material_class, const double camera_pos[3], const double look_at[3],
                     const double up[3], double vfov_deg, int width, int height, const float* field,
                     double step_scale, const double background[3], float* img, sf_stream stream);

/* ---- instrumentation (per-stage CUDA-event timing) -------------- */
enum sf_stage {
    SF_STAGE_CONFIG = 0,             /* make_config rows */
    SF_STAGE_FEATURES_DIFFUSE = 1,   /* sample_features, diffuse template */
    SF_STAGE_FEATURES_HIGHLIGHT = 2, /* sample_features, highlight template */
    SF_STAGE_SLICE = 3,              /* per-layer sort + pools */
    SF_STAGE_BACKBONE = 4,           /* network forward + decode */
    SF_STAGE_SAMPLE_SORT = 5,        /* fused features + sort/pool + bf16 operand packing */
    SF_STAGE_MARCH = 6,              /* graded transmittance, every level (sf_scene_relight) */
    SF_STAGE_COMBINER = 7,           /* the 3D-CNN combiner: conv3 + combine (sf_scene_relight) */
    SF_STAGE_RECORDS = 8,            /* query records of the new volume (sf_scene_relight) */
    SF_STAGE_COUNT = 9
};
/* When enabled, sf_query/sf_predict/sf_scene_relight record a CUDA event pair around every stage on
 * the caller's stream (no synchronization). sf_profile_read synchronizes on those
 * events, writes the summed device milliseconds and launch counts per stage, and
 * resets the accumulators. */
int sf_profile_enable(int on);
int sf_profile_read(double stage_ms[SF_STAGE_COUNT], int64_t stage_launches[SF_STAGE_COUNT]);
/* Page-locked host buffers for the host-memory query path (no reference counterpart: the
 * reference computes on host vectors). Allocated 2 MiB-aligned with transparent huge pages
 * requested (madvise), touched, then registered with CUDA: the DMA engine's address
 * translations stay few and warm, where 4 KiB-page pinned memory starts ~4x slower on its
 * first transfers (tools/e2e_state.py). sf_host_free unregisters and frees. */
int sf_host_alloc(size_t bytes, void** out);
int sf_host_free(void* p);
/* Number of kernels this library has launched since load (all entry points). */
int64_t sf_launch_count(void);
/* Diagnostics (parity tests): the production (bf16 path) sampler's fp32 per-layer pools for
 * query rows h/d [n][9] — slice_layers' {mean, max} per feature type (src/predictor.cpp:153-191)
 * as k_sample_sort computes them before the bf16 packing: pools h/d [n_layers][n][8] =
 * {mean density, phase, transmittance, max density, phase, transmittance, 0, 0}, layers
 * diffuse then highlight in template order. Runs the bf16 query (F discarded). */
int sf_debug_query_pools(const sf_scene* s, const sf_backbone* b, const sf_medium_params* medium, int64_t n,
                         const double* queries, float* pools, sf_stream stream);
/* Diagnostics: with SF_DEBUG_TC set in the environment, CTA 0 of the tensor-core
 * backbone accumulates clock64 cycles per phase (0 bundle wait FC-1, 1 attention,
 * 2 FC-1 MMA, 3 FC-1 epilogue, 4 bundle wait FC-2, 5 FC-2 MMA, 6 FC-2 epilogue,
 * 7 other, 8 total); reading resets them. */
int sf_debug_tc_profile(uint64_t out[16]);
/* Diagnostics (no reference counterpart): L2 read bandwidth in GB/s of 32-byte loads (the
 * sampler's gather width) streaming `reps` times over an L2-resident buffer of `bytes`;
 * bench.py reports the sampling kernel's roofline against it next to the HBM figure. */
int sf_probe_l2_read(size_t bytes, int reps, double* gbs);

#ifdef __cplusplus
}
#endif
#endif /* SCATTERFIELD_B200_H */
