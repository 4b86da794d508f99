/* oracle/sf_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's per-shading-point hot path
 * (arxiv/paper_2401_14051 "scatterfield", /root/reference/proj/core). It is the
 * CHECKER for the B200 product in paper_2401_14051_b200/: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may call it. It is
 * pinned against the reference itself (oracle/_ref/libsf_ref.so, compiled from
 * the reference sources) by tests/test_oracle_pin.py and against the committed
 * golden fixtures under tests/golden/.
 *
 * Numeric conventions follow the reference exactly: FP64 geometry and
 * interpolation over float storage, FP32 network arithmetic with sequential
 * `acc = b; acc += w*x` accumulation, no FMA contraction (built with plain
 * -O2, no -march, like proj/core/CMakeLists.txt:31).
 */
#ifndef SF_ORACLE_H
#define SF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene for sample_features (proj/core/src/feature_pipeline.cpp:139-172). */
typedef struct {
    const float* density; /* level-0 grid, x-fastest (inc/volume_grid.h:28-33) */
    const float* tvol;    /* transmittance feature volume, same geometry */
    int nx, ny, nz;
    double vs;
    double origin[3];
    /* diffuse template: per-layer point counts, points (x,y,z f64), cap radii */
    int nl_d;
    const int* counts_d;
    const double* pts_d;
    const double* caps_d;
    /* highlight template */
    int nl_h;
    const int* counts_h;
    const double* pts_h;
    const double* caps_h;
    double gen_distance;
    /* phase model (inc/phase.h:13-41): kind 0 iso, 1 HG, 2 multi-HG */
    int phase_kind;
    int n_lobes;
    double lobe_w[3];
    double lobe_g[3];
    const float* table; /* [g][angle][aperture] */
    int g_res, a_res, h_res;
    double template_scale;
} or_scene;

/* BackboneConfig (inc/predictor.h:33-46). */
typedef struct {
    int nl_d;
    int counts_d[16];
    int nl_h;
    int counts_h[16];
    int width, merge_width, head_width;
    int literal;
    double gamma;
    uint64_t seed;
} or_backbone_cfg;

double or_sample_trilinear(const float* v, int nx, int ny, int nz, double vs,
                           const double origin[3], const double p[3]);
int or_pyramid(const float* vals, int nx, int ny, int nz, float* out, int* n_levels,
               int* dims_out /* 3 per level */);
int or_graded(const float* vals, int nx, int ny, int nz, double vs, const double origin[3],
              int level, const double light[3], double lambda, double step, float* out);
void or_conv3(const float* in, int nx, int ny, int nz, const float k27[27], float* out);
int or_build_tvol(const float* vals, int nx, int ny, int nz, double vs, const double origin[3],
                  const double light[3], double lambda, double step_scale,
                  const float* kernels, const float* scales, float* out);
void or_gauss_legendre(int n, double* nodes, double* weights);
void or_phase_table(int g_res, int a_res, int h_res, int nodes, float* out);
double or_lookup_hg(const float* table, int g_res, int a_res, int h_res, double g,
                    double angle, double half);
void or_light_entry_point(const double lo[3], const double hi[3], const double p[3],
                          const double light[3], double out[3]);
int or_place_highlight(const or_scene* s, const double p[3], const double omega[3],
                       const double entry[3], double* out_pts, double* out_caps);
int or_features(const or_scene* s, int64_t q, const double* centers9, float* out);

int64_t or_backbone_param_count(const or_backbone_cfg* cfg);
void or_backbone_init(const or_backbone_cfg* cfg, float* params);
int or_predict(const or_backbone_cfg* cfg, const float* params, int64_t q, const float* feats,
               const double* cfg8, double* y_out, double* F_out);

uint64_t or_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif
#endif
