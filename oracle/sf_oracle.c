/* oracle/sf_oracle.c — TEST INFRASTRUCTURE ONLY (see sf_oracle.h).
 *
 * CPU restatement of the reference hot path. Every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj/core). Pinned by
 * tests/test_oracle_pin.py against oracle/_ref/libsf_ref.so (the reference
 * compiled from its own sources) and by tests/test_oracle_golden.py against the
 * committed fixtures in tests/golden/.
 */
#include "sf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846
#define OR_INV4PI (1.0 / (4.0 * OR_PI))

/* ---- small vector helpers (inc/math.h:15-65) -------------------------------- */

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double len3(const double* a) { return sqrt(dot3(a, a)); }
static double clampd(double v, double lo, double hi) {
    /* std::min(hi, std::max(lo, v)) */
    double m = (lo < v) ? v : lo; /* std::max(lo, v) returns lo unless lo < v */
    return (m < hi) ? m : hi;     /* std::min(hi, m) returns hi unless m < hi  */
}
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* inc/math.h:53-56 */
static double angle_between(const double* a, const double* b) {
    double c = dot3(a, b) / sqrt(dot3(a, a) * dot3(b, b));
    return acos(clampd(c, -1.0, 1.0));
}

/* inc/math.h:59-65 (Duff et al. basis) */
static void orthonormal_basis(const double* n, double* t, double* b) {
    double sign = copysign(1.0, n[2]);
    double a = -1.0 / (sign + n[2]);
    double c = n[0] * n[1] * a;
    t[0] = 1.0 + sign * n[0] * n[0] * a; t[1] = sign * c; t[2] = -sign * n[0];
    b[0] = c; b[1] = sign + n[1] * n[1] * a; b[2] = -n[1];
}

/* inc/math.h:85-107 slab test */
static int intersect_box(const double* lo, const double* hi, const double* o, const double* d,
                         double* t0o, double* t1o) {
    double t0 = -1e300, t1 = 1e300;
    for (int i = 0; i < 3; ++i) {
        if (d[i] == 0.0) {
            if (o[i] < lo[i] || o[i] > hi[i]) return 0;
            continue;
        }
        double inv = 1.0 / d[i];
        double ta = (lo[i] - o[i]) * inv;
        double tb = (hi[i] - o[i]) * inv;
        if (ta > tb) { double s = ta; ta = tb; tb = s; }
        t0 = (t0 < ta) ? ta : t0; /* std::max(t0, ta) */
        t1 = (tb < t1) ? tb : t1; /* std::min(t1, tb) */
        if (t0 > t1) return 0;
    }
    *t0o = t0;
    *t1o = t1;
    return 1;
}

static void grid_bounds(int nx, int ny, int nz, double vs, const double* o, double* lo, double* hi) {
    lo[0] = o[0]; lo[1] = o[1]; lo[2] = o[2];
    hi[0] = o[0] + nx * vs; hi[1] = o[1] + ny * vs; hi[2] = o[2] + nz * vs;
}

static int contains(const double* lo, const double* hi, const double* p) {
    return p[0] >= lo[0] && p[0] <= hi[0] && p[1] >= lo[1] && p[1] <= hi[1] &&
           p[2] >= lo[2] && p[2] <= hi[2];
}

/* ---- DensityGrid (src/volume_grid.cpp:35-78) --------------------------------- */

double or_sample_trilinear(const float* v, int nx, int ny, int nz, double vs,
                           const double origin[3], const double p[3]) {
    double lo[3], hi[3];
    grid_bounds(nx, ny, nz, vs, origin, lo, hi);
    if (!contains(lo, hi, p)) return 0.0;
    double fx = (p[0] - origin[0]) / vs - 0.5;
    double fy = (p[1] - origin[1]) / vs - 0.5;
    double fz = (p[2] - origin[2]) / vs - 0.5;
    int x0 = (int)floor(fx), y0 = (int)floor(fy), z0 = (int)floor(fz);
    double tx = fx - x0, ty = fy - y0, tz = fz - z0;
    int x1 = clampi(x0 + 1, 0, nx - 1), y1 = clampi(y0 + 1, 0, ny - 1), z1 = clampi(z0 + 1, 0, nz - 1);
    x0 = clampi(x0, 0, nx - 1); y0 = clampi(y0, 0, ny - 1); z0 = clampi(z0, 0, nz - 1);
#define AT(x, y, z) ((double)v[((size_t)(z) * ny + (y)) * nx + (x)])
#define LERP(a, b, t) ((a) + (t) * ((b) - (a)))
    double c00 = LERP(AT(x0, y0, z0), AT(x1, y0, z0), tx);
    double c10 = LERP(AT(x0, y1, z0), AT(x1, y1, z0), tx);
    double c01 = LERP(AT(x0, y0, z1), AT(x1, y0, z1), tx);
    double c11 = LERP(AT(x0, y1, z1), AT(x1, y1, z1), tx);
    return LERP(LERP(c00, c10, ty), LERP(c01, c11, ty), tz);
#undef AT
}

/* src/volume_grid.cpp:64-78 midpoint rule */
static double optical_depth(const float* v, int nx, int ny, int nz, double vs, const double* o,
                            const double* p, const double* q, double step) {
    double d[3] = {q[0] - p[0], q[1] - p[1], q[2] - p[2]};
    double len = len3(d);
    if (len == 0.0) return 0.0;
    int n = (int)ceil(len / step);
    if (n < 1) n = 1;
    double h = len / n;
    double inv = 1.0 / len;
    double dir[3] = {d[0] * inv, d[1] * inv, d[2] * inv};
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        double s = (i + 0.5) * h;
        double x[3] = {p[0] + dir[0] * s, p[1] + dir[1] * s, p[2] + dir[2] * s};
        sum += or_sample_trilinear(v, nx, ny, nz, vs, o, x);
    }
    return sum * h;
}

/* src/volume_grid.cpp:91-126: 8-child FP64 mean, clamped children, stop at max dim 1 */
int or_pyramid(const float* vals, int nx, int ny, int nz, float* out, int* n_levels, int* dims_out) {
    size_t n0 = (size_t)nx * ny * nz;
    memcpy(out, vals, n0 * sizeof(float));
    int L = 1;
    if (dims_out) { dims_out[0] = nx; dims_out[1] = ny; dims_out[2] = nz; }
    const float* src = out;
    float* dst = out + n0;
    int sx = nx, sy = ny, sz = nz;
    while ((sx > sy ? (sx > sz ? sx : sz) : (sy > sz ? sy : sz)) > 1) {
        int dx = sx / 2 > 1 ? sx / 2 : 1, dy = sy / 2 > 1 ? sy / 2 : 1, dz = sz / 2 > 1 ? sz / 2 : 1;
        for (int z = 0; z < dz; ++z)
            for (int y = 0; y < dy; ++y)
                for (int x = 0; x < dx; ++x) {
                    double sum = 0.0;
                    int count = 0;
                    for (int cz = 0; cz < 2; ++cz)
                        for (int cy = 0; cy < 2; ++cy)
                            for (int cx = 0; cx < 2; ++cx) {
                                int ix = 2 * x + cx < sx - 1 ? 2 * x + cx : sx - 1;
                                int iy = 2 * y + cy < sy - 1 ? 2 * y + cy : sy - 1;
                                int iz = 2 * z + cz < sz - 1 ? 2 * z + cz : sz - 1;
                                sum += src[((size_t)iz * sy + iy) * sx + ix];
                                ++count;
                            }
                    dst[((size_t)z * dy + y) * dx + x] = (float)(sum / count);
                }
        if (dims_out) { dims_out[3 * L] = dx; dims_out[3 * L + 1] = dy; dims_out[3 * L + 2] = dz; }
        ++L;
        src = dst;
        dst += (size_t)dx * dy * dz;
        sx = dx; sy = dy; sz = dz;
    }
    *n_levels = L;
    return 0;
}

static int level_of(int nx, int ny, int nz, int level, int* dims, size_t* offset) {
    size_t off = 0;
    int sx = nx, sy = ny, sz = nz;
    for (int i = 0; i < level; ++i) {
        if ((sx > sy ? (sx > sz ? sx : sz) : (sy > sz ? sy : sz)) <= 1) return -1;
        off += (size_t)sx * sy * sz;
        sx = sx / 2 > 1 ? sx / 2 : 1; sy = sy / 2 > 1 ? sy / 2 : 1; sz = sz / 2 > 1 ? sz / 2 : 1;
    }
    dims[0] = sx; dims[1] = sy; dims[2] = sz;
    *offset = off;
    return 0;
}

static size_t pyramid_size(int nx, int ny, int nz, int* levels) {
    size_t total = 0;
    int L = 0;
    for (;;) {
        total += (size_t)nx * ny * nz;
        ++L;
        if ((nx > ny ? (nx > nz ? nx : nz) : (ny > nz ? ny : nz)) <= 1) break;
        nx = nx / 2 > 1 ? nx / 2 : 1; ny = ny / 2 > 1 ? ny / 2 : 1; nz = nz / 2 > 1 ? nz / 2 : 1;
    }
    *levels = L;
    return total;
}

/* src/feature_pipeline.cpp:37-68 graded transmittance of one level */
static void graded_level(const float* lv, int nx, int ny, int nz, double vs, const double* o,
                         int level, const double* light, double lambda, double step, float* out) {
    double len = len3(light);
    double ld[3] = {light[0] / len, light[1] / len, light[2] / len}; /* normalize(light) */
    double to_source[3] = {-ld[0], -ld[1], -ld[2]};
    double coeff = pow(lambda, level + 1);
    double lo[3], hi[3];
    grid_bounds(nx, ny, nz, vs, o, lo, hi);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                double p[3] = {o[0] + (x + 0.5) * vs, o[1] + (y + 0.5) * vs, o[2] + (z + 0.5) * vs};
                double t0, t1, tau = 0.0;
                if (intersect_box(lo, hi, p, to_source, &t0, &t1) && t1 > 0.0) {
                    double q[3] = {p[0] + to_source[0] * t1, p[1] + to_source[1] * t1,
                                   p[2] + to_source[2] * t1};
                    tau = optical_depth(lv, nx, ny, nz, vs, o, p, q, step);
                }
                out[((size_t)z * ny + y) * nx + x] = (float)exp(-coeff * tau);
            }
}

int or_graded(const float* vals, int nx, int ny, int nz, double vs, const double origin[3],
              int level, const double light[3], double lambda, double step, float* out) {
    int L;
    size_t total = pyramid_size(nx, ny, nz, &L);
    if (level < 0 || level >= L) return -1;
    float* pyr = (float*)malloc(total * sizeof(float));
    or_pyramid(vals, nx, ny, nz, pyr, &L, NULL);
    int dims[3];
    size_t off;
    level_of(nx, ny, nz, level, dims, &off);
    double lvs = vs;
    for (int i = 0; i < level; ++i) lvs = lvs * 2.0; /* src/volume_grid.cpp:104 */
    graded_level(pyr + off, dims[0], dims[1], dims[2], lvs, origin, level, light, lambda, step, out);
    free(pyr);
    return 0;
}

/* src/feature_pipeline.cpp:70-92 replicate-padded 3x3x3, FP64 accumulate */
void or_conv3(const float* in, int nx, int ny, int nz, const float k27[27], float* out) {
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                double acc = 0.0;
                int t = 0;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx, ++t) {
                            int sx = clampi(x + dx, 0, nx - 1);
                            int sy = clampi(y + dy, 0, ny - 1);
                            int sz = clampi(z + dz, 0, nz - 1);
                            acc += (double)k27[t] * in[((size_t)sz * ny + sy) * nx + sx];
                        }
                out[((size_t)z * ny + y) * nx + x] = (float)acc;
            }
}

/* src/feature_pipeline.cpp:94-128 + :200-211 (step = step_scale * level voxel size) */
int or_build_tvol(const float* vals, int nx, int ny, int nz, double vs, const double origin[3],
                  const double light[3], double lambda, double step_scale,
                  const float* kernels, const float* scales, float* out) {
    int L;
    size_t total = pyramid_size(nx, ny, nz, &L);
    float* pyr = (float*)malloc(total * sizeof(float));
    float* field = (float*)malloc((size_t)nx * ny * nz * sizeof(float));
    float* conv = (float*)malloc((size_t)nx * ny * nz * sizeof(float));
    or_pyramid(vals, nx, ny, nz, pyr, &L, NULL);
    size_t n0 = (size_t)nx * ny * nz;
    for (size_t i = 0; i < n0; ++i) out[i] = 0.0f;
    double lvs = vs;
    for (int li = 0; li < L; ++li) {
        int d[3];
        size_t off;
        level_of(nx, ny, nz, li, d, &off);
        graded_level(pyr + off, d[0], d[1], d[2], lvs, origin, li, light, lambda,
                     step_scale * lvs, field);
        float k[27];
        float sc;
        if (kernels) {
            memcpy(k, kernels + 27 * li, sizeof(k));
            sc = scales[li];
        } else { /* CombinerWeights::identity, src/feature_pipeline.cpp:29-35 */
            memset(k, 0, sizeof(k));
            k[13] = 1.0f;
            sc = (float)(1.0 / L);
        }
        or_conv3(field, d[0], d[1], d[2], k, conv);
        double scale = sc;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    double c[3] = {origin[0] + (x + 0.5) * vs, origin[1] + (y + 0.5) * vs,
                                   origin[2] + (z + 0.5) * vs};
                    double v = or_sample_trilinear(conv, d[0], d[1], d[2], lvs, origin, c);
                    size_t idx = ((size_t)z * ny + y) * nx + x;
                    out[idx] += (float)(scale * v);
                }
        lvs = lvs * 2.0;
    }
    free(pyr);
    free(field);
    free(conv);
    return 0;
}

/* ---- phase (src/quadrature.cpp:16-56, src/phase.cpp:78-253) ------------------ */

void or_gauss_legendre(int n, double* nodes, double* weights) {
    const int m = (n + 1) / 2;
    for (int i = 0; i < m; ++i) {
        double x = cos(3.14159265358979323846 * (i + 0.75) / (n + 0.5));
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
            if (fabs(dx) < 1e-15) break;
        }
        nodes[i] = -x;
        nodes[n - 1 - i] = x;
        double w = 2.0 / ((1.0 - x * x) * pp * pp);
        weights[i] = w;
        weights[n - 1 - i] = w;
    }
}

static double hg_phase(double g, double c) {
    double denom = 1.0 + g * g - 2.0 * g * c;
    denom = (denom < 1e-12) ? 1e-12 : denom; /* std::max(denom, 1e-12) */
    return OR_INV4PI * (1.0 - g * g) / (denom * sqrt(denom));
}

/* src/phase.cpp:124-145 for a single HG lobe (eval_unchecked = 0 + 1*hg) */
static double cap_integral_hg(double g, double cos_fixed, double half, int nodes,
                              const double* gn, const double* gw) {
    double mu_lo = cos(half < OR_PI ? half : OR_PI);
    int n_psi = 2 * nodes;
    double s_f = sqrt((0.0 < 1.0 - cos_fixed * cos_fixed) ? 1.0 - cos_fixed * cos_fixed : 0.0);
    double sum = 0.0;
    for (int i = 0; i < nodes; ++i) {
        double mu = 0.5 * (1.0 + mu_lo) + 0.5 * (1.0 - mu_lo) * gn[i];
        double w_mu = 0.5 * (1.0 - mu_lo) * gw[i];
        double s_mu = sqrt((0.0 < 1.0 - mu * mu) ? 1.0 - mu * mu : 0.0);
        double inner = 0.0;
        for (int j = 0; j < n_psi; ++j) {
            double psi = 2.0 * OR_PI * (j + 0.5) / n_psi;
            double cg = clampd(cos_fixed * mu + s_f * s_mu * cos(psi), -1.0, 1.0);
            inner += 0.0 + 1.0 * hg_phase(g, cg);
        }
        sum += w_mu * inner * (2.0 * OR_PI / n_psi);
    }
    return sum;
}

/* src/phase.cpp:159-177 */
void or_phase_table(int g_res, int a_res, int h_res, int nodes, float* out) {
    double* gn = (double*)malloc(sizeof(double) * nodes);
    double* gw = (double*)malloc(sizeof(double) * nodes);
    or_gauss_legendre(nodes, gn, gw);
    for (int gi = 0; gi < g_res; ++gi) {
        double g = -0.99 + 1.98 * gi / (double)(g_res - 1);
        for (int ai = 0; ai < a_res; ++ai) {
            double angle = OR_PI * ai / (double)(a_res - 1);
            double cf = cos(angle);
            for (int hi = 0; hi < h_res; ++hi) {
                double half = OR_PI * hi / (double)(h_res - 1);
                double v = half > 0.0 ? cap_integral_hg(g, cf, half, nodes, gn, gw) : 0.0;
                out[((size_t)gi * a_res + ai) * h_res + hi] = (float)v;
            }
        }
    }
    free(gn);
    free(gw);
}

/* src/phase.cpp:191-219 */
static void grid_coord(double v, double lo, double hi, int res, int* i0, double* t) {
    double u = (clampd(v, lo, hi) - lo) / (hi - lo) * (res - 1);
    int i = (int)u;
    *i0 = i < res - 2 ? i : res - 2;
    *t = u - *i0;
}

double or_lookup_hg(const float* table, int g_res, int a_res, int h_res, double g,
                    double angle, double half) {
    int gi, ai, hi;
    double gt, at, ht;
    grid_coord(g, -0.99, 0.99, g_res, &gi, &gt);
    grid_coord(angle, 0.0, OR_PI, a_res, &ai, &at);
    grid_coord(half, 0.0, OR_PI, h_res, &hi, &ht);
    double v = 0.0;
    for (int dg = 0; dg < 2; ++dg) {
        double wg = dg ? gt : 1.0 - gt;
        for (int da = 0; da < 2; ++da) {
            double wa = da ? at : 1.0 - at;
            for (int dh = 0; dh < 2; ++dh) {
                double wh = dh ? ht : 1.0 - ht;
                v += wg * wa * wh *
                     (double)table[((size_t)(gi + dg) * a_res + (ai + da)) * h_res + (hi + dh)];
            }
        }
    }
    return v;
}

/* src/phase.cpp:221-230 */
static double table_lookup(const or_scene* s, const double* fixed_dir, const double* axis,
                           double half) {
    double angle = angle_between(fixed_dir, axis);
    if (s->phase_kind == 0)
        return or_lookup_hg(s->table, s->g_res, s->a_res, s->h_res, 0.0, angle, half);
    double v = 0.0;
    for (int k = 0; k < s->n_lobes; ++k)
        v += s->lobe_w[k] *
             or_lookup_hg(s->table, s->g_res, s->a_res, s->h_res, s->lobe_g[k], angle, half);
    return v;
}

/* ---- sampling (src/feature_pipeline.cpp:130-172, src/templates.cpp:207-256) -- */

void or_light_entry_point(const double lo[3], const double hi[3], const double p[3],
                          const double light[3], double out[3]) {
    double len = len3(light);
    double ld[3] = {light[0] / len, light[1] / len, light[2] / len};
    double ts[3] = {-ld[0], -ld[1], -ld[2]};
    double t0, t1;
    if (!intersect_box(lo, hi, p, ts, &t0, &t1)) {
        for (int i = 0; i < 3; ++i) out[i] = p[i] - ld[i] * 1e-9;
        return;
    }
    double t = (t1 < 1e-9) ? 1e-9 : t1; /* std::max(t1, 1e-9) */
    for (int i = 0; i < 3; ++i) out[i] = p[i] + ts[i] * t;
}

static int total_points(int nl, const int* counts) {
    int n = 0;
    for (int i = 0; i < nl; ++i) n += counts[i];
    return n;
}

int or_place_highlight(const or_scene* s, const double p[3], const double omega[3],
                       const double entry[3], double* out_pts, double* out_caps) {
    double span[3] = {p[0] - entry[0], p[1] - entry[1], p[2] - entry[2]};
    double len = len3(span);
    if (len <= 0.0) return -1;
    double il = 1.0 / len;
    double axis[3] = {span[0] * il, span[1] * il, span[2] * il};
    double od = dot3(omega, axis);
    double t[3] = {omega[0] - axis[0] * od, omega[1] - axis[1] * od, omega[2] - axis[2] * od};
    double tl = len3(t), b[3];
    if (tl > 1e-9) {
        double it = 1.0 / tl;
        t[0] *= it; t[1] *= it; t[2] *= it;
        b[0] = axis[1] * t[2] - axis[2] * t[1];
        b[1] = axis[2] * t[0] - axis[0] * t[2];
        b[2] = axis[0] * t[1] - axis[1] * t[0];
    } else {
        orthonormal_basis(axis, t, b);
    }
    double scale = len / s->gen_distance;
    int k = 0;
    for (int l = 0; l < s->nl_h; ++l)
        for (int j = 0; j < s->counts_h[l]; ++j, ++k) {
            const double* q = s->pts_h + 3 * k;
            for (int c = 0; c < 3; ++c) {
                double v = t[c] * q[0] + b[c] * q[1];
                v = v + axis[c] * q[2];
                out_pts[3 * k + c] = entry[c] + v * scale;
            }
            out_caps[k] = s->caps_h[l] * scale;
        }
    return 0;
}

static int features_one(const or_scene* s, int kind, const double* p, const double* omega,
                        const double* light, float* out) {
    double lo[3], hi[3];
    grid_bounds(s->nx, s->ny, s->nz, s->vs, s->origin, lo, hi);
    double entry[3];
    or_light_entry_point(lo, hi, p, light, entry);
    int nl = kind == 0 ? s->nl_d : s->nl_h;
    const int* counts = kind == 0 ? s->counts_d : s->counts_h;
    int n = total_points(nl, counts);
    double* pts = (double*)malloc(sizeof(double) * 3 * n);
    double* caps = (double*)malloc(sizeof(double) * n);
    if (kind == 0) {
        int k = 0;
        for (int l = 0; l < nl; ++l)
            for (int j = 0; j < counts[l]; ++j, ++k) {
                for (int c = 0; c < 3; ++c) pts[3 * k + c] = p[c] + s->pts_d[3 * k + c] * s->template_scale;
                caps[k] = s->caps_d[l] * s->template_scale;
            }
    } else if (or_place_highlight(s, p, omega, entry, pts, caps) != 0) {
        free(pts);
        free(caps);
        return -1;
    }
    for (int i = 0; i < n; ++i) {
        const double* x = pts + 3 * i;
        out[i] = (float)or_sample_trilinear(s->density, s->nx, s->ny, s->nz, s->vs, s->origin, x);
        out[n + i] = contains(lo, hi, x)
                         ? (float)or_sample_trilinear(s->tvol, s->nx, s->ny, s->nz, s->vs, s->origin, x)
                         : 1.0f;
        double d[3] = {x[0] - p[0], x[1] - p[1], x[2] - p[2]};
        double dist = len3(d);
        double f;
        if (dist <= 0.0) {
            f = 1.0;
        } else {
            double half = caps[i] >= dist ? OR_PI : asin(caps[i] / dist);
            double il = 1.0 / dist; /* phase_feature: d * (1.0 / len) */
            double axis[3] = {d[0] * il, d[1] * il, d[2] * il};
            f = table_lookup(s, omega, axis, half) * table_lookup(s, light, axis, half);
        }
        out[2 * n + i] = (float)f;
    }
    free(pts);
    free(caps);
    return 0;
}

int or_features(const or_scene* s, int64_t q, const double* centers9, float* out) {
    int nd = total_points(s->nl_d, s->counts_d), nh = total_points(s->nl_h, s->counts_h);
    size_t stride = (size_t)3 * (nd + nh);
    for (int64_t i = 0; i < q; ++i) {
        const double* c = centers9 + 9 * i;
        if (features_one(s, 0, c, c + 3, c + 6, out + stride * i) != 0) return -1;
        if (features_one(s, 1, c, c + 3, c + 6, out + stride * i + 3 * nd) != 0) return -1;
    }
    return 0;
}

/* ---- rng (inc/rng.h:12-66) --------------------------------------------------- */

uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

typedef struct { uint64_t state, inc; } pcg32;

static uint32_t pcg_next(pcg32* r) {
    uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((~rot + 1u) & 31));
}

static void pcg_init(pcg32* r, uint64_t seed, uint64_t seq) {
    r->state = 0;
    r->inc = (or_splitmix64(seq) << 1u) | 1u;
    pcg_next(r);
    r->state += or_splitmix64(seed);
    pcg_next(r);
}

static double pcg_double(pcg32* r) {
    uint64_t hi = pcg_next(r);
    uint64_t lo = pcg_next(r);
    return (double)((hi << 21) ^ (lo >> 11)) * 0x1p-53;
}

/* ---- backbone (src/predictor.cpp:62-148, 153-235, 308-409; src/neural.cpp) ---- */

/* walk_params order (src/predictor.cpp:62-109). Calls fn(rows, cols, fan_in) per
 * tensor; bias tensors report cols = 0 and fan_in = 0. */
typedef void (*walk_fn)(void* ctx, int rows, int cols, int fan_in);

static void walk_params(const or_backbone_cfg* c, walk_fn fn, void* ctx) {
    int W = c->width;
    for (int k = 0; k < 2; ++k) {
        int nl = k == 0 ? c->nl_d : c->nl_h;
        const int* counts = k == 0 ? c->counts_d : c->counts_h;
        for (int t = 0; t < 3; ++t) {
            fn(ctx, W, 7, 7);
            fn(ctx, W, 0, 0);
            for (int i = 0; i < nl; ++i) {
                if (!c->literal) {
                    fn(ctx, 4, 8, 8);
                    fn(ctx, 4, 0, 0);
                    fn(ctx, 3, 4, 4);
                    fn(ctx, 3, 0, 0);
                }
                int ld = counts[i] + 2;
                fn(ctx, W, W + ld, W + ld);
                fn(ctx, W, 0, 0);
                fn(ctx, W, W, W);
                fn(ctx, W, 0, 0);
            }
        }
    }
    int M = c->merge_width;
    for (int t = 0; t < 3; ++t) {
        fn(ctx, M, 2 * W, 2 * W);
        fn(ctx, M, 0, 0);
    }
    fn(ctx, M, 3 * M, 3 * M);
    fn(ctx, M, 0, 0);
    int H = c->head_width;
    int outs[3] = {H, H, 3}, ins[3] = {M, H, H};
    for (int l = 0; l < 3; ++l) {
        fn(ctx, outs[l], ins[l], ins[l]);
        fn(ctx, outs[l], 0, 0);
    }
}

static void count_fn(void* ctx, int rows, int cols, int fan_in) {
    (void)fan_in;
    *(int64_t*)ctx += (int64_t)rows * (cols > 0 ? cols : 1);
}

int64_t or_backbone_param_count(const or_backbone_cfg* cfg) {
    int64_t n = 0;
    walk_params(cfg, count_fn, &n);
    return n;
}

typedef struct { const or_backbone_cfg* cfg; float* out; size_t off; uint64_t ordinal; } init_ctx;

static void init_fn(void* vctx, int rows, int cols, int fan_in) {
    init_ctx* c = (init_ctx*)vctx;
    size_t n = (size_t)rows * (cols > 0 ? cols : 1);
    uint64_t seed = or_splitmix64(c->cfg->seed + 0x5eedu * (c->ordinal + 1));
    if (fan_in > 0) { /* he_uniform, src/neural.cpp:444-452 */
        double bound = sqrt(6.0 / (double)fan_in);
        pcg32 r;
        pcg_init(&r, seed, 0xfeedu);
        for (size_t i = 0; i < n; ++i) c->out[c->off + i] = (float)((2.0 * pcg_double(&r) - 1.0) * bound);
    } else {
        for (size_t i = 0; i < n; ++i) c->out[c->off + i] = 0.0f;
    }
    c->off += n;
    c->ordinal += 1;
}

void or_backbone_init(const or_backbone_cfg* cfg, float* params) {
    init_ctx c = {cfg, params, 0, 0};
    walk_params(cfg, init_fn, &c);
}

/* Tape<float>::dense (src/neural.cpp:86-101): acc = b; acc += w*x, sequential. */
static void dense(const float* W, const float* b, int m, int n, const float* x, float* y) {
    for (int i = 0; i < m; ++i) {
        float acc = b[i];
        const float* row = W + (size_t)i * n;
        for (int j = 0; j < n; ++j) acc += row[j] * x[j];
        y[i] = acc;
    }
}

static float relu(float v) { return (v < 0.0f) ? 0.0f : v; }
static float sigmoidf_(float v) { return 1.0f / (1.0f + expf(-v)); }

static int cmp_desc(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x < y) - (x > y);
}

typedef struct {
    float sorted[3][64];
    float mean[3];
    float max[3];
} layer_slice;

/* src/predictor.cpp:153-191, channel order {density, phase, transmittance} */
static void slice_layers(const float* block, int n_total, int nl, const int* counts,
                         layer_slice* out) {
    const float* ch[3] = {block, block + 2 * n_total, block + n_total};
    int off = 0;
    for (int i = 0; i < nl; ++i) {
        int n = counts[i];
        for (int t = 0; t < 3; ++t) {
            float* dst = out[i].sorted[t];
            memcpy(dst, ch[t] + off, sizeof(float) * n);
            qsort(dst, (size_t)n, sizeof(float), cmp_desc);
            float acc = 0.0f;
            for (int j = 0; j < n; ++j) acc += dst[j];
            out[i].mean[t] = acc / (float)n;
            out[i].max[t] = dst[0];
        }
        off += n;
    }
}

/* Parameter cursor mirroring collect_ids (src/predictor.cpp:111-148). */
typedef struct { const float* p; size_t off; } cursor;
static const float* take(cursor* c, size_t n) { const float* r = c->p + c->off; c->off += n; return r; }

/* run_stack (src/predictor.cpp:206-235) */
static void run_stack(const or_backbone_cfg* cfg, cursor* cur, int tau, const float* cfgv,
                      const layer_slice* L, int nl, const int* counts, float g_mean,
                      float alpha, float* o_out) {
    int W = cfg->width;
    const float* iW = take(cur, (size_t)W * 7);
    const float* ib = take(cur, (size_t)W);
    float o[64], o_att[64], u[64], x[256], t2[64];
    dense(iW, ib, W, 7, cfgv, o);
    for (int j = 0; j < W; ++j) o[j] = relu(o[j]);
    for (int i = 0; i < nl; ++i) {
        float v[8] = {L[i].mean[0], L[i].mean[1], L[i].mean[2], L[i].max[0], L[i].max[1],
                      L[i].max[2], g_mean, alpha};
        float w;
        if (cfg->literal) { /* attention_weight_literal, src/neural.cpp:473-480 */
            float acc = 0.0f;
            for (int j = 0; j < 8; ++j) acc += (v[j] < 0.0f) ? 0.0f : v[j];
            float mean = acc / (float)8.0;
            w = 1.0f / (1.0f + expf(-mean));
        } else { /* attention_weights_learned, src/neural.cpp:482-487 */
            const float* W1 = take(cur, 32);
            const float* b1 = take(cur, 4);
            const float* W2 = take(cur, 12);
            const float* b2 = take(cur, 3);
            float h[4], w3[3];
            dense(W1, b1, 4, 8, v, h);
            for (int j = 0; j < 4; ++j) h[j] = relu(h[j]);
            dense(W2, b2, 3, 4, h, w3);
            for (int j = 0; j < 3; ++j) w3[j] = sigmoidf_(w3[j]);
            w = w3[tau];
        }
        for (int j = 0; j < W; ++j) o_att[j] = o[j] * w;
        int n = counts[i];
        int K = W + n + 2;
        memcpy(x, o_att, sizeof(float) * W);
        memcpy(x + W, L[i].sorted[tau], sizeof(float) * n);
        x[W + n] = L[i].mean[tau];
        x[W + n + 1] = L[i].max[tau];
        const float* f1W = take(cur, (size_t)W * K);
        const float* f1b = take(cur, (size_t)W);
        const float* f2W = take(cur, (size_t)W * W);
        const float* f2b = take(cur, (size_t)W);
        dense(f1W, f1b, W, K, x, u);
        for (int j = 0; j < W; ++j) u[j] = relu(u[j]);
        dense(f2W, f2b, W, W, u, t2);
        for (int j = 0; j < W; ++j) o[j] = relu(t2[j]) + o_att[j];
    }
    memcpy(o_out, o, sizeof(float) * W);
}

/* backbone_forward (src/predictor.cpp:352-387) on one query */
static void forward_one(const or_backbone_cfg* cfg, const float* params, const float* feats,
                        const double* c8, float y[3]) {
    int nd = total_points(cfg->nl_d, cfg->counts_d), nh = total_points(cfg->nl_h, cfg->counts_h);
    layer_slice dl[16], hl[16];
    slice_layers(feats, nd, cfg->nl_d, cfg->counts_d, dl);
    slice_layers(feats + 3 * nd, nh, cfg->nl_h, cfg->counts_h, hl);
    int ng = (int)c8[0];
    float g_mean = 0.0f;
    for (int i = 0; i < ng; ++i) g_mean += (float)c8[1 + i];
    if (ng > 0) g_mean /= (float)(double)ng;
    float alpha = (float)c8[7];
    float cfgv[7] = {0, 0, 0, (float)c8[4], (float)c8[5], (float)c8[6], (float)c8[7]};
    for (int i = 0; i < ng && i < 3; ++i) cfgv[i] = (float)c8[1 + i];

    /* Stack parameter blocks are laid out [kind][tau] in walk order; locate them. */
    int W = cfg->width, M = cfg->merge_width, H = cfg->head_width;
    size_t stack_size[2];
    for (int k = 0; k < 2; ++k) {
        int nl = k == 0 ? cfg->nl_d : cfg->nl_h;
        const int* counts = k == 0 ? cfg->counts_d : cfg->counts_h;
        size_t s = (size_t)W * 7 + W;
        for (int i = 0; i < nl; ++i) {
            if (!cfg->literal) s += 32 + 4 + 12 + 3;
            s += (size_t)W * (W + counts[i] + 2) + W + (size_t)W * W + W;
        }
        stack_size[k] = s;
    }
    size_t merge_off = 3 * (stack_size[0] + stack_size[1]);
    float merged[3][128], od[64], oh[64], cat[512];
    for (int t = 0; t < 3; ++t) {
        cursor cd = {params, (size_t)t * stack_size[0]};
        cursor ch = {params, 3 * stack_size[0] + (size_t)t * stack_size[1]};
        run_stack(cfg, &cd, t, cfgv, dl, cfg->nl_d, cfg->counts_d, g_mean, alpha, od);
        run_stack(cfg, &ch, t, cfgv, hl, cfg->nl_h, cfg->counts_h, g_mean, alpha, oh);
        memcpy(cat, od, sizeof(float) * W);
        memcpy(cat + W, oh, sizeof(float) * W);
        const float* mW = params + merge_off + (size_t)t * ((size_t)M * 2 * W + M);
        dense(mW, mW + (size_t)M * 2 * W, M, 2 * W, cat, merged[t]);
        for (int j = 0; j < M; ++j) merged[t][j] = relu(merged[t][j]);
    }
    size_t off = merge_off + 3 * ((size_t)M * 2 * W + M);
    for (int t = 0; t < 3; ++t) memcpy(cat + t * M, merged[t], sizeof(float) * M);
    float cross[128], h1[128], h2[128];
    dense(params + off, params + off + (size_t)M * 3 * M, M, 3 * M, cat, cross);
    for (int j = 0; j < M; ++j) cross[j] = relu(cross[j]);
    off += (size_t)M * 3 * M + M;
    dense(params + off, params + off + (size_t)H * M, H, M, cross, h1);
    for (int j = 0; j < H; ++j) h1[j] = relu(h1[j]);
    off += (size_t)H * M + H;
    dense(params + off, params + off + (size_t)H * H, H, H, h1, h2);
    for (int j = 0; j < H; ++j) h2[j] = relu(h2[j]);
    off += (size_t)H * H + H;
    dense(params + off, params + off + (size_t)3 * H, 3, H, h2, y);
    for (int j = 0; j < 3; ++j) y[j] = fabsf(y[j]);
}

/* predict_y + decode_prediction (src/predictor.cpp:389-409) */
int or_predict(const or_backbone_cfg* cfg, const float* params, int64_t q, const float* feats,
               const double* cfg8, double* y_out, double* F_out) {
    int nd = total_points(cfg->nl_d, cfg->counts_d), nh = total_points(cfg->nl_h, cfg->counts_h);
    size_t stride = (size_t)3 * (nd + nh);
    for (int64_t i = 0; i < q; ++i) {
        float y[3];
        const double* c8 = cfg8 + 8 * i;
        forward_one(cfg, params, feats + stride * i, c8, y);
        for (int c = 0; c < 3; ++c) {
            double eg = pow(c8[4 + c], cfg->gamma);
            y_out[3 * i + c] = (double)y[c];
            F_out[3 * i + c] = eg * expm1((double)y[c]);
        }
    }
    return 0;
}
