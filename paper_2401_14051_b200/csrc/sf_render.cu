// sf_render.cu — the image entry point around the query: bake_field (src/predictor.cpp:
// 549-581) and render_volume (src/rte.cpp:407-447), the two loops render_neural
// (src/predictor.cpp:585-614) runs around the per-shading-point query.
//
// Bake: the occupied voxels (density > 0) are compacted on the device (ordered, k_occ_*), one
// query row (p = voxel centre, omega = normalize(p - camera), l) is written per voxel,
// the fused query runs over the rows, and F is scattered into three float grids (zero
// elsewhere). Render: one thread per pixel marches the camera ray through the box in
// FP64 with the reference's operation order (second-order midpoint attenuation), the
// in-scatter provider being the FP64 trilinear of the baked grids.

#include "sf_internal.h"

namespace sfb {

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(size_t n, int block = kBlock) {
    size_t g = (n + block - 1) / block;
    return unsigned(g > 0x7fffffff ? 0x7fffffff : (g == 0 ? 1 : g));
}

// Ordered compaction of the occupied voxels (density > 0) into their indices: per-block counts,
// a two-level exclusive scan of the counts, then every block writes its voxels in order.
constexpr int kOccBlock = 1024;

__global__ void __launch_bounds__(kOccBlock) k_occ_count(const float* __restrict__ v, int n, int* __restrict__ cnts) {
    const int i = blockIdx.x * kOccBlock + threadIdx.x;
    const int c = __syncthreads_count(i < n && v[i] > 0.0f);
    if (threadIdx.x == 0) cnts[blockIdx.x] = c;
}

// In-place exclusive scan of cnts[0, m) in tiles of 1024; tile totals to tsum[]
__global__ void __launch_bounds__(1024) k_occ_tile_scan(int* __restrict__ cnts, int m, int* __restrict__ tsum) {
    __shared__ int ws[32];
    const int i = blockIdx.x * 1024 + threadIdx.x;
    int total;
    const int ex = block_exclusive_scan(i < m ? cnts[i] : 0, ws, total);
    if (i < m) cnts[i] = ex;
    if (threadIdx.x == 0) tsum[blockIdx.x] = total;
}

// Exclusive scan of the tile totals (at most 1024 tiles); the grand total -> *count
__global__ void __launch_bounds__(1024) k_occ_sum_scan(int* __restrict__ tsum, int tiles, int* __restrict__ count) {
    __shared__ int ws[32];
    int total;
    const int ex = block_exclusive_scan(int(threadIdx.x) < tiles ? tsum[threadIdx.x] : 0, ws, total);
    if (int(threadIdx.x) < tiles) tsum[threadIdx.x] = ex;
    if (threadIdx.x == 0) *count = total;
}

__global__ void __launch_bounds__(kOccBlock) k_occ_write(const float* __restrict__ v, int n, const int* __restrict__ cnts,
                                                       const int* __restrict__ tsum, int* __restrict__ idx) {
    __shared__ int ws[32];
    const int i = blockIdx.x * kOccBlock + threadIdx.x;
    const bool occ = i < n && v[i] > 0.0f;
    int total;
    const int ex = block_exclusive_scan(occ ? 1 : 0, ws, total);
    if (occ) idx[cnts[blockIdx.x] + tsum[blockIdx.x >> 10] + ex] = i;
}

// One query row per occupied voxel (bake_field's body, src/predictor.cpp:566-575).
__global__ void k_bake_rows(GridDev g, const int* __restrict__ idx, const int* __restrict__ count, double cx,
                            double cy, double cz, double lx, double ly, double lz, double* __restrict__ rows) {
    const int m = *count;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
        const int i = idx[k];
        const int x = i % g.nx, y = (i / g.nx) % g.ny, z = i / (g.nx * g.ny);
        // grid.origin() + Vec3{(x + 0.5) * vs, (y + 0.5) * vs, (z + 0.5) * vs}
        const double p[3] = {g.ox + (x + 0.5) * g.vs, g.oy + (y + 0.5) * g.vs, g.oz + (z + 0.5) * g.vs};
        double d[3] = {p[0] - cx, p[1] - cy, p[2] - cz};
        const double len = sqrt(dot3(d, d));  // normalize(p - camera.position()) = v / length(v)
        double* r = rows + 9 * size_t(k);
        r[0] = p[0];
        r[1] = p[1];
        r[2] = p[2];
        r[3] = d[0] / len;
        r[4] = d[1] / len;
        r[5] = d[2] / len;
        r[6] = lx;
        r[7] = ly;
        r[8] = lz;
    }
}

// field.{r,g,b}.set(x, y, z, float(F.{x,y,z}))
__global__ void k_scatter_field(const int* __restrict__ idx, const int* __restrict__ count, size_t plane,
                                const double* __restrict__ F, float* __restrict__ out) {
    const int m = *count;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
        const size_t i = size_t(idx[k]);
        out[i] = float(F[3 * size_t(k)]);
        out[plane + i] = float(F[3 * size_t(k) + 1]);
        out[2 * plane + i] = float(F[3 * size_t(k) + 2]);
    }
}

struct RenderArgs {
    GridDev density;
    const float* field;  // [3][nz][ny][nx] baked F, or null (F = 0)
    double mu[3], albedo[3], bg[3];
    double pos[3], fwd[3], right[3], up[3];
    double tan_half, aspect;
    int width, height;
    double step;
};

// render_volume (src/rte.cpp:407-447) for pixel (px, py): camera.primary_ray(px, py)
// (src/camera.cpp:26-31, dx = dy = 0.5), closed-box slab test, midpoint march.
__global__ void k_render(RenderArgs a, float* __restrict__ img) {
    const int n_px = a.width * a.height;
    const double lo[3] = {a.density.ox, a.density.oy, a.density.oz};
    const double hi[3] = {a.density.hx, a.density.hy, a.density.hz};
    const size_t plane = size_t(a.density.nx) * a.density.ny * a.density.nz;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_px; idx += gridDim.x * blockDim.x) {
        const int px = idx % a.width, py = idx / a.width;
        const double sx = (2.0 * ((px + 0.5) / a.width) - 1.0) * a.aspect * a.tan_half;
        const double sy = (1.0 - 2.0 * ((py + 0.5) / a.height)) * a.tan_half;
        double dir[3];
        for (int c = 0; c < 3; ++c) dir[c] = a.fwd[c] + sx * a.right[c] + sy * a.up[c];
        const double dl = sqrt(dot3(dir, dir));
        for (int c = 0; c < 3; ++c) dir[c] = dir[c] / dl;
        double L[3] = {0.0, 0.0, 0.0}, T[3] = {1.0, 1.0, 1.0};
        double t0, t1;
        if (intersect_box(lo, hi, a.pos, dir, t0, t1) && t1 > 0.0) {
            t0 = t0 > 0.0 ? t0 : 0.0;  // std::max(t0, 0.0)
            int n = int(ceil((t1 - t0) / a.step));
            n = n > 1 ? n : 1;
            const double h = (t1 - t0) / n;
            for (int k = 0; k < n; ++k) {
                const double s = t0 + (k + 0.5) * h;
                const double x = a.pos[0] + dir[0] * s, y = a.pos[1] + dir[1] * s, z = a.pos[2] + dir[2] * s;
                const double rho = trilinear(a.density, x, y, z);
                if (rho > 0.0) {
                    double F[3] = {0.0, 0.0, 0.0};
                    if (a.field) {  // BakedField::sample: trilinear of each channel grid
                        GridDev fg = a.density;
                        for (int c = 0; c < 3; ++c) {
                            fg.v = a.field + c * plane;
                            F[c] = trilinear(fg, x, y, z);
                        }
                    }
                    for (int c = 0; c < 3; ++c) {
                        const double st = a.mu[c] * rho;  // sigma_t = mu_t_scale * rho
                        const double ss = a.albedo[c] * st;  // sigma_s = albedo * sigma_t
                        const double tmid = T[c] * exp(-0.5 * h * st);
                        L[c] += tmid * ss * F[c] * h;
                        T[c] = T[c] * exp(-h * st);
                    }
                }
            }
        }
        float* o = img + 3 * size_t(idx);
        for (int c = 0; c < 3; ++c) o[c] = float(L[c] + T[c] * a.bg[c]);
    }
}

void normalize_h(double* v) {
    const double l = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int c = 0; c < 3; ++c) v[c] = v[c] / l;
}

void cross_h(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

int64_t launch_occupied(const sf_grid& g, int* idx, int* count, void* tmp, size_t& tmp_bytes, cudaStream_t s) {
    const size_t n64 = g.count();
    if (n64 >= (size_t(1) << 30)) fail(SF_ERR_BAD_DIMS, "occupied voxels: grid too large");
    const int n = int(n64), nb = (n + kOccBlock - 1) / kOccBlock, tiles = (nb + 1023) / 1024;
    if (!tmp) {  // size query: block counts + tile totals
        tmp_bytes = (size_t(nb) + 1024) * sizeof(int);
        return 0;
    }
    int* cnts = static_cast<int*>(tmp);
    int* tsum = cnts + nb;
    if (n == 0) {
        SFB_CUDA(cudaMemsetAsync(count, 0, sizeof(int), s));
        return 0;
    }
    k_occ_count<<<nb, kOccBlock, 0, s>>>(g.d, n, cnts);
    k_occ_tile_scan<<<tiles, 1024, 0, s>>>(cnts, nb, tsum);
    k_occ_sum_scan<<<1, 1024, 0, s>>>(tsum, tiles, count);
    k_occ_write<<<nb, kOccBlock, 0, s>>>(g.d, n, cnts, tsum, idx);
    SFB_CUDA(cudaGetLastError());
    for (int k = 0; k < 4; ++k) count_launch();
    return 0;
}

void launch_bake_rows(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double cam[3],
                      const double light[3], double* rows, cudaStream_t s) {
    k_bake_rows<<<grid_for(size_t(max_rows)), kBlock, 0, s>>>(g.dev(), idx, count, cam[0], cam[1], cam[2], light[0],
                                                               light[1], light[2], rows);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_scatter_field(const sf_grid& g, const int* idx, const int* count, int64_t max_rows, const double* F,
                          float* out, cudaStream_t s) {
    k_scatter_field<<<grid_for(size_t(max_rows)), kBlock, 0, s>>>(idx, count, g.count(), F, out);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

void launch_render(const sf_grid& density, const float* field, const double mu[3], const double albedo[3],
                   const double pos[3], const double look_at[3], const double up[3], double vfov_deg, int width,
                   int height, double step_scale, const double bg[3], float* img, cudaStream_t s) {
    RenderArgs a{};
    a.density = density.dev();
    a.field = field;
    for (int c = 0; c < 3; ++c) {
        a.mu[c] = mu[c];
        a.albedo[c] = albedo[c];
        a.bg[c] = bg[c];
        a.pos[c] = pos[c];
    }
    // Camera::Camera (src/camera.cpp:12-24)
    for (int c = 0; c < 3; ++c) a.fwd[c] = look_at[c] - pos[c];
    normalize_h(a.fwd);
    cross_h(a.fwd, up, a.right);
    normalize_h(a.right);
    cross_h(a.right, a.fwd, a.up);
    a.tan_half = std::tan(0.5 * vfov_deg * kPi / 180.0);
    a.aspect = double(width) / double(height);
    a.width = width;
    a.height = height;
    a.step = step_scale * density.vs;  // opts.step_scale * medium.grid.voxel_size()
    k_render<<<grid_for(size_t(width) * height, 128), 128, 0, s>>>(a, img);
    SFB_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace sfb
