"""Seeded synthetic inputs for the BASELINE.json configurations (harness side).

* ``procedural_cloud`` restates the reference's ``generate_medium(ProceduralCloud)``
  (src/scene_gen.cpp:16-52, 74-109) bit-for-bit in vectorised numpy (C1 input).
* ``fractal_ellipsoid`` (C2), ``smoke_plume`` (C3), ``mixed_medium`` (C4) and
  ``noise_volume`` + ``rotating_light`` (C5) are this repo's generators for the
  configurations the reference has no generator for.
* ``draw_centers`` restates src/feature_pipeline.cpp:174-198 (uniform occupied
  voxel + jitter, omega uniform on S^2) with one PCG32 stream per center.

No public dataset is involved: every input is a seeded synthetic volume.
"""
from __future__ import annotations

import math

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _u64(x):
    return np.asarray(x, dtype=np.uint64)


def splitmix64(x):
    """inc/rng.h:12-17 on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = _u64(x) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


class Pcg32:
    """Vectorised PCG32 (inc/rng.h:22-66): one independent stream per array element."""

    MUL = np.uint64(6364136223846793005)

    def __init__(self, seed, seq):
        seed, seq = np.broadcast_arrays(_u64(seed), _u64(seq))
        self.state = np.zeros(seed.shape, np.uint64)
        self.inc = (splitmix64(seq) << np.uint64(1)) | np.uint64(1)
        self.next_u32()
        with np.errstate(over="ignore"):
            self.state = self.state + splitmix64(seed)
        self.next_u32()

    def next_u32(self):
        old = self.state
        with np.errstate(over="ignore"):
            self.state = old * self.MUL + self.inc
        xs = (((old >> np.uint64(18)) ^ old) >> np.uint64(27)) & np.uint64(0xFFFFFFFF)
        rot = old >> np.uint64(59)
        left = (xs << ((~rot + np.uint64(1)) & np.uint64(31))) & np.uint64(0xFFFFFFFF)
        return ((xs >> rot) | left).astype(np.uint64)

    def next_double(self):
        hi = self.next_u32()
        lo = self.next_u32()
        return ((hi << np.uint64(21)) ^ (lo >> np.uint64(11))).astype(np.float64) * 2.0 ** -53

    def next_below(self, n):
        m = self.next_u32() * _u64(n)
        return (m >> np.uint64(32)).astype(np.int64)

    def next_unit_vector(self):
        z = 1.0 - 2.0 * self.next_double()
        phi = 2.0 * np.pi * self.next_double()
        r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        # libm cos/sin (as the reference's std::cos/std::sin), not numpy's SIMD variants
        return np.stack([r * _libm(math.cos, phi), r * _libm(math.sin, phi), z], axis=-1)


def _libm(fn, a):
    a = np.asarray(a, np.float64)
    return np.fromiter((fn(v) for v in a.reshape(-1)), np.float64, a.size).reshape(a.shape)


def _lattice_value(seed, x, y, z):
    """src/scene_gen.cpp:16-23."""
    with np.errstate(over="ignore"):
        h = _u64(seed)
        h = splitmix64(h ^ (x.astype(np.uint64) * np.uint64(0x8DA6B343)))
        h = splitmix64(h ^ (y.astype(np.uint64) * np.uint64(0xD8163841)))
        h = splitmix64(h ^ (z.astype(np.uint64) * np.uint64(0xCB1AB31F)))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _smooth(t):
    return t * t * (3.0 - 2.0 * t)


def _value_noise(seed, px, py, pz):
    """src/scene_gen.cpp:27-41 (trilinear value noise, smoothstep weights)."""
    fx, fy, fz = np.floor(px), np.floor(py), np.floor(pz)
    ix, iy, iz = fx.astype(np.int64), fy.astype(np.int64), fz.astype(np.int64)
    tx, ty, tz = _smooth(px - fx), _smooth(py - fy), _smooth(pz - fz)
    acc = np.zeros_like(px)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                w = (tx if dx else 1.0 - tx) * (ty if dy else 1.0 - ty) * (tz if dz else 1.0 - tz)
                acc = acc + w * _lattice_value(seed, ix + dx, iy + dy, iz + dz)
    return acc


def _fbm(seed, px, py, pz, octaves):
    """src/scene_gen.cpp:44-56."""
    acc = np.zeros_like(px)
    amp, norm, freq = 1.0, 0.0, 1.0
    for o in range(octaves):
        with np.errstate(over="ignore"):
            s = (np.uint64(seed) + np.uint64(o) * np.uint64(0x9E3779B9)) & M64
        acc = acc + amp * _value_noise(s, px * freq, py * freq, pz * freq)
        norm += amp
        amp *= 0.5
        freq *= 2.0
    return acc / norm


def _unit_coords(dims, z0, z1):
    idx = np.arange(dims, dtype=np.float64)
    u = (idx + 0.5) / dims
    uz, uy, ux = np.meshgrid(u[z0:z1], u, u, indexing="ij")
    return ux, uy, uz


def procedural_cloud(dims, seed, chunk=16):
    """generate_medium(ProceduralCloud, dims, seed) (src/scene_gen.cpp:93-102): [z,y,x] f32."""
    if dims < 2 or dims & (dims - 1):
        raise ValueError("medium dims must be a power of two >= 2")
    out = np.zeros((dims, dims, dims), np.float32)
    for z0 in range(0, dims, chunk):
        z1 = min(dims, z0 + chunk)
        ux, uy, uz = _unit_coords(dims, z0, z1)
        qx, qy, qz = 2.0 * ux - 1.0, 2.0 * uy - 1.0, 2.0 * uz - 1.0
        length = np.sqrt(qx * qx + qy * qy + qz * qz)
        falloff = np.clip(1.3 - 1.5 * length, 0.0, 1.0)
        noise = _fbm(seed, ux * 4.0, uy * 4.0, uz * 4.0, 4)
        out[z0:z1] = np.clip(2.0 * (noise - 0.4) * falloff, 0.0, 1.0).astype(np.float32)
    return out


def fractal_ellipsoid(dims, seed, chunk=16):
    """C2: seeded 6-octave fractal value noise plus a hard-edged ellipsoid, values in [0,1]."""
    out = np.zeros((dims, dims, dims), np.float32)
    for z0 in range(0, dims, chunk):
        z1 = min(dims, z0 + chunk)
        ux, uy, uz = _unit_coords(dims, z0, z1)
        qx, qy, qz = 2.0 * ux - 1.0, 2.0 * uy - 1.0, 2.0 * uz - 1.0
        falloff = np.clip(1.25 - 1.4 * np.sqrt(qx * qx + qy * qy + qz * qz), 0.0, 1.0)
        noise = _fbm(seed, ux * 5.0, uy * 5.0, uz * 5.0, 6)
        cloud = np.clip(2.2 * (noise - 0.38) * falloff, 0.0, 1.0)
        ell = ((qx - 0.15) / 0.45) ** 2 + ((qy + 0.1) / 0.3) ** 2 + ((qz - 0.05) / 0.38) ** 2 <= 1.0
        out[z0:z1] = np.where(ell, np.maximum(cloud, 0.85), cloud).astype(np.float32)
    return out


def draw_centers(grid, count, seed, light, voxel_size=None, origin=(-1.0, -1.0, -1.0)):
    """draw_centers (src/feature_pipeline.cpp:174-198): [count, 9] rows (p, omega, l)."""
    nz, ny, nx = grid.shape
    vs = 2.0 / nx if voxel_size is None else voxel_size
    flat = grid.reshape(-1)
    occupied = np.nonzero(flat > 0.0)[0].astype(np.int64)
    if len(occupied) == 0:
        raise ValueError("draw_centers: medium has no occupied voxel")
    lv = np.asarray(light, np.float64)
    n = np.sqrt(lv[0] * lv[0] + lv[1] * lv[1] + lv[2] * lv[2])
    l = np.array([lv[0] / n, lv[1] / n, lv[2] / n])
    rng = Pcg32(np.uint64(seed), np.arange(count, dtype=np.uint64) + np.uint64(1000))
    vidx = occupied[rng.next_below(len(occupied))]
    x = vidx % nx
    y = (vidx // nx) % ny
    z = vidx // (nx * ny)
    jx, jy, jz = rng.next_double(), rng.next_double(), rng.next_double()
    p = np.stack([origin[0] + (x + jx) * vs, origin[1] + (y + jy) * vs, origin[2] + (z + jz) * vs], axis=-1)
    omega = rng.next_unit_vector()
    return np.concatenate([p, omega, np.broadcast_to(l, (count, 3))], axis=1)


def config_rows(centers, g, albedo):
    """ConfigParams rows built directly (C1/C2 bypass make_config's class check):
    n_g, g0..g2, albedo.xyz, alpha = angle_between(omega, l) (inc/math.h:53-56)."""
    w, l = centers[:, 3:6], centers[:, 6:9]
    dot = w[:, 0] * l[:, 0] + w[:, 1] * l[:, 1] + w[:, 2] * l[:, 2]
    ww = w[:, 0] * w[:, 0] + w[:, 1] * w[:, 1] + w[:, 2] * w[:, 2]
    ll = l[:, 0] * l[:, 0] + l[:, 1] * l[:, 1] + l[:, 2] * l[:, 2]
    alpha = _libm(math.acos, np.clip(dot / np.sqrt(ww * ll), -1.0, 1.0))
    g = list(g)
    rows = np.zeros((len(centers), 8))
    rows[:, 0] = len(g)
    rows[:, 1:1 + len(g)] = g
    rows[:, 4:7] = albedo
    rows[:, 7] = alpha
    return rows


LIGHT = (0.2, -1.0, 0.1)


def _box_blur(v, r, axis):
    """Separable box filter of radius r along one axis (edge-clamped), float64."""
    n = v.shape[axis]
    pad = [(0, 0)] * v.ndim
    pad[axis] = (r + 1, r)
    c = np.cumsum(np.pad(v, pad, mode="edge"), axis=axis)
    hi = np.take(c, np.arange(2 * r + 1, 2 * r + 1 + n), axis=axis)
    lo = np.take(c, np.arange(0, n), axis=axis)
    return (hi - lo) / (2 * r + 1)


def _curl_velocity(seed, n=24):
    """Divergence-free velocity on an n^3 lattice over [0,1]^3: curl of a 3-component
    value-noise potential (central differences), for the C3 plume advection."""
    u = (np.arange(n) + 0.5) / n
    uz, uy, ux = np.meshgrid(u, u, u, indexing="ij")
    psi = [_fbm((seed + 101 * (k + 1)) & 0xFFFFFFFF, ux * 3.0, uy * 3.0, uz * 3.0, 3) for k in range(3)]
    d = lambda f, ax: np.gradient(f, 1.0 / n, axis=ax)  # noqa: E731 (axis 0 = z, 1 = y, 2 = x)
    vx = d(psi[2], 1) - d(psi[1], 0)
    vy = d(psi[0], 0) - d(psi[2], 2)
    vz = d(psi[1], 2) - d(psi[0], 1)
    return np.stack([vx, vy, vz], axis=-1)


def _lattice_lookup(field, p):
    """Nearest-cell lookup of an [n,n,n,3] lattice field at points p in [0,1)^3."""
    n = field.shape[0]
    i = np.clip((p * n).astype(np.int64), 0, n - 1)
    return field[i[:, 2], i[:, 1], i[:, 0]]


def smoke_plume(dims, seed, particles=None, steps=24, empty=0.70):
    """C3: seeded curl-noise-advected smoke blob, [z,y,x] f32 in [0,1], with ``empty``
    (default 70%) of the voxels exactly zero. Particles are emitted from a Gaussian source
    near the bottom, rise with buoyancy while a curl-noise field advects them, are splatted
    into the grid, box-blurred, and the lowest 70% of voxels are cut to zero."""
    rng = np.random.default_rng(seed)
    npart = particles or max(20000, dims ** 3 // 8)
    p = rng.normal([0.5, 0.2, 0.5], [0.06, 0.04, 0.06], size=(npart, 3))
    birth = rng.uniform(0.0, 1.0, npart)
    vel = _curl_velocity(seed)
    dt = 0.7 / steps
    for k in range(steps):
        live = birth <= (k + 1) / steps
        v = _lattice_lookup(vel, np.clip(p, 0.0, 0.999999)) * 0.6
        v[:, 1] += 1.0  # buoyancy (+y)
        p[live] += dt * v[live]
    p = p[np.all((p >= 0.0) & (p < 1.0), axis=1)]
    idx = (p * dims).astype(np.int64)
    vol = np.zeros((dims, dims, dims), np.float64)
    np.add.at(vol, (idx[:, 2], idx[:, 1], idx[:, 0]), 1.0)
    r = max(1, dims // 16)
    for ax in range(3):
        vol = _box_blur(vol, r, ax)
    cut = np.quantile(vol, empty)
    vol = np.where(vol > cut, vol - cut, 0.0)
    vol /= max(vol.max(), 1e-30)
    return np.clip(vol, 0.0, 1.0).astype(np.float32)


def mixed_medium(dims, seed, chunk=16):
    """C4: seeded noise density in [0,1] with per-voxel albedo in [0.9, 0.999] and per-voxel HG
    g in [0.3, 0.9]; returns (density, albedo, g), each [z,y,x] f32."""
    dens = np.zeros((dims, dims, dims), np.float32)
    alb = np.zeros_like(dens)
    gg = np.zeros_like(dens)
    for z0 in range(0, dims, chunk):
        z1 = min(dims, z0 + chunk)
        ux, uy, uz = _unit_coords(dims, z0, z1)
        qx, qy, qz = 2.0 * ux - 1.0, 2.0 * uy - 1.0, 2.0 * uz - 1.0
        falloff = np.clip(1.3 - 1.5 * np.sqrt(qx * qx + qy * qy + qz * qz), 0.0, 1.0)
        dens[z0:z1] = np.clip(2.0 * (_fbm(seed, ux * 4.0, uy * 4.0, uz * 4.0, 4) - 0.4) * falloff, 0.0, 1.0)
        alb[z0:z1] = 0.9 + 0.099 * _fbm((seed + 7) & 0xFFFFFFFF, ux * 2.0, uy * 2.0, uz * 2.0, 2)
        gg[z0:z1] = 0.3 + 0.6 * _fbm((seed + 13) & 0xFFFFFFFF, ux * 2.0, uy * 2.0, uz * 2.0, 2)
    return dens, alb, gg


def mixed_medium_large(dims, seed, base=128):
    """C4 at 512^3: mixed_medium generated at `base`^3 (the noise's finest octave spans 16
    voxels at 512^3, so nothing is lost) and trilinearly upsampled to dims^3, float32."""
    if dims <= base:
        return mixed_medium(dims, seed)
    from scipy.ndimage import zoom
    f = dims / base
    return tuple(np.clip(zoom(a, f, order=1, mode="nearest", grid_mode=True), lo, hi).astype(np.float32)
                 for a, (lo, hi) in zip(mixed_medium(base, seed), ((0.0, 1.0), (0.9, 0.999), (0.3, 0.9))))


def sample_media(albedo, g, centers, voxel_size=None, origin=(-1.0, -1.0, -1.0)):
    """Per-query medium rows [n, 4] = (g, albedo rgb) for C4: FP64 trilinear of the per-voxel
    g / albedo grids at each query's p (DensityGrid::sample_trilinear semantics, clamp-to-edge
    cell; queries lie inside the grid). Grey albedo (r = g = b)."""
    nz, ny, nx = g.shape
    vs = 2.0 / nx if voxel_size is None else voxel_size
    f = (centers[:, :3] - np.asarray(origin)) / vs - 0.5
    i0 = np.floor(f).astype(np.int64)
    t = f - i0
    dims = np.array([nx, ny, nz])
    out = []
    for grid in (g, albedo):
        acc = np.zeros(len(centers))
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    d = np.array([dx, dy, dz])
                    ii = np.clip(i0 + d, 0, dims - 1)
                    w = np.prod(np.where(d == 1, t, 1.0 - t), axis=1)
                    acc += w * grid[ii[:, 2], ii[:, 1], ii[:, 0]].astype(np.float64)
        out.append(acc)
    gq, aq = out
    return np.stack([gq, aq, aq, aq], axis=1)


def noise_volume(dims, seed, chunk=16):
    """C5: seeded 5-octave value-noise volume in [0,1] (static across the sequence)."""
    out = np.zeros((dims, dims, dims), np.float32)
    for z0 in range(0, dims, chunk):
        z1 = min(dims, z0 + chunk)
        ux, uy, uz = _unit_coords(dims, z0, z1)
        qx, qy, qz = 2.0 * ux - 1.0, 2.0 * uy - 1.0, 2.0 * uz - 1.0
        falloff = np.clip(1.2 - 1.3 * np.sqrt(qx * qx + qy * qy + qz * qz), 0.0, 1.0)
        out[z0:z1] = np.clip(2.0 * (_fbm(seed, ux * 4.0, uy * 4.0, uz * 4.0, 5) - 0.42) * falloff, 0.0, 1.0)
    return out


def rotating_light(frame, n_frames, base=LIGHT):
    """C5: LIGHT rotated by 360 deg * frame / n_frames about +Y (normalised)."""
    a = 2.0 * math.pi * frame / n_frames
    x, y, z = base
    c, s_ = math.cos(a), math.sin(a)
    v = (c * x + s_ * z, y, -s_ * x + c * z)
    n = math.sqrt(sum(t * t for t in v))
    return tuple(t / n for t in v)


def c3_lights():
    """C3: four directional lights (LIGHT plus three rotated about Y) with intensities."""
    return [rotating_light(k, 4) for k in range(4)], [1.0, 0.6, 0.4, 0.3]
