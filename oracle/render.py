"""Oracle (test infrastructure only): numpy restatement of the image entry point around the
query — Camera::primary_ray, bake_field and render_volume — for small images.

  Camera::Camera / primary_ray : src/camera.cpp:12-31
  bake_field                   : src/predictor.cpp:559-581 (F at occupied voxel centres,
                                 omega = normalize(p - camera), stored float)
  render_volume                : src/rte.cpp:407-447 (closed-box slab test, midpoint march,
                                 second-order attenuation, background)
  BakedField::sample           : src/predictor.cpp:549-556 (trilinear per channel, 0 outside)

F at the voxel centres comes from the C restatement (oracle/sf_oracle.c features + predict),
pinned against the reference; the whole composition is pinned against the reference's own
render_neural output (tests/golden/render.npz, tests/test_oracle.py). Pure-Python loops:
small images only. Never imported by the product path.
"""
from __future__ import annotations

import math

import numpy as np


def _norm(v):
    v = np.asarray(v, np.float64)
    return v / math.sqrt(float(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]))


def _cross(a, b):
    return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])


class Camera:
    def __init__(self, position, look_at, up, vfov, width, height):
        self.position = np.asarray(position, np.float64)
        self.forward = _norm(np.asarray(look_at, np.float64) - self.position)
        self.right = _norm(_cross(self.forward, np.asarray(up, np.float64)))
        self.up = _cross(self.right, self.forward)
        self.tan_half = math.tan(0.5 * vfov * math.pi / 180.0)
        self.aspect = float(width) / float(height)
        self.width, self.height = width, height

    def primary_ray(self, px, py):
        sx = (2.0 * ((px + 0.5) / self.width) - 1.0) * self.aspect * self.tan_half
        sy = (1.0 - 2.0 * ((py + 0.5) / self.height)) * self.tan_half
        return self.position, _norm(self.forward + sx * self.right + sy * self.up)


def trilinear(grid, vs, origin, p):
    """DensityGrid::sample_trilinear (src/volume_grid.cpp:40-62)."""
    nz, ny, nx = grid.shape
    lo = np.asarray(origin, np.float64)
    hi = lo + np.array([nx, ny, nz]) * vs
    if np.any(p < lo) or np.any(p > hi):
        return 0.0
    f = (p - lo) / vs - 0.5
    i0 = np.floor(f).astype(int)
    t = f - i0
    n = np.array([nx, ny, nz])
    a = np.clip(i0, 0, n - 1)
    b = np.clip(i0 + 1, 0, n - 1)
    v = lambda x, y, z: float(grid[z, y, x])  # noqa: E731
    lerp = lambda u, w, s: u + s * (w - u)  # noqa: E731
    c00 = lerp(v(a[0], a[1], a[2]), v(b[0], a[1], a[2]), t[0])
    c10 = lerp(v(a[0], b[1], a[2]), v(b[0], b[1], a[2]), t[0])
    c01 = lerp(v(a[0], a[1], b[2]), v(b[0], a[1], b[2]), t[0])
    c11 = lerp(v(a[0], b[1], b[2]), v(b[0], b[1], b[2]), t[0])
    return lerp(lerp(c00, c10, t[1]), lerp(c01, c11, t[1]), t[2])


def intersect_box(lo, hi, o, d):
    """inc/math.h:85-107."""
    t0, t1 = -1e300, 1e300
    for i in range(3):
        if d[i] == 0.0:
            if o[i] < lo[i] or o[i] > hi[i]:
                return None
            continue
        inv = 1.0 / d[i]
        ta, tb = (lo[i] - o[i]) * inv, (hi[i] - o[i]) * inv
        if ta > tb:
            ta, tb = tb, ta
        t0 = ta if t0 < ta else t0
        t1 = tb if tb < t1 else t1
        if t0 > t1:
            return None
    return t0, t1


def bake_rows(grid, vs, origin, camera_pos, light):
    """bake_field's query rows: (voxel index, p, omega, l) per occupied voxel."""
    nz, ny, nx = grid.shape
    o = np.asarray(origin, np.float64)
    idx = np.nonzero(grid.reshape(-1) > 0.0)[0]
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    p = np.stack([o[0] + (x + 0.5) * vs, o[1] + (y + 0.5) * vs, o[2] + (z + 0.5) * vs], axis=1)
    d = p - np.asarray(camera_pos, np.float64)
    w = d / np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])[:, None]
    rows = np.concatenate([p, w, np.broadcast_to(np.asarray(light, np.float64), (len(idx), 3))], axis=1)
    return idx, rows


def field_from(grid, idx, F):
    """BakedField grids [3, nz, ny, nx]: float(F) at the occupied voxels, 0 elsewhere."""
    out = np.zeros((3,) + grid.shape, np.float32)
    for c in range(3):
        out[c].reshape(-1)[idx] = F[:, c].astype(np.float32)
    return out


def render_volume(grid, vs, origin, sigma_t, albedo, cam: Camera, field, step_scale=0.5, background=(0, 0, 0)):
    nz, ny, nx = grid.shape
    lo = np.asarray(origin, np.float64)
    hi = lo + np.array([nx, ny, nz]) * vs
    step = step_scale * vs
    img = np.zeros((cam.height, cam.width, 3), np.float32)
    mu, alb, bg = (np.asarray(a, np.float64) for a in (sigma_t, albedo, background))
    for py in range(cam.height):
        for px in range(cam.width):
            o, d = cam.primary_ray(px, py)
            L = np.zeros(3)
            T = np.ones(3)
            hit = intersect_box(lo, hi, o, d)
            if hit is not None and hit[1] > 0.0:
                t0, t1 = max(hit[0], 0.0), hit[1]
                n = max(1, int(math.ceil((t1 - t0) / step)))
                h = (t1 - t0) / n
                for k in range(n):
                    x = o + d * (t0 + (k + 0.5) * h)
                    rho = trilinear(grid, vs, origin, x)
                    if rho > 0.0:
                        st = mu * rho
                        ss = alb * st
                        F = np.array([trilinear(field[c], vs, origin, x) for c in range(3)]) if field is not None \
                            else np.zeros(3)
                        tmid = T * np.exp(-0.5 * h * st)
                        L += tmid * ss * F * h
                        T = T * np.exp(-h * st)
            img[py, px] = (L + T * bg).astype(np.float32)
    return img
