"""Multi-light (C3), per-query medium (C4) and animated (C5) drivers over the hot path.

The reference handles one light and one scene-wide medium per call; these
configurations compose its own entry points:

* C3 — several directional lights: one transmittance feature volume per light (rebuilt per
  light), the same shading points (p, omega) queried against each, and the builder's
  extension F = sum_l I_l * F_l.
* C4 — per-voxel albedo / g: the caller samples them at p (scenes.sample_media) and each
  query runs with PhaseModel::hg(g) and ConfigParams{g, albedo} (sf_query_media).
* C5 — a static volume under a light rotating about +Y: the pyramid is built once, the
  transmittance volume every frame, then the frame's queries; per-stage device times.

Every function takes and returns host numpy arrays unless CUDA tensors are passed in.
"""
from __future__ import annotations

import numpy as np

from . import api, scenes


def with_light(rows, light):
    """Query rows (p, omega, l) with l replaced by the normalised `light`."""
    out = np.array(rows, np.float64, copy=True)
    lv = np.asarray(light, np.float64)
    out[:, 6:9] = lv / np.sqrt(np.dot(lv, lv))
    return out


def multi_light_query(grid, pyramid, lights, intensities, rows, dt, ht, model, table, medium, net,
                      precision=api.FP32, weights=None, cfg=None, template_scale=1.0):
    """C3: F = sum_l I_l F_l over `lights`; returns (F [n,3], [F_l]). One scene: its
    transmittance volume is rebuilt in place for each light (Scene.relight: no per-light
    allocation or host synchronisation) before that light's queries."""
    total = np.zeros((len(rows), 3))
    per = []
    scene = None
    for light, inten in zip(lights, intensities):
        if scene is None:
            tvol = api.build_transmittance_volume(pyramid, light, weights, cfg)
            scene = api.Scene(grid, tvol, dt, ht, model, table, template_scale)
        else:
            scene.relight(pyramid, light, weights, cfg)
        F = api.query(scene, net, medium, with_light(rows, light), precision)
        per.append(F)
        total += inten * F
    return total, per


def animated_sequence(grid, n_frames, rows, dt, ht, model, table, medium, net, precision=api.BF16,
                      frames=None, stream=None, timer=None):
    """C5: for each frame f, light = scenes.rotating_light(f, n_frames); rebuild the
    transmittance volume from the (static) pyramid and run the frame's queries.

    `timer(name)` (optional) is called around stages for per-stage device timing; returns
    the list of per-frame F."""
    pyramid = api.DensityPyramid(grid, stream=stream)
    out = []
    scene = None
    for f in (range(n_frames) if frames is None else frames):
        light = scenes.rotating_light(f, n_frames)
        if timer:
            timer("transmittance")
        if scene is None:  # the first frame's volume makes the scene; later frames rebuild it in place
            tvol = api.build_transmittance_volume(pyramid, light, stream=stream)
            scene = api.Scene(grid, tvol, dt, ht, model, table)
        else:
            scene.relight(pyramid, light, stream=stream)
        if timer:
            timer("query")
        out.append(api.query(scene, net, medium, with_light(rows, light), precision, stream=stream))
        if timer:
            timer("end")
    return out
