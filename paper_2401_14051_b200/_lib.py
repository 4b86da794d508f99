"""ctypes binding of libsf_b200.so (the C ABI in include/scatterfield_b200.h).

There is no fallback: if the CUDA library is missing or fails to load, importing
the package raises. Array arguments accept numpy arrays (host) or torch tensors
(host or CUDA); device tensors are passed as device pointers (zero copy).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SF_B200_LIB", os.path.join(HERE, "libsf_b200.so"))

ERRC = {
    1: "io", 2: "malformed_header", 3: "bad_dims", 4: "bad_value", 5: "truncated",
    6: "invalid_argument", 7: "shape_mismatch", 8: "provenance_mismatch", 9: "numeric", 100: "cuda",
}


class ScatterfieldError(RuntimeError):
    """Mirror of scatterfield::Error (inc/error.h:23-32): carries the Errc name."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRC.get(code, code)}] {msg}")
        self.code = code
        self.errc = ERRC.get(code, str(code))


class SfPhaseModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_lobes", C.c_int), ("weight", C.c_double * 3), ("g", C.c_double * 3)]


class SfBackboneConfig(C.Structure):
    _fields_ = [
        ("n_diffuse_layers", C.c_int), ("diffuse_counts", C.c_int * 16),
        ("n_highlight_layers", C.c_int), ("highlight_counts", C.c_int * 16),
        ("width", C.c_int), ("merge_width", C.c_int), ("head_width", C.c_int),
        ("gamma", C.c_double), ("seed", C.c_uint64), ("literal_attention", C.c_int),
    ]


class SfMediumParams(C.Structure):
    _fields_ = [("n_g", C.c_int), ("g", C.c_double * 3), ("albedo", C.c_double * 3)]


P = C.c_void_p
I, I64, D, U64 = C.c_int, C.c_int64, C.c_double, C.c_uint64
PP = C.POINTER(C.c_void_p)

_SIGS = {
    "sf_last_error": (C.c_char_p, []),
    "sf_version": (C.c_char_p, []),
    "sf_device_count": (I, []),
    "sf_grid_create": (I, [I, I, I, D, P, P, PP]),
    "sf_grid_info": (I, [P, P, P, P]),
    "sf_grid_device_ptr": (P, [P]),
    "sf_grid_download": (I, [P, P, P]),
    "sf_grid_destroy": (None, [P]),
    "sf_grid_sample_trilinear": (I, [P, I64, P, P, P]),
    "sf_pyramid_build": (I, [P, PP, P]),
    "sf_pyramid_level_count": (I, [P]),
    "sf_pyramid_level": (P, [P, I]),
    "sf_pyramid_destroy": (None, [P]),
    "sf_graded_transmittance": (I, [P, I, P, D, D, PP, P]),
    "sf_conv3_replicate": (I, [P, P, PP, P]),
    "sf_combine_transmittance": (I, [P, I, P, P, P, PP, P]),
    "sf_build_transmittance_volume": (I, [P, P, P, P, D, D, PP, P]),
    "sf_build_transmittance_slab": (I, [P, P, P, P, D, D, I, I, I, P, P]),
    "sf_build_transmittance_volume_ex": (I, [P, P, P, P, D, D, I, PP, P]),
    "sf_tvol_from_values": (I, [I, I, I, D, P, P, P, PP]),
    "sf_tvol_values": (P, [P]),
    "sf_tvol_destroy": (None, [P]),
    "sf_light_entry_point": (I, [P, P, P, P, P]),
    "sf_phase_table_build": (I, [I, I, I, I, PP, P]),
    "sf_phase_table_from_values": (I, [I, I, I, P, PP]),
    "sf_phase_table_info": (I, [P, P]),
    "sf_phase_table_download": (I, [P, P, P]),
    "sf_phase_table_lookup_hg": (I, [P, I64, P, P, P, P, P]),
    "sf_phase_table_destroy": (None, [P]),
    "sf_template_create": (I, [I, I, P, P, P, D, D, PP]),
    "sf_template_total_points": (I, [P]),
    "sf_place_template": (I, [P, I64, P, P, P, D, P, P, P]),
    "sf_template_destroy": (None, [P]),
    "sf_sample_features": (I, [P, P, P, P, P, D, I64, P, P, P]),
    "sf_backbone_create": (I, [P, P, PP]),
    "sf_backbone_param_count": (I64, [P]),
    "sf_backbone_download_params": (I, [P, P, P]),
    "sf_backbone_destroy": (None, [P]),
    "sf_predict": (I, [P, I64, P, P, I, P, P, P]),
    "sf_scene_create": (I, [P, P, P, P, P, P, D, PP]),
    "sf_scene_destroy": (None, [P]),
    "sf_scene_relight": (I, [P, P, P, P, P, D, D, I, P]),
    "sf_scene_tvol_storage": (I, [P, PP]),
    "sf_scene_commit_tvol": (I, [P, P, P]),
    "sf_debug_query_pools": (I, [P, P, P, I64, P, P, P]),
    "sf_query": (I, [P, P, P, I64, P, I, P, P, P]),
    "sf_query_media": (I, [P, P, I64, P, P, I, P, P, P]),
    "sf_bake_field": (I, [P, P, P, P, I, P, P]),
    "sf_render_volume": (I, [P, P, P, I, P, P, P, D, I, I, P, D, P, P, P]),
    "sf_profile_enable": (I, [I]),
    "sf_profile_read": (I, [P, P]),
    "sf_launch_count": (I64, []),
    "sf_host_alloc": (I, [C.c_size_t, PP]),
    "sf_host_free": (I, [P]),
    "sf_debug_tc_profile": (I, [P]),
    "sf_probe_l2_read": (I, [C.c_size_t, I, P]),
}

STAGES = ("config", "features_diffuse", "features_highlight", "slice", "backbone", "sample_sort", "march", "combiner",
          "records")


def profile_read():
    """Summed device ms and launch counts per stage since the last read."""
    ms = (C.c_double * len(STAGES))()
    n = (C.c_int64 * len(STAGES))()
    check(lib.sf_profile_read(ms, n))
    return {s: (ms[i], n[i]) for i, s in enumerate(STAGES)}

EXPORTS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_2401_14051_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int):
    if rc != 0:
        raise ScatterfieldError(rc, lib.sf_last_error().decode())


def ptr(a):
    """Raw pointer of a numpy array / torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def dvec(v):
    return (C.c_double * 3)(*[float(x) for x in v])
