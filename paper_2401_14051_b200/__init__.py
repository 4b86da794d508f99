"""paper_2401_14051_b200 — B200-native per-shading-point hot path of the neural
in-scattering renderer of arXiv 2401.14051 (reference: "scatterfield").

The compute lives in libsf_b200.so (hand-written sm_100a CUDA behind the C ABI
in include/scatterfield_b200.h); this package is the Python mirror of the
reference's C++ API over that ABI. Importing fails loudly if the library is
missing — there is no CPU fallback.
"""
from ._lib import EXPORTS, LIB_PATH, ScatterfieldError, lib  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import (BF16, DIFFUSE, FP16, FP32, HIGHLIGHT, Backbone, BackboneConfig, CombinerWeights, ConfigParams,  # noqa
                  DensityGrid, DensityPyramid, FeatureConfig, MediumParams, PhaseModel, PhaseTable,
                  SamplingTemplate, Scene, TransmittanceFeatureVolume, angle_between, build_pyramid,
                  build_transmittance_slab, build_transmittance_volume, combine_transmittance, config_rows, conv3_replicate,
                  decode_prediction, encode_label, graded_transmittance, light_entry_point, load_template,
                  make_backbone, make_config, place_template, predict, predict_y, query, query_media, sample_features,
                  Camera, RenderOptions, bake_field, render_volume, render_neural, pinned_empty,
                  save_template, debug_query_pools)

__version__ = "0.1.0"
