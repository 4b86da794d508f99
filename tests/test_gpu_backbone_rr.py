"""The round-robin tensor-core backbone (k_backbone_rr, opt-in with SF_TC_RR=1: the three
feature-type chains of a tile interleaved in one CTA behind an MMA-issuer warp) is bit-identical to
the default one-chain kernel (k_backbone_tc): same GEMMs on the same 16-bit operands in the same
K order, fp32 epilogues in the same order. Both kernels run in subprocesses (the selection is read
once per process), on a ragged batch (partial last tile), bf16 and fp16 operands, learned and
literal attention."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys
sys.path.insert(0, os.environ["SF_ROOT"])
import numpy as np
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
data = os.path.join(os.path.dirname(sf.__file__), "data")
vol = scenes.procedural_cloud(64, 2)
g = sf.DensityGrid.from_array(vol, 2.0 / 64, (-1.0, -1.0, -1.0))
sc = sf.Scene(g, sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT),
              sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")),
              sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")),
              sf.PhaseModel.hg(0.7), sf.PhaseTable(64, 128, 32, 16))
rows = scenes.draw_centers(vol, 5000, 3, scenes.LIGHT)
med = sf.MediumParams((0.7,), (0.99,) * 3)
out = {}
for literal in (False, True):
    net = sf.make_backbone(sf.BackboneConfig(seed=0, literal_attention=literal))
    for name, prec in (("bf16", sf.BF16), ("fp16", sf.FP16)):
        y = np.empty((len(rows), 3), np.float32)
        F = sf.query(sc, net, med, rows, prec, y_out=y)
        out[f"{name}_{int(literal)}_y"] = y
        out[f"{name}_{int(literal)}_F"] = F
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, rr):
    out = str(tmp_path / f"rr{rr}.npz")
    env = dict(os.environ, SF_ROOT=ROOT, SF_TC_RR=str(rr))
    r = subprocess.run([sys.executable, "-c", SCRIPT, out], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_rr_bit_identical(tmp_path):
    a, b = _run(tmp_path, 0), _run(tmp_path, 1)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.all(np.isfinite(a[k])), k
        assert np.array_equal(a[k], b[k]), (k, np.abs(a[k] - b[k]).max())
