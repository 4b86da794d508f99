"""Morton-order processing of large batches (sf_capi.cpp query path, SF_MORTON) changes only
the order queries are processed in: every row's F must be bit-identical to in-order
processing, for device and host I/O and for per-query media (C4)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

CODE = r"""
import os, sys
sys.path.insert(0, os.environ["SF_ROOT"])
import numpy as np, torch
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
d, a, gg = scenes.mixed_medium(64, 3)
g = sf.DensityGrid.from_array(d, 2.0 / 64, (-1.0, -1.0, -1.0))
tv = sf.build_transmittance_volume(sf.DensityPyramid(g), scenes.LIGHT)
data = os.path.join(os.path.dirname(sf.__file__), "data")
sc = sf.Scene(g, tv, sf.load_template(os.path.join(data, "diffuse_seed7.vtmpl")),
              sf.load_template(os.path.join(data, "highlight_seed8.vtmpl")), sf.PhaseModel.hg(0.6),
              sf.PhaseTable(64, 128, 32, 16))
net = sf.make_backbone(sf.BackboneConfig(seed=0))
rows = scenes.draw_centers(d, 20000, 4, scenes.LIGHT)
med = sf.MediumParams((0.6,), (0.97,) * 3)
F_host = sf.query(sc, net, med, rows, sf.BF16)
Fd = torch.empty((len(rows), 3), dtype=torch.float64, device="cuda")
sf.query(sc, net, med, torch.from_numpy(rows).cuda(), sf.BF16, F_out=Fd)
F_media = sf.query_media(sc, net, rows, scenes.sample_media(a, gg, rows), sf.BF16)
np.save(sys.argv[1], np.stack([F_host, Fd.cpu().numpy(), F_media]))
"""


def test_morton_order_is_bit_identical(tmp_path):
    out = {}
    for mode in ("0", "1"):
        path = str(tmp_path / f"F{mode}.npy")
        env = dict(os.environ, SF_MORTON=mode, SF_ROOT=ROOT)
        r = subprocess.run([sys.executable, "-c", CODE, path], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = np.load(path)
    assert np.array_equal(out["0"], out["1"])
    assert np.array_equal(out["0"][0], out["0"][1])  # host and device I/O agree
