"""Artifact formats against files written by the reference itself
(tests/golden/io/, tests/golden/make_golden.py io): readers recover the reference's values,
writers reproduce its bytes, loads fail with the reference's Errc."""
import os
import struct

import numpy as np
import pytest

from conftest import DATA, GOLD, LIGHT, ORIGIN
from oracle.oracle import BackboneCfg, PhaseModel
from paper_2401_14051_b200 import io
from paper_2401_14051_b200._lib import ScatterfieldError
from paper_2401_14051_b200.scenes import procedural_cloud

IO = os.path.join(GOLD, "io")


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", ["small.vgrid", "small.vfeat", "tiny.vnet", "lit.vnet"])
def test_round_trip_bytes_identical(tmp_path, name):
    src = os.path.join(IO, name)
    dst = str(tmp_path / name)
    if name.endswith(".vgrid"):
        io.save_density_array(*io.load_density_array(src), dst)
    elif name.endswith(".vfeat"):
        io.save_feature_table(io.load_feature_table(src), dst)
    else:
        io.write_network(*io.read_network(src), dst)
    assert _bytes(dst) == _bytes(src)


def test_vgrid_values():
    v, vs, origin = io.load_density_array(os.path.join(IO, "small.vgrid"))
    assert vs == 0.125 and origin == (-1.0, -1.0, -1.0)
    assert np.array_equal(v, procedural_cloud(16, 3))


def test_vfeat_blocks_match_oracle(oracle, templates):
    t = io.load_feature_table(os.path.join(IO, "small.vfeat"))
    assert (t.lambda_, t.template_scale) == (0.6, 1.5) and t.phase_table.shape == (9, 17, 5)
    assert np.array_equal(t.kernels[:, 13], np.ones(5, np.float32)) and np.allclose(t.scales, 0.2)
    assert np.allclose(t.centers[:, 6:], LIGHT)
    g = procedural_cloud(16, 3)
    tv = oracle.build_tvol(g, 0.125, ORIGIN, LIGHT)
    table = oracle.phase_table(9, 17, 5, 8)
    assert np.array_equal(t.phase_table, table)
    sc = oracle.make_scene(g, tv, 0.125, ORIGIN, templates[0], templates[1], PhaseModel.hg(0.7), table, 1.5)
    assert np.array_equal(t.features(), oracle.features(sc, t.centers))


@pytest.mark.parametrize("name,lit", [("tiny.vnet", False), ("lit.vnet", True)])
def test_vnet_params_match_oracle_init(oracle, name, lit):
    cfg, params = io.read_network(os.path.join(IO, name))
    assert (cfg.diffuse_counts, cfg.highlight_counts, cfg.width, cfg.merge_width, cfg.head_width, cfg.seed,
            cfg.literal_attention) == ((2, 3), (2,), 4, 8, 8, 5, lit)
    ocfg = BackboneCfg(diffuse_counts=(2, 3), highlight_counts=(2,), width=4, merge_width=8, head_width=8, seed=5,
                       literal_attention=lit)
    assert np.array_equal(params, oracle.backbone_init(ocfg))
    assert sum(int(np.prod(s)) for _, s in io.param_layout(cfg)) == len(params)


def test_load_errors(tmp_path):
    good = _bytes(os.path.join(IO, "small.vgrid"))
    cases = {
        "magic.vgrid": (b"XGRD" + good[4:], 2),
        "trunc.vgrid": (good[:-3], 5),
        "dims.vgrid": (good[:8] + struct.pack("<I", 12) + good[12:], 3),
        "neg.vgrid": (good[:36] + struct.pack("<f", -1.0) + good[40:], 4),
    }
    net = bytearray(_bytes(os.path.join(IO, "tiny.vnet")))
    net[76] ^= 1  # a byte of the config JSON: digest mismatch
    cases["digest.vnet"] = (bytes(net), 8)
    feat = _bytes(os.path.join(IO, "small.vfeat"))
    cases["trunc.vfeat"] = (feat[:100], 5)
    for name, (data, code) in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(ScatterfieldError) as e:
            if name.endswith(".vgrid"):
                io.load_density_array(str(p))
            elif name.endswith(".vnet"):
                io.read_network(str(p))
            else:
                io.load_feature_table(str(p))
        assert e.value.code == code, name
    with pytest.raises(ScatterfieldError) as e:
        io.load_density_array(str(tmp_path / "missing.vgrid"))
    assert e.value.code == 1
