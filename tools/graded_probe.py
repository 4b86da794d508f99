"""One transmittance build per (grid, march) for ncu kernel timing."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2401_14051_b200 as sf
from paper_2401_14051_b200 import scenes
N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
fast = len(sys.argv) > 2 and sys.argv[2] == "fp32"
vol = scenes.fractal_ellipsoid(N, 1) if N == 128 else scenes.noise_volume(N, 5)
pyr = sf.DensityPyramid(sf.DensityGrid.from_array(vol, 2.0 / N, (-1.0, -1.0, -1.0)))
sf.build_transmittance_volume(pyr, scenes.LIGHT, fast=fast)
print("ok")
