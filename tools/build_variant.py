"""Build a variant of libsf_b200.so with extra nvcc defines into OUT.so (A/B tooling):
python tools/build_variant.py OUT.so -DFOO -DBAR"""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2401_14051_b200"))
import build as B  # noqa: E402
out, defs = sys.argv[1], sys.argv[2:]
tmp = out + ".objs"
os.makedirs(tmp, exist_ok=True)
objs = []
for src in B.SOURCES:
    o = os.path.join(tmp, os.path.splitext(src)[0] + ".o")
    r = subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o], capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    objs.append(o)
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-cudart", "static"], capture_output=True, text=True)
sys.exit(r.returncode and r.stderr)
