"""Several library builds / env settings on the C5 frame query (tools/ab_c5.py's workload):
device ms per query call, per-stage ms, and whether F is identical to the first arm's.
usage: python tools/ab_multi.py NAME=LIB[@K=V,K=V] ...   (LIB "tree" = the in-tree build)"""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
from ab_c5 import code  # noqa: E402

first = None
for arg in sys.argv[1:]:
    name, spec = arg.split("=", 1)
    lib, _, envs = spec.partition("@")
    env = dict(os.environ)
    if lib != "tree":
        env["SF_B200_LIB"] = os.path.abspath(lib)
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    out = f"/tmp/abm_{name}.npy"
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True)
    res = {"arm": name, "result": r.stdout.strip() or r.stderr[-400:]}
    if os.path.exists(out):
        F = np.load(out)
        if first is None:
            first = F
        res["identical_to_first"] = bool(np.array_equal(F, first))
    print(json.dumps(res), flush=True)
