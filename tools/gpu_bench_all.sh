# The four bench lines of this build (C5 default with the CPU baseline; C3; C2; C4 without the 116 s
# reference build) into gpurun_out/bench_<config>.json, plus a one-line summary of each.
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --config c3 --steps 8 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config c2 --steps 100 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for c in c5 c3 c2 c4; do
python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
print(c, round(d["value"] / 1e6, 2), "Mq/s", round(d["ms_per_step"], 3), "ms/step e2e", round(d["e2e"]["value"] / 1e6, 2),
      "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: round(v, 3) for k, v in d["stages"]["per_step_ms"].items()},
      "par", (d.get("parity") or {}).get("max_dy_equiv"), (d.get("parity") or {}).get("n_over_bound"),
      "cpu", (d.get("cpu_baseline") or {}).get("value"))
PY
done
