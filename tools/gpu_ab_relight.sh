# A/B of the side-stream priority on Scene.relight (C5 per-frame build) and on the C5 bench line
cd $GRAFT_REPO_ROOT
python tools/ab_relight.py lo=tree@SF_SIDE_PRIO=0 hi=tree lo2=tree@SF_SIDE_PRIO=0 hi2=tree > gpurun_out/ab_relight.log 2>&1
cat gpurun_out/ab_relight.log
SF_SIDE_PRIO=0 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_lo.json 2> gpurun_out/bench_lo.err
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_hi.json 2> gpurun_out/bench_hi.err
python -c "
import json
for a in ('lo','hi'):
    d=json.load(open(f'gpurun_out/bench_{a}.json')); print(a, d['value']/1e6, d['ms_per_step'], {k: round(v,3) for k,v in d['stages']['per_step_ms'].items()})"
