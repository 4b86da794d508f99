# A/B of variants/base.so against the in-tree build on the C5 frame query + relight, then the GPU suite
cd $GRAFT_REPO_ROOT
python tools/ab_multi.py base=variants/base.so new=tree base2=variants/base.so new2=tree > gpurun_out/ab_multi.log 2>&1
python tools/ab_build.py base=variants/base.so new=tree > gpurun_out/ab_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cat gpurun_out/ab_multi.log gpurun_out/ab_build.log; tail -2 gpurun_out/pytest_gpu.log; tail -c 400 gpurun_out/bench_c5.json
