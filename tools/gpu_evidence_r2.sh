set -x
cd $GRAFT_REPO_ROOT
timeout -k 10 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_(graded_cols|sample_sort|backbone_tc|tap_build|query_prep|conv3_zwin|combine_blk|xpair)" -c 16 -o gpurun_out/r2_c5_final python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_final.log 2>&1
tail -3 gpurun_out/ncu_final.log
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c5_frame.csv python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
python bench.py --config c2 --steps 100 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 300 gpurun_out/bench_c2.json
python bench.py --config c3 --steps 8 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 300 gpurun_out/bench_c4.json
ls -la gpurun_out/
