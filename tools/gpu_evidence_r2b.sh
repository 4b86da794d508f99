# Round-2 evidence on the current build: the launch list of one C5 frame and two ncu --set full
# captures of the last of two C5 frames (query kernels; level 0's first graded pass), for
# tools/ncu_summary.py -> profiles/ncu_c5.json.
cd $GRAFT_REPO_ROOT
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c5_frame.csv python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
timeout -k 10 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_(sample_sort|backbone_tc|query_prep)" -c 3 -f -o gpurun_out/r2_c5_query python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_query.log 2>&1
tail -2 gpurun_out/ncu_query.log
timeout -k 10 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_(graded_cols|tap_build|conv3_zwin|combine_blk|xpair)" -c 60 -f -o gpurun_out/r2_c5_build python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_build.log 2>&1
tail -2 gpurun_out/ncu_build.log
ls -la gpurun_out
# summarise on the box (the build report is too large to bring back) and keep only the query report
python tools/ncu_summary.py gpurun_out/r2_c5_build.ncu-rep,gpurun_out/r2_c5_query.ncu-rep "ncu --set full --clock-control none of the last of 2 C5 frames (tools/profile_c5.py --frames 2 --profile-last, fp16 query, FP32-sum tap build), first launch of each kernel: r2_c5_build (build kernels) + r2_c5_query (k_query_prep, k_sample_sort and k_backbone_tc on the first 524,288-query chunk), B200, current build" gpurun_out/ncu_c5.json > gpurun_out/ncu_summary.log 2>&1
tail -2 gpurun_out/ncu_summary.log
rm -f gpurun_out/r2_c5_build.ncu-rep gpurun_out/ss_full.ncu-rep
