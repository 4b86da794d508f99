cd $GRAFT_REPO_ROOT
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c5_frame.csv python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
timeout -k 10 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_(sample_sort|graded_cols|backbone_tc)" -c 3 -o gpurun_out/ss_full python tools/profile_c5.py --frames 2 --profile-last > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
