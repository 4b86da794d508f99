# A/B of build variants on the C5 per-frame rebuild (tvol identity + device ms)
cd $GRAFT_REPO_ROOT
python tools/ab_build.py base=variants/base.so comb4=variants/comb4.so comb3=variants/comb3.so grad4=variants/grad4.so base2=variants/base.so comb4b=variants/comb4.so > gpurun_out/ab_build2.log 2>&1
cat gpurun_out/ab_build2.log
