# Round profile evidence: bench line, launch list of one C3 prefill, ncu --set full of layer 0 + head
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
tail -2 gpurun_out/r2_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches.csv > gpurun_out/r2_launches.txt; cat gpurun_out/r2_launches.txt
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -c 9 \
  -o gpurun_out/r2_full_layer0 -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-skip 198 -c 1 \
  -o gpurun_out/r2_full_head -f python tools/profile_step.py >> gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
