# Round-end evidence on the final code: GPU suite, C3 / C2 / C5 bench lines, launch list + ncu of layer 0,
# sanitizers on the chain
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputests.log
tail -3 gpurun_out/r2_gputests.log
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
tail -c 400 gpurun_out/r2_bench.log
timeout 900 python bench.py --workload C2 > gpurun_out/r2_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_c2.log
timeout 900 python bench.py --workload C5 > gpurun_out/r2_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches.csv > gpurun_out/r2_launches.txt; head -9 gpurun_out/r2_launches.txt
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -c 9 \
  -o gpurun_out/r2_full_layer0 -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_chain.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log; tail -2 gpurun_out/sanitize_$tool.log
done
