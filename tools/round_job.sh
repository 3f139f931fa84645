# Round-end evidence: C2 and C5 bench lines, sanitizers on the chain, launch list + ncu of layer 0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload C2 > gpurun_out/r2_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_c2.log
tail -c 600 gpurun_out/r2_bench_c2.log
timeout 900 python bench.py --workload C5 > gpurun_out/r2_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_c5.log
tail -c 600 gpurun_out/r2_bench_c5.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_chain.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log; tail -3 gpurun_out/sanitize_$tool.log
done
