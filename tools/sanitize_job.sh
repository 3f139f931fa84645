# compute-sanitizer over the C1 + C2x2 chain (tools/sanitize_chain.py); summaries into gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_chain.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
