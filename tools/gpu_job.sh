# GPU suite + bench (+ optional synccheck) on the box; logs into gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --maxfail=15 > gpurun_out/r2_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputests.log
tail -30 gpurun_out/r2_gputests.log
if [ -z "$NOBENCH" ]; then
  timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
  tail -5 gpurun_out/r2_bench.log
fi
if [ -n "$SYNCCHECK" ]; then
  timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_chain.py > gpurun_out/sanitize_synccheck.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_synccheck.log; tail -4 gpurun_out/sanitize_synccheck.log
fi
