cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --maxfail=15 > gpurun_out/r2_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputests.log
tail -30 gpurun_out/r2_gputests.log
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
tail -5 gpurun_out/r2_bench.log
