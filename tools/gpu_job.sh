cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi -L) > gpurun_out/r2a_host.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2a_bench.log
for t in memcheck synccheck racecheck; do timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_chain.py > gpurun_out/r2a_san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_san_$t.log; done
tail -3 gpurun_out/r2a_pytest.log; tail -c 600 gpurun_out/r2a_bench.log
