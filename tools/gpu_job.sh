cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "paged or relocate" -p no:cacheprovider > gpurun_out/r2c_kern.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_kern.log
tail -15 gpurun_out/r2c_kern.log
