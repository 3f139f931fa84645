cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:attn_paged -s 5 -c 1 -o gpurun_out/attn_se1 -f python tools/attn_paged_bench.py 1 > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log
