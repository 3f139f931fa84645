cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_ttft.py base= nonorm=defer_norm:0 > gpurun_out/ab1.log 2>&1
cat gpurun_out/ab1.log | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r2a.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r2a.csv
