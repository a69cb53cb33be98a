cd $GRAFT_REPO_ROOT
for c in 2 3 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n1_launch_c$c.csv \
    python tools/prof_case.py --config $c --sweeps 1 --graph 0 --profile 0 > gpurun_out/n1_ncu_c$c.log 2>&1
done
