# Timeline (CPQR_TRACE, eager) and ncu launch lists of C2 and C5 eager sweeps.
cd $GRAFT_REPO_ROOT
for c in 2 5; do
  CPQR_TRACE=1 timeout 300 python tools/trace_case.py $c > /dev/null 2> gpurun_out/t_trace_c$c.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t_launch_c$c.csv \
    python tools/prof_case.py --config $c --sweeps 2 --graph 0 --profile 0 > gpurun_out/t_ncu_c$c.log 2>&1
done
