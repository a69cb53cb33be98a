# Round evidence: bench lines per config, ncu launch list of the default bench command, one
# ncu --set full capture of the C5 stream kernels.  Run from the repo root on a B200 (gpurun).
set -u
R=${ROUND:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5_$R.json 2> gpurun_out/bench_c5.err
for cv in "3 QR" "3 SVD" "4 SVD" "2 QR" "2 NE"; do
  set -- $cv
  timeout 600 python bench.py --config $1 --variant $2 --steps 100 --warmup 5 > gpurun_out/bench_c$1$(echo $2 | tr A-Z a-z)_$R.json 2>> gpurun_out/bench_other.err
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && timeout 900 \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$R.csv \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_case.py --config 5 --sweeps 1 --graph 0 --profile 0 > /dev/null 2>&1 && timeout 900 \
  ncu -f --set full --import-source on --clock-control none -k regex:"k_strided_tma|k_fiber_tma" -s 4 -c 4 \
      -o /tmp/c5_stream_$R python tools/prof_case.py --config 5 --sweeps 1 --graph 0 --profile 0 \
      > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/c5_stream_$R.ncu-rep --page raw --csv > gpurun_out/c5_stream_$R.csv 2>/dev/null
bash tools/prof_hbm.sh
ls -la gpurun_out
