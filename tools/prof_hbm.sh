mkdir -p gpurun_out
timeout 300 python tools/prof_case.py --config 2 --sweeps 1 --graph 0 --profile 0 > /dev/null 2>&1 && timeout 600 \
  ncu --set full --import-source on --clock-control none -k regex:"k_strided_tma" -s 2 -c 1 \
      -o gpurun_out/c2_stream python tools/prof_case.py --config 2 --sweeps 1 --graph 0 --profile 0 > gpurun_out/ncu_c2.log 2>&1
timeout 300 python tools/prof_case.py --config 3 --sweeps 1 --graph 0 --profile 0 > /dev/null 2>&1 && timeout 600 \
  ncu --set full --import-source on --clock-control none -k regex:"k_slice_tma|k_strided_tma" -s 0 -c 3 \
      -o gpurun_out/c3_stream python tools/prof_case.py --config 3 --sweeps 1 --graph 0 --profile 0 > gpurun_out/ncu_c3.log 2>&1
ls gpurun_out
