# ncu --set full of the HBM-bound configs' stream-X kernels (C2 strided, C3 strided + fused slice,
# C4 fused last-two-modes strided + small slice), one launch each; summaries -> profiles/ncu_hbm_stream_r01.json
mkdir -p gpurun_out
for cfg in "2 k_strided_tma 0" "3 k_strided_tma 0" "3 k_slice_tma 0" "4 k_strided2_tma 0" "4 k_slice_small_tma 0"; do
  set -- $cfg
  timeout 300 python tools/prof_case.py --config $1 --sweeps 1 --graph 0 --profile 0 > /dev/null 2>&1 && timeout 600 \
    ncu -f --set full --import-source on --clock-control none -k regex:"$2" -s $3 -c 1 \
        -o /tmp/hbm_c$1_$2 python tools/prof_case.py --config $1 --sweeps 1 --graph 0 --profile 0 > gpurun_out/ncu_hbm_c$1_$2.log 2>&1
  ncu -i /tmp/hbm_c$1_$2.ncu-rep --page raw --csv > gpurun_out/hbm_c$1_$2.csv 2>/dev/null
done
ls gpurun_out | grep hbm_
# the L2-resident intermediate TTM (k_ttm_small) is captured warm (--cache-control none): its input
# was just written by the stream pass in the sweep
timeout 300 python tools/prof_case.py --config 2 --sweeps 1 --graph 0 --profile 0 > /dev/null 2>&1 && timeout 600 \
  ncu -f --set full --import-source on --clock-control none --cache-control none -k regex:"k_ttm_small" -s 0 -c 3 \
      -o /tmp/hbm_c2_k_ttm_small python tools/prof_case.py --config 2 --sweeps 1 --graph 0 --profile 0 > gpurun_out/ncu_hbm_c2_k_ttm_small.log 2>&1
ncu -i /tmp/hbm_c2_k_ttm_small.ncu-rep --page raw --csv > gpurun_out/hbm_c2_k_ttm_small.csv 2>/dev/null
