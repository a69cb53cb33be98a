cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "tall_factor or pinv or debug_calls or svd_trunc" 2>&1 | tail -40 > gpurun_out/r2c_newpar.log
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_fuzz.py -q -rf -k "pinv or PINV" 2>&1 | tail -30 > gpurun_out/r2c_pinv.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rf -k "PINV" 2>&1 | tail -30 > gpurun_out/r2c_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_c5p8.csv python tools/prof_case.py --config 5 --world 8 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2c_c5p8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_c5p1.csv python tools/prof_case.py --config 5 --world 1 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2c_c5p1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_c2p1.csv python tools/prof_case.py --config 2 --world 1 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2c_c2p1.log 2>&1
