cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "svd_truncation or edivergred or tall_factor or debug_calls" 2>&1 | tail -30 > gpurun_out/r2b_newpar.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rf 2>&1 | tail -30 > gpurun_out/r2b_full.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2b_bench_c5.json 2> gpurun_out/r2b_bench_c5.err
timeout 1200 python tools/slab_projection.py --configs 3 4 5 > gpurun_out/r2b_proj.txt 2>&1
