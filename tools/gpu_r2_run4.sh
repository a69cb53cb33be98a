cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "streamk" 2>&1 | tail -20 > gpurun_out/r2d_sk.log
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -rf -x 2>&1 | tail -20 > gpurun_out/r2d_slabs.log
for c in 5 2; do CPQR_LIB=$PWD/paper_2112_10855_b200/libcpqr_dbg.so timeout 300 python tools/prof_case.py --config $c --sweeps 1 --graph 1 --profile 0 > gpurun_out/r2d_dbg_c$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_c5p8.csv python tools/prof_case.py --config 5 --world 8 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2d_c5p8.log 2>&1
for sk in 0 -1; do CPQR_STREAMK=$sk timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2d_bench_c5_sk$sk.json 2>/dev/null; done
CPQR_STREAMK=0 timeout 600 python tools/slab_projection.py --configs 5 > gpurun_out/r2d_proj_sk0.txt 2>&1
timeout 600 python tools/slab_projection.py --configs 5 > gpurun_out/r2d_proj_sk.txt 2>&1
