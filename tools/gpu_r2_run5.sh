cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "streamk or kruskal" 2>&1 | tail -20 > gpurun_out/r2e_tests.log
timeout 600 python tools/sine_curves.py > gpurun_out/r2e_sine.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_c5p8.csv python tools/prof_case.py --config 5 --world 8 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2e_c5p8.log 2>&1
for sk in 0 -1 0 -1; do CPQR_STREAMK=$sk timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sk $sk', d['value'], d['roofline']['frac'], d.get('dimension_tree',{}).get('value'))" >> gpurun_out/r2e_bench.txt; done
timeout 600 python tools/slab_projection.py --configs 5 > gpurun_out/r2e_proj.txt 2>&1
