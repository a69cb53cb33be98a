cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "overlap" 2>&1 | tail -15 > gpurun_out/r2h_ov.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_slabs.py tests/test_gpu_solver.py -q -rf 2>&1 | tail -15 > gpurun_out/r2h_all.log
for rep in 1 2; do
for c in 2 3 4; do for ov in 0 1; do
  CPQR_OVERLAP=$ov timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c ov $ov', round(d['value'],1), round(d['roofline']['frac'],3), round(d.get('dimension_tree',{}).get('value',0),1))" >> gpurun_out/r2h_bench.txt
done; done; done
CPQR_OVERLAP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_c2ov.csv python tools/prof_case.py --config 2 --graph 1 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2h_c2ov.log 2>&1
