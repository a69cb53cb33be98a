cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -rf -x 2>&1 | tail -15 > gpurun_out/r2f_tests.log
for rep in 1 2; do
for c in 2 5 3 4; do for pdl in 0 1; do
  CPQR_PDL=$pdl timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c pdl $pdl', round(d['value'],1), round(d['roofline']['frac'],3), round(d.get('dimension_tree',{}).get('value',0),1))" >> gpurun_out/r2f_bench.txt
done; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_c5p8.csv python tools/prof_case.py --config 5 --world 8 --graph 0 --profile 0 --warm 1 --sweeps 1 > gpurun_out/r2f_c5p8.log 2>&1
