cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "multi_sweep" 2>&1 | tail -3 > gpurun_out/r2p_tests.log
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1), round(d.get('dimension_tree',{}).get('value',0),1))" >> gpurun_out/r2p_bench.txt; }
for rep in 1 2 3; do
for c in 2 4; do
CPQR_OVERLAP=0 b $c "c$c serial"
CPQR_OVERLAP=1 b $c "c$c overlap"
done; done
