cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "multi_sweep or overlap or profile or determinism" 2>&1 | tail -8 > gpurun_out/r2o_tests.log
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1), round(d.get('dimension_tree',{}).get('value',0),1))" >> gpurun_out/r2o_bench.txt; }
for rep in 1 2; do
for c in 2 3 4 5; do
CPQR_GRAPH_SWEEPS=1 b $c "c$c g1"
CPQR_GRAPH_SWEEPS=2 b $c "c$c g2"
CPQR_GRAPH_SWEEPS=4 b $c "c$c g4"
done; done
