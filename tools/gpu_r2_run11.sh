cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "overlap or profile" 2>&1 | tail -5 > gpurun_out/r2k_ov.log
CPQR_OVERLAP=1 CPQR_TRACE=1 timeout 300 python tools/trace_case.py 2 > gpurun_out/r2k_trace_c2.txt 2>&1
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1))" >> gpurun_out/r2k_bench.txt; }
for rep in 1 2; do
for c in 2 3 4; do
CPQR_OVERLAP=0 b $c "c$c serial"
CPQR_OVERLAP=1 b $c "c$c ov"
done; done
