# new kernels: parity first, then interleaved A/B bench lines
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "small_ttm or householder_tail or streamk or overlap or debug_mode" 2>&1 | tail -8 > gpurun_out/ab1_tests.log
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 4 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1), round(d.get('dimension_tree',{}).get('value',0),1), d['gpu_launches'])" >> gpurun_out/ab1_bench.txt; }
for rep in 1 2; do
for c in 2 3 4 5; do
CPQR_TTM_SMALL=0 CPQR_SK_FIXUP=1 CPQR_RQ_SERIAL=0 b $c "c$c old"
b $c "c$c new"
CPQR_TTM_SMALL=0 b $c "c$c nosmall"
done; done
