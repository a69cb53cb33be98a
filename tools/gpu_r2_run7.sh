cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for c in 2 3 5; do for pdl in 0 1; do
  CPQR_PDL=$pdl timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c pdl $pdl', round(d['value'],1), round(d['roofline']['frac'],3), round(d.get('dimension_tree',{}).get('value',0),1))" >> gpurun_out/r2g_bench.txt
done; done; done
timeout 600 python tools/plan_table.py > gpurun_out/r2g_plans.md 2>&1
