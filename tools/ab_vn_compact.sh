for r in 1 2; do for c in 3 4 5 2; do for e in "CPQR_VN_TREE=0" "CPQR_VN_TREE=1,CPQR_VN_COMPACT=0" "CPQR_VN_TREE=1"; do
  env $(echo $e | tr ',' ' ') timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $e', round(d['value'],1), 'tree', round(d['dimension_tree']['value'],1))"
done; done; done
