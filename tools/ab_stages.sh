# stream-ring depth sweep: "$1" = configs, "$2" = list of env settings (comma-separated vars)
for r in 1 2; do for c in $1; do for e in $2; do
  env $(echo $e | tr ',' ' ') timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $e', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'tree', round(d['dimension_tree']['value'],1))"
done; done; done
