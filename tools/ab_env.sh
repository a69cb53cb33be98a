# A/B an environment switch on one box: bash tools/ab_env.sh VAR "valA valB" "configs" [reps]
VAR=$1; VALS=$2; CFGS=$3; REPS=${4:-2}
for r in $(seq $REPS); do
 for c in $CFGS; do
  for v in $VALS; do
   env $VAR=$v python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d.get('dimension_tree',{}).get('value'); print('$c', '$VAR=$v', round(d['value'],1), 'tree', round(t,1) if t else None)"
  done
 done
done
