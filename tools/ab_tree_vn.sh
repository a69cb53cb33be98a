# A/B of the tree-mode V_n QR choice (CPQR_VN_TREE=0: side-stream Householder; 1: inline CholeskyQR2)
cfgs=${1:-"5 3 4"}
for r in 1 2; do for c in $cfgs; do
  for mode in "CPQR_VN_TREE=0" "CPQR_VN_TREE=1"; do
    env $mode timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$mode', round(d['value'],1), 'tree', round(d['dimension_tree']['value'],1))"
  done
done; done
