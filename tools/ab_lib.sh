# A/B of two builds: "$1" configs, "$2" variant (optional); old library at build_ab/libcpqr_old.so vs the in-tree one
for r in 1 2; do for c in $1; do for L in build_ab/libcpqr_old.so paper_2112_10855_b200/libcpqr.so; do
  CPQR_LIB=$PWD/$L timeout 200 python bench.py --config $c ${2:+--variant $2} --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $(basename $L)', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'tree', round(d.get('dimension_tree',{}).get('value',0),1))"
done; done; done
