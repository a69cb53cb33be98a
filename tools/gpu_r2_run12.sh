cd $GRAFT_REPO_ROOT
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1))" >> gpurun_out/r2l_bench.txt; }
for rep in 1 2; do
for c in 2 4 3; do
CPQR_OVERLAP=0 b $c "c$c serial"
CPQR_OVERLAP=1 b $c "c$c ov"
CPQR_OVERLAP=1 CPQR_OVERLAP_CW1=0 b $c "c$c ov nocw1"
CPQR_OVERLAP=1 CPQR_OVERLAP_CW1=0 CPQR_OVERLAP_SMS=1 b $c "c$c ov nocw1 r1"
done; done
