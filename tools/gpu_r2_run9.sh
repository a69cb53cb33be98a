cd $GRAFT_REPO_ROOT
b() { timeout 600 python bench.py --config $1 --steps 40 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value'],1))" >> gpurun_out/r2i_bench.txt; }
for rep in 1 2; do
CPQR_OVERLAP=0 b 2 "c2 serial"
CPQR_OVERLAP=1 b 2 "c2 ov r4"
CPQR_OVERLAP=1 CPQR_VN_QR=cq b 2 "c2 ov r4 vncq"
CPQR_OVERLAP=1 CPQR_OVERLAP_SMS=8 b 2 "c2 ov r8"
CPQR_OVERLAP=1 CPQR_OVERLAP_SMS=8 CPQR_VN_QR=cq b 2 "c2 ov r8 vncq"
CPQR_OVERLAP=1 CPQR_OVERLAP_SMS=16 CPQR_VN_QR=cq b 2 "c2 ov r16 vncq"
CPQR_OVERLAP=0 CPQR_VN_QR=cq b 2 "c2 serial vncq"
CPQR_OVERLAP=0 CPQR_STR_CW=8 b 2 "c2 serial cw8"
done
