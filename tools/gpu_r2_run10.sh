cd $GRAFT_REPO_ROOT
CPQR_OVERLAP=1 CPQR_TRACE=1 timeout 300 python tools/trace_case.py 2 > gpurun_out/r2j_trace_c2.txt 2>&1
CPQR_OVERLAP=1 CPQR_TRACE=1 timeout 300 python tools/trace_case.py 4 > gpurun_out/r2j_trace_c4.txt 2>&1
