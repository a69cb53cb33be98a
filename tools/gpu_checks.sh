# Correctness tooling without compute-sanitizer (closed on this pool): guard-band canaries around
# every device allocation + NaN poisoning of fresh allocations over the whole GPU suite and the
# kernel-coverage cases of tools/sanitize.py, then run-to-run bitwise determinism probes.
cd $GRAFT_REPO_ROOT
CPQR_CANARY=1 CPQR_POISON=1 timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/chk_suite.log
CPQR_CANARY=1 CPQR_POISON=1 timeout 600 python tools/sanitize.py > gpurun_out/chk_cases.log 2>&1; echo "rc=$?" >> gpurun_out/chk_cases.log
timeout 1500 python tools/stress_sweep.py 2,3,4,5 10 both > gpurun_out/chk_stress.log 2>&1; echo "rc=$?" >> gpurun_out/chk_stress.log
