cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "staircase" 2>&1 | tail -5 > gpurun_out/r2m_stair.log
timeout 1500 python tools/q0_stair_bench.py > gpurun_out/r2m_stair_bench.md 2>&1
