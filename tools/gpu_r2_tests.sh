cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -rf -x 2>&1 | tail -30 > gpurun_out/r2_slabs.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_solver.py -q -rf 2>&1 | tail -30 > gpurun_out/r2_parity.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -rf 2>&1 | tail -30 > gpurun_out/r2_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
