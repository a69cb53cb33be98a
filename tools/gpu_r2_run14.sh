cd $GRAFT_REPO_ROOT
timeout 900 python tools/collinear_grid.py 10 12 > gpurun_out/r2n_collinear.txt 2>&1
timeout 900 python tools/batched_grid.py > gpurun_out/r2n_batched.txt 2>&1
