# Round evidence on one B200 (run from the repo root under gpurun): whole GPU suite + smoke, then
# tools/round_profile.sh (bench lines C2-C5, the default bench command's ncu launch list, ncu
# --set full of the C5 stream kernels and of the HBM-bound passes), the slab projection and a
# C2 launch list.  Outputs under gpurun_out/; summaries are copied into profiles/ by hand.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export ROUND=${ROUND:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi_$ROUND.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/suite_$ROUND.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$ROUND.log 2>&1
bash tools/round_profile.sh > gpurun_out/round_profile_$ROUND.log 2>&1
timeout 1200 python tools/slab_projection.py --configs 3 4 5 > gpurun_out/slab_projection_$ROUND.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$ROUND.csv \
  python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
