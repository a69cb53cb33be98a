# Exchange-path measurements on one B200 (run under gpurun from the repo root): the one-rank
# in-graph exchanges (none / NCCL / peer push) on C5 and C2, and the virtual ranks' projection with
# the sum-kernel exchange against the fused peer push-reduce.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in 5 2; do
  for comm in auto nccl peer; do
    steps=20; [ $cfg = 2 ] && steps=200
    python bench.py --config $cfg --steps $steps --warmup 5 --no-e2e --no-cpu --comm $comm \
      > gpurun_out/bench_c${cfg}_comm_${comm}.json 2> gpurun_out/bench_c${cfg}_comm_${comm}.err
  done
done
# the serial schedule without an exchange: the baseline of the one-rank exchanges on C2 (R <= 16
# runs the overlap schedule by default, the exchange paths do not)
CPQR_OVERLAP=0 python bench.py --config 2 --steps 200 --warmup 5 --no-e2e --no-cpu \
  > gpurun_out/bench_c2_comm_none_serial.json 2> /dev/null
timeout 900 python tools/slab_projection.py --configs 5 --ps 1 2 4 8 --comm local > gpurun_out/slab_c5_local.txt 2>&1
timeout 900 python tools/slab_projection.py --configs 5 --ps 2 4 8 --comm local_peer > gpurun_out/slab_c5_local_peer.txt 2>&1
