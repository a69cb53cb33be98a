# Round-2 (session 2) baseline at HEAD: whole GPU suite, smoke, default bench, per-config bench lines.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/b_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/b_bench_default.json 2> gpurun_out/b_bench_default.err
for c in 2 3 4; do
  timeout 600 python bench.py --config $c --steps 40 --warmup 4 --no-cpu > gpurun_out/b_bench_c$c.json 2>/dev/null
done
timeout 600 python bench.py --config 2 --variant NE --steps 40 --warmup 4 --no-cpu > gpurun_out/b_bench_c2ne.json 2>/dev/null
timeout 600 python bench.py --config 3 --variant SVD --steps 40 --warmup 4 --no-cpu > gpurun_out/b_bench_c3svd.json 2>/dev/null
