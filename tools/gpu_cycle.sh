set -o pipefail
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for c in 5 3 2 4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/b$c.err | tail -1 > gpurun_out/b$c.json; done
python - <<PY
import json
for c in (5,3,2,4):
    try:
        d=json.loads(open(f"gpurun_out/b{c}.json").read())
        print(c, round(d["value"],1), round(d["ms_per_step"],4), {k: round(v,3) for k,v in d["phase_ms_per_sweep"].items()}, round(d["roofline"]["frac"],3))
    except Exception as e: print(c, "ERR", e)
PY
if [ -n "$DBG" ]; then CPQR_DEBUG_TIMING=1 python -m paper_2112_10855_b200.build --force > /dev/null 2>&1; for c in 5 2; do python tools/prof_case.py --config $c --sweeps 1 --graph 1 --profile 0 2>&1 | tail -4; done; fi
