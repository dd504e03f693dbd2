mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "grid or modes" 2>&1 | tail -5
timeout 60 python scripts/trace.py c2 grid 2>&1 | tail -7
timeout 120 python bench.py --steps 30 --warmup 5 --mode grid --no-cpu-baseline --json-out gpurun_out/bench_c2_grid.json > gpurun_out/bench_c2_grid.log 2>&1; tail -c 300 gpurun_out/bench_c2_grid.log
timeout 240 python bench.py --steps 5 --warmup 3 --config c3 --mode grid --no-cpu-baseline --json-out gpurun_out/bench_c3_grid.json > gpurun_out/bench_c3_grid.log 2>&1; tail -c 300 gpurun_out/bench_c3_grid.log
python - <<'P'
import json
for f in ["bench_c2_grid","bench_c3_grid"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.json")); print(f, round(d['value'],1), "Mpx/s", round(d['ms_per_step'],4), "ms")
    except Exception as e: print(f, e)
P
