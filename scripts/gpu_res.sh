mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or modes" 2>&1 | tail -15
timeout 300 python bench.py --steps 30 --warmup 5 --mode resident --no-cpu-baseline --json-out gpurun_out/bench_c2_resident.json > gpurun_out/bench_c2_resident.log 2>&1; tail -c 300 gpurun_out/bench_c2_resident.log
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --mode resident --no-cpu-baseline --json-out gpurun_out/bench_c3_resident.json > gpurun_out/bench_c3_resident.log 2>&1; tail -c 300 gpurun_out/bench_c3_resident.log
timeout 120 python scripts/trace.py c2 resident > gpurun_out/trace_c2.txt 2>&1; tail -5 gpurun_out/trace_c2.txt
