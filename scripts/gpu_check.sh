mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for m in graph resident; do
  timeout 300 python bench.py --steps 30 --warmup 5 --mode $m --no-cpu-baseline --json-out gpurun_out/bench_c2_$m.json > gpurun_out/bench_c2_$m.log 2>&1; tail -c 600 gpurun_out/bench_c2_$m.log
  timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --mode $m --no-cpu-baseline --json-out gpurun_out/bench_c3_$m.json > gpurun_out/bench_c3_$m.log 2>&1; tail -c 600 gpurun_out/bench_c3_$m.log
done
timeout 120 python tools_trace.py c2 > gpurun_out/trace_c2.txt 2>&1; tail -30 gpurun_out/trace_c2.txt
