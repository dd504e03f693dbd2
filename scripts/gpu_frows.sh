# measurements of the SURVEY 8(f) rows: LAB pre-pass, metrics (means: scripts/gpu_means.sh)
mkdir -p gpurun_out/frows
for c in c2 c3 c5; do
  st=20; [ $c != c2 ] && st=5
  timeout 300 python bench.py --config $c --steps $st --warmup 3 --colour lab --no-cpu-baseline --json-out gpurun_out/frows/${c}_lab.json > gpurun_out/frows/${c}_lab.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/frows/${c}_lab.json'));print('$c lab', round(d['value'],1), 'Mpx/s', round(d['ms_per_step'],4), 'ms')" 2>/dev/null || tail -2 gpurun_out/frows/${c}_lab.log
done
timeout 300 python scripts/metrics_bench.py > gpurun_out/frows/metrics.jsonl 2>&1; cut -c1-160 gpurun_out/frows/metrics.jsonl
