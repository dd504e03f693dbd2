mkdir -p gpurun_out/frows
for c in c2 c3 c5; do
  st=20; [ $c != c2 ] && st=5
  timeout 300 python bench.py --config $c --steps $st --warmup 3 --compact --no-cpu-baseline --json-out gpurun_out/frows/${c}_compact.json > gpurun_out/frows/${c}_compact.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/frows/${c}_compact.json'));print('$c compact', round(d['value'],1), 'Mpx/s', round(d['ms_per_step'],4), 'ms')" 2>/dev/null || tail -2 gpurun_out/frows/${c}_compact.log
done
