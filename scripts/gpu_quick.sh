# quick c2 bench lines for A/B comparisons: MODES / CFG / STEPS
for m in ${MODES:-grid}; do
  rm -f /tmp/b.json; timeout 120 python bench.py --steps ${STEPS:-30} --warmup 5 --config ${CFG:-c2} --mode $m --no-cpu-baseline --json-out /tmp/b.json > /tmp/b.log 2>&1
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$m', '${CFG:-c2}', round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms', 'e2e', round(d['e2e']['value'],1))" 2>/dev/null || tail -3 /tmp/b.log
done
