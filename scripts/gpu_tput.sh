for cfg in c3 c4 c5; do
  st=5; [ $cfg = c4 ] && st=3; [ $cfg = c5 ] && st=3
  timeout 300 python bench.py --config $cfg --steps $st --warmup 2 --no-cpu-baseline --json-out /tmp/b.json > /tmp/b.log 2>&1 && \
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg', d['config']['grid_ctas'], round(d['value'],1),'Mpx/s', round(d['ms_per_step'],3),'ms')" || tail -3 /tmp/b.log
done
