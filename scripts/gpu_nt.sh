for nt in 512 128; do for cfg in c3 c5; do
  st=5; [ $cfg = c5 ] && st=3
  SEEDS_GRID_NT=$nt timeout 300 python bench.py --config $cfg --steps $st --warmup 2 --no-cpu-baseline --json-out /tmp/b.json > /tmp/b.log 2>&1
  python -c "import json;d=json.load(open('/tmp/b.json'));print('nt $nt', '$cfg', d['config']['grid_ctas'], d['config']['grid_tiles_per_frame'], round(d['value'],1),'Mpx/s', round(d['ms_per_step'],3),'ms')" || tail -3 /tmp/b.log
done; done
