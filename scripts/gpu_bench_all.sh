mkdir -p gpurun_out/bench
for cfg in c2 c3 c4 c5; do
  for m in ${MODES:-auto graph}; do
    st=30; [ $cfg = c3 ] && st=5; [ $cfg = c4 ] && st=3; [ $cfg = c5 ] && st=3
    timeout 400 python bench.py --config $cfg --mode $m --steps $st --warmup 3 --cpu-budget 10 --json-out gpurun_out/bench/${cfg}_${m}.json > gpurun_out/bench/${cfg}_${m}.log 2>&1
    python -c "import json;d=json.load(open('gpurun_out/bench/${cfg}_${m}.json'));print('$cfg', '$m', d['config']['exec_mode'], round(d['value'],1),'Mpx/s', round(d['ms_per_step'],3),'ms/step', 'e2e', round(d['e2e']['value'],1), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'] or 0,4), 'cpu', round(d.get('cpu_baseline',{}).get('value',0),2))" 2>/dev/null || tail -3 gpurun_out/bench/${cfg}_${m}.log
  done
done
