# bench lines of the means post-processing (reading M1)
mkdir -p gpurun_out/means
for c in c2 c3 c5; do for m in 0 1 2; do
  st=20; [ $c != c2 ] && st=5
  timeout 300 python bench.py --config $c --steps $st --warmup 3 --means-iters $m --no-cpu-baseline --json-out gpurun_out/means/${c}_m$m.json > gpurun_out/means/${c}_m$m.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/means/${c}_m$m.json'));print('$c means $m', round(d['value'],1), 'Mpx/s', round(d['ms_per_step'],4), 'ms')" 2>/dev/null || tail -2 gpurun_out/means/${c}_m$m.log
done; done
