# c1 / c2: fewer, larger single tiles (SEEDS_GRID_CTAS caps the CTAs; cheaper grid barrier vs longer per-CTA chains)
cd $GRAFT_REPO_ROOT; O=gpurun_out/c2ctas; mkdir -p $O
for i in 1 2; do for c in c2 c1; do for n in 148 136 100 72 50 36; do
  rm -f /tmp/b.json
  SEEDS_GRID_CTAS=$n SEEDS_PLAN_DEBUG=1 timeout 200 python bench.py --steps 40 --warmup 5 --config $c --no-cpu-baseline --extra none --json-out /tmp/b.json > /tmp/b.log 2>&1
  echo "$c ctas<=$n $(grep 'seeds plan' /tmp/b.log | tail -1 | sed 's/seeds plan: //') $(python -c "import json;d=json.load(open('/tmp/b.json'));c=d['config'];print(c['refine_kernel'],c['grid_ctas'],round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms')" 2>/dev/null || tail -2 /tmp/b.log)" >> $O/sweep.txt
done; done; done
