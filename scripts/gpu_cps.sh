# 128-thread plans at fewer CTAs per SM (more shared memory per CTA, larger tiles): SEEDS_SMALL_CPS, and the 512-thread plan
cd $GRAFT_REPO_ROOT; O=gpurun_out/cps; mkdir -p $O
for c in c5 c3 c4; do for v in "SEEDS_SMALL_CPS=4" "SEEDS_SMALL_CPS=3" "SEEDS_SMALL_CPS=2" "SEEDS_GRID_NT=512" "SEEDS_TILE_COST=4000 SEEDS_SMALL_CPS=3"; do
  rm -f /tmp/b.json
  env $v SEEDS_PLAN_DEBUG=1 timeout 200 python bench.py --steps 15 --warmup 3 --config $c --no-cpu-baseline --extra none --json-out /tmp/b.json > /tmp/b.log 2>&1
  echo "$c $v $(grep 'seeds plan' /tmp/b.log | grep -v 'nf=1 nt=512 G=14[0-9] tiles=14[0-9] ' | tail -1) $(python -c "import json;d=json.load(open('/tmp/b.json'));print(round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms')" 2>/dev/null || tail -2 /tmp/b.log)" >> $O/sweep.txt
done; done
