# tile planner sweep 2: SEEDS_TILE_COST x SEEDS_HALO_W on c3 / c5 / c4 (+ c2's plan)
cd $GRAFT_REPO_ROOT; O=gpurun_out/tc2; mkdir -p $O
for c in c3 c5 c4; do for tc in 300 1000; do for hw in 2 4 8 16; do
  rm -f /tmp/b.json
  SEEDS_PLAN_DEBUG=1 SEEDS_TILE_COST=$tc SEEDS_HALO_W=$hw timeout 200 python bench.py --steps 15 --warmup 3 --config $c --no-cpu-baseline --extra none --json-out /tmp/b.json > /tmp/b.log 2>&1
  echo "$c tc=$tc hw=$hw $(grep 'seeds plan' /tmp/b.log | grep 'nt=128\|nf=1 nt=512' | tail -1) $(python -c "import json;d=json.load(open('/tmp/b.json'));print(round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms')" 2>/dev/null || tail -2 /tmp/b.log)" >> $O/sweep.txt
done; done; done
for tc in 0 1000; do SEEDS_PLAN_DEBUG=1 SEEDS_TILE_COST=$tc timeout 200 python bench.py --steps 30 --warmup 3 --config c2 --no-cpu-baseline --extra none --json-out /tmp/b.json > /tmp/b.log 2>&1; echo "c2 tc=$tc $(grep 'seeds plan' /tmp/b.log | tail -1) $(python -c "import json;d=json.load(open('/tmp/b.json'));print(round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms')")" >> $O/sweep.txt; done
