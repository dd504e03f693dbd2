# per-tile cost term of the tile planner (SEEDS_TILE_COST, pixel equivalents): plans and bench lines on c3 / c4 / c5
cd $GRAFT_REPO_ROOT; O=gpurun_out/tc; mkdir -p $O
for i in 1 2; do for c in c3 c5 c4; do for tc in 0 1000 3000 8000 20000; do
  rm -f /tmp/b.json
  SEEDS_PLAN_DEBUG=1 SEEDS_TILE_COST=$tc timeout 200 python bench.py --steps 15 --warmup 3 --config $c --no-cpu-baseline --extra none --json-out /tmp/b.json > /tmp/b.log 2>&1
  echo "$c tc=$tc $(grep 'seeds plan' /tmp/b.log | grep 'nt=128\|nf=1 nt=512' | tail -1) $(python -c "import json;d=json.load(open('/tmp/b.json'));print(round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms')" 2>/dev/null || tail -2 /tmp/b.log)" >> $O/sweep.txt
done; done; done
