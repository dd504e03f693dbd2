# c3: the balanced assignment under other per-tile costs (the plan itself is the same for 300-20000)
O=gpurun_out/balcost; mkdir -p $O
for i in 1 2; do for tc in 1000 0 2000 4000 8000 16000; do
  echo -n "tile_cost=$tc: "; SEEDS_TILE_COST=$tc CFG=c3 STEPS=8 bash scripts/gpu_quick.sh
done; done > $O/ab.txt 2>&1
for tc in 0 4000 16000; do SEEDS_TILE_COST=$tc SEEDS_PLAN_DEBUG=1 timeout 200 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --extra none 2>&1 | grep "seeds plan" | grep -v nt=512 | sort | uniq -c | head -4; done > $O/plans.txt 2>&1
cat $O/ab.txt $O/plans.txt
