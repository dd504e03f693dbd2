# Balanced tile assignment (SEEDS_TILE_BALANCE, the planner's table order): the plan lines,
# A/B against frame order on c3 / c5 / c4, then the whole GPU suite on the new assignment.
O=gpurun_out/balance; mkdir -p $O
for c in c3 c5 c4; do
  SEEDS_PLAN_DEBUG=1 timeout 200 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --extra none 2>&1 | grep "seeds plan" | sort | uniq -c > $O/plan_$c.txt
done
ENVAB="SEEDS_TILE_BALANCE=0" CFGS="c3 c5 c4" STEPS=8 bash scripts/gpu_envab.sh > $O/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for c in c3 c4 c5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --json-out $O/bench_$c.json > $O/bench_$c.log 2>&1; done
timeout 600 python bench.py --steps 30 --warmup 5 --json-out $O/bench_c2.json > $O/bench_c2.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c3b -f python scripts/run_once.py c3 auto 2 256 > /dev/null 2>&1
$NCU -i /tmp/full_c3b.ncu-rep --page details --csv > $O/ncu_full_c3_details.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/full_c3b.ncu-rep > $O/ncu_full_summary_c3.json 2>/dev/null
tail -3 $O/pytest.log; cat $O/ab.txt; cat $O/plan_*.txt
