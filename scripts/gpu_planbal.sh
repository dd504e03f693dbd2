# SEEDS_PLAN_BAL=1: the plan score of multi-frame batches by the balanced assignment's busiest CTA; A/B on c3 / c4
O=gpurun_out/planbal; mkdir -p $O
for i in 1 2; do for c in c3 c4; do
  echo -n "default: "; CFG=$c STEPS=8 bash scripts/gpu_quick.sh
  echo -n "plan_bal: "; SEEDS_PLAN_BAL=1 CFG=$c STEPS=8 bash scripts/gpu_quick.sh
done; done > $O/ab.txt 2>&1
for c in c3 c4; do SEEDS_PLAN_BAL=1 SEEDS_PLAN_DEBUG=1 timeout 200 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --extra none 2>&1 | grep "seeds plan" | sort | uniq -c; done > $O/plans.txt 2>&1
SEEDS_PLAN_BAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
cat $O/ab.txt $O/plans.txt; tail -n 3 $O/pytest.log
