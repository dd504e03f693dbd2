# verification after the tile-cost planner: GPU suite, smoke, bench lines c2 (default, with extra c3/c5), c4,
# a launch list of c5, an ncu --set full capture of c5's k_grid and of c3's
cd $GRAFT_REPO_ROOT; O=gpurun_out/v2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_default.log 2>&1; echo "exit $?" >> $O/pytest_default.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --json-out $O/bench_c2.json > $O/bench_c2.log 2>&1; echo "exit $?" >> $O/bench_c2.log
for c in c3 c4 c5; do SEEDS_PLAN_DEBUG=1 timeout 600 python bench.py --config $c --json-out $O/bench_$c.json > $O/bench_$c.log 2>&1; echo "exit $?" >> $O/bench_$c.log; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --extra none > $O/ncu_launch_c5.log 2>&1
for c in c3 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grid -s 1 -c 1 -o /tmp/full_$c -f python scripts/run_once.py $c auto 2 $([ $c = c3 ] && echo 256) > $O/ncu_full_$c.log 2>&1
  ncu -i /tmp/full_$c.ncu-rep --page details --csv > $O/ncu_full_${c}_details.csv 2>/dev/null
  ncu -i /tmp/full_$c.ncu-rep --page raw --csv > $O/ncu_full_${c}_raw.csv 2>/dev/null
done
python scripts/ncu_summary.py /tmp/full_c3.ncu-rep /tmp/full_c5.ncu-rep > $O/ncu_full_summary.json 2>&1
