# Final check of the round's last tree: the GPU suite on the bounds-checked build (seed kernels included) and on
# the default build, smoke, the default bench line (c2 with its extra map) and the c3 / c4 / c5 lines.
O=gpurun_out/final_head; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt 2>&1
[ -n "$SKIP_CHECKED" ] || { SEEDS_LIB=scripts/alt_checked.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_checked.log 2>&1; echo "exit $?" >> $O/pytest_checked.log; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_default.log 2>&1; echo "exit $?" >> $O/pytest_default.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --json-out $O/bench_default.json > $O/bench_default.log 2>&1
for c in c3 c4 c5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --json-out $O/bench_$c.json > $O/bench_$c.log 2>&1; done
tail -n 3 $O/pytest_checked.log 2>/dev/null; tail -n 3 $O/pytest_default.log; cat $O/smoke.log
