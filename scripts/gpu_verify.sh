# full verification of the current tree: the GPU suite on the default build and on the
# bounds-checked build (-DSEEDS_CHECKED, scripts/alt_checked.so), smoke, the default bench line
cd $GRAFT_REPO_ROOT; O=gpurun_out/verify; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_default.log 2>&1; echo "exit $?" >> $O/pytest_default.log
SEEDS_LIB=scripts/alt_checked.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_checked.log 2>&1; echo "exit $?" >> $O/pytest_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --json-out $O/bench_default.json > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
