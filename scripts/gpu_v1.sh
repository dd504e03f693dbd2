cd $GRAFT_REPO_ROOT; O=gpurun_out/v1; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_default.log 2>&1; echo "exit $?" >> $O/pytest_default.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --json-out $O/bench_default.json > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
