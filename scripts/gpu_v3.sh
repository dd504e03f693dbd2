# late round 2: the bounds-checked build's GPU suite on the tile-cost plans, c5 4-band and c4 video bench lines
cd $GRAFT_REPO_ROOT; O=gpurun_out/v3; mkdir -p $O
SEEDS_LIB=scripts/alt_checked.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_checked.log 2>&1; echo "exit $?" >> $O/pytest_checked.log
timeout 600 python bench.py --config c5 --bands 4 --no-cpu-baseline --json-out $O/bench_c5_bands4.json > $O/bench_c5_bands4.log 2>&1; echo "exit $?" >> $O/bench_c5_bands4.log
timeout 600 python bench.py --config c1 --no-cpu-baseline --json-out $O/bench_c1.json > $O/bench_c1.log 2>&1; echo "exit $?" >> $O/bench_c1.log
