# Tile-order experiment (SEEDS_TILE_ORDER=rows / cols: a contiguous run of tiles per CTA) against the
# default (every G-th tile, balanced for multi-frame batches); parity of the experiment orders on the
# multi-tile tests.
O=gpurun_out/tileorder; mkdir -p $O
for i in 1 2; do for c in c5 c3 c4; do
  echo -n "default: "; CFG=$c STEPS=8 bash scripts/gpu_quick.sh
  echo -n "rows: "; SEEDS_TILE_ORDER=rows CFG=$c STEPS=8 bash scripts/gpu_quick.sh
  echo -n "cols: "; SEEDS_TILE_ORDER=cols CFG=$c STEPS=8 bash scripts/gpu_quick.sh
  echo -n "rows, no balance: "; SEEDS_TILE_BALANCE=0 SEEDS_TILE_ORDER=rows CFG=$c STEPS=8 bash scripts/gpu_quick.sh
done; done > $O/ab.txt 2>&1
SEEDS_TILE_ORDER=cols timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > $O/pytest_cols.log 2>&1; echo "exit $?" >> $O/pytest_cols.log
SEEDS_TILE_ORDER=rows timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_rows.log 2>&1; echo "exit $?" >> $O/pytest_rows.log
cat $O/ab.txt; tail -2 $O/pytest_cols.log $O/pytest_rows.log
