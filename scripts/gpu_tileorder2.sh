# Tile-order experiment 2: the default interleave (every G-th tile) over a column-major walk (C) or a walk by
# panels of n tile columns (P<n>) -- the simultaneous tiles form a tall block instead of a full-width stripe.
O=gpurun_out/tileorder2; mkdir -p $O
for i in 1 2; do for c in c5 c4; do
  echo -n "default: "; CFG=$c STEPS=8 bash scripts/gpu_quick.sh
  for o in C P4 P8 P16 P24 P36; do echo -n "$o: "; SEEDS_TILE_ORDER=$o CFG=$c STEPS=8 bash scripts/gpu_quick.sh; done
done; done > $O/ab.txt 2>&1
SEEDS_TILE_ORDER=P8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > $O/pytest_P8.log 2>&1; echo "exit $?" >> $O/pytest_P8.log
cat $O/ab.txt; tail -n 3 $O/pytest_P8.log
