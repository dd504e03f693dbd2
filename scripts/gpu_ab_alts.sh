# parity + fuzz suites on each SEEDS_LIB build in $ALTS, then the A/B timing of
# the in-tree lib against them on $CFGS (scripts/gpu_ab.sh)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for a in $ALTS; do
  echo "== $a"; SEEDS_LIB=$a timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
done > gpurun_out/alts_pytest.log 2>&1
ALTS="$ALTS" CFGS="${CFGS:-c2 c1}" bash scripts/gpu_ab.sh > gpurun_out/alts_ab.txt 2>&1
