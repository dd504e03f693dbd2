timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2i_pytest.log
for c in "c2" "c3 256" "c4 8" "c5"; do python scripts/kinds.py $c; done > gpurun_out/r2i_kinds.txt 2>&1
ALTS="scripts/alt_pred.so" CFGS="c2 c3 c4 c5" bash scripts/gpu_ab.sh > gpurun_out/r2i_ab.txt 2>&1
