timeout 600 python -m pytest tests/test_gpu_seed.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2g_pytest.log
for i in 1 2; do for c in "c2" "c3 256" "c4 8" "c5"; do python scripts/seed_time.py $c; SEEDS_LIB=scripts/alt_pred.so python scripts/seed_time.py $c; done; done > gpurun_out/r2g_seed.txt 2>&1
ALTS="scripts/alt_pred.so" CFGS="c2 c3 c5" bash scripts/gpu_ab.sh > gpurun_out/r2g_ab.txt 2>&1
