timeout 900 python -m pytest tests/test_gpu_seed.py tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_fuzz.py tests/test_gpu_means.py tests/test_gpu_compact.py tests/test_gpu_levels.py tests/test_gpu_lab.py -q -x -p no:cacheprovider > gpurun_out/r2h_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2h_pytest.log
for c in "c2" "c3 256" "c4 8" "c5"; do python scripts/seed_time.py $c; done > gpurun_out/r2h_seed.txt 2>&1
ALTS="scripts/alt_pred.so" CFGS="c2 c3 c4 c5" bash scripts/gpu_ab.sh > gpurun_out/r2h_ab.txt 2>&1
