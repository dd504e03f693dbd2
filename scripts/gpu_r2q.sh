timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_bands.py tests/test_gpu_levels.py -q -x -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2q_pytest.log
ALTS="scripts/alt_prev.so" CFGS="c2 c3 c5" bash scripts/gpu_ab.sh > gpurun_out/r2q_ab.txt 2>&1
