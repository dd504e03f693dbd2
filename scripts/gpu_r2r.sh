SEEDS_LIB=scripts/alt_cps6.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_large.py -q -p no:cacheprovider > gpurun_out/r2r_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2r_pytest.log
ALTS="scripts/alt_cps6.so" CFGS="c3 c4 c5" bash scripts/gpu_ab.sh > gpurun_out/r2r_ab.txt 2>&1
