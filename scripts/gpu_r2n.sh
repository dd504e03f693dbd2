timeout 900 python -m pytest tests/test_gpu_seed.py tests/test_gpu_parity.py tests/test_bands.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2n_pytest.log
for c in "c2" "c3 256" "c4 8" "c5"; do python scripts/kinds.py $c; done > gpurun_out/r2n_kinds.txt 2>&1
for c in c2 c3 c4 c5; do CFG=$c bash scripts/gpu_quick.sh; done > gpurun_out/r2n_quick.txt 2>&1
