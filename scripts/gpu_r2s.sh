timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -k "band or budget" -p no:cacheprovider -rs > gpurun_out/r2s_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2s_pytest.log
