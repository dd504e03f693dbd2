timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2m_pytest.log
ENVAB="SEEDS_PQUAD=0" CFGS="c1 c2" bash scripts/gpu_envab.sh > gpurun_out/r2m_ab.txt 2>&1
SEEDS_LIB=scripts/alt_trace.so python scripts/trace.py c2 grid > gpurun_out/r2m_trace_c2.txt 2>&1
