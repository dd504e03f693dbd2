# k_tile1 iteration: parity + fuzz + warm/seed tests, A/B against scripts/alt_head.so (c2, c1), chain trace and spread
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_seed.py tests/test_gpu_boundary.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "exit $?" >> gpurun_out/it_pytest.log
ALTS=scripts/alt_head.so CFGS="c2 c1" bash scripts/gpu_ab.sh > gpurun_out/it_ab.txt 2>&1
SEEDS_LIB=scripts/alt_trace.so timeout 200 python scripts/trace_t1.py c2 2>&1 | grep -v Warn | grep -v nanmean > gpurun_out/it_trace.txt 2>&1
SEEDS_LIB=scripts/alt_trace.so timeout 200 python scripts/trace_skew.py c2 >> gpurun_out/it_trace.txt 2>&1
