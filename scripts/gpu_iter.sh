# one iteration on a k_tile1 change: parity + fuzz suites, A/B against
# scripts/alt_prev.so on c2 / c1, and the chain trace (scripts/alt_trace.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "exit $?" >> gpurun_out/it_pytest.log
ALTS=scripts/alt_prev.so CFGS="c2 c1" bash scripts/gpu_ab.sh > gpurun_out/it_ab.txt 2>&1
TRACE_S=0,15,48,64,80,99 SEEDS_LIB=scripts/alt_trace.so timeout 120 python scripts/trace_t1.py c2 2>&1 | grep -v Warn | grep -v nanmean > gpurun_out/it_trace.txt 2>&1
