# A/B of the in-tree lib against scripts/alt_prev.so on c2 / c1 (+ the parity / fuzz suites)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/t1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/t1_pytest.log
ALTS=scripts/alt_prev.so CFGS="c2 c1" bash scripts/gpu_ab.sh > gpurun_out/t1_ab.txt 2>&1
