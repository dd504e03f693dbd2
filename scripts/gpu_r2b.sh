mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k5.py tests/test_gpu_boundary.py -q -rs -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2b_pytest.log
for alt in scripts/alt_acq0.so scripts/alt_acq2.so; do echo "== ALT $alt"; ALT=$alt CFGS="c2 c3" STEPS=30 bash scripts/gpu_ab3.sh; done > gpurun_out/r2b_ab_barrier.txt 2>&1
TMO=400 bash scripts/gpu_sanitize.sh
