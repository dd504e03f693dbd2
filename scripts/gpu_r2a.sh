# round 2, first box run: full GPU suite, c2 bench, barrier A/B (acquire fence vs relaxed)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2a_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err
ALT=scripts/alt_relaxed.so CFGS="c2 c3" STEPS=30 bash scripts/gpu_ab3.sh > gpurun_out/r2a_ab_barrier.txt 2>&1
