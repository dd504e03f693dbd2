timeout 600 python -m pytest tests -m gpu -x -q -k "grid or large or modes" 2>&1 | tail -3
MODES=auto bash scripts/gpu_bench_all.sh
