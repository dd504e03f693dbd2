mkdir -p gpurun_out
timeout 120 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --show-backtrace no python scripts/run_once.py c1 grid 1 2>&1 | grep -v "^=========     " | head -40
