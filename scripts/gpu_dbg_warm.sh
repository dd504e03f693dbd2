cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( echo "== new, isolated"; timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "warm_start" 2>&1 | tail -3
  echo "== head"; SEEDS_LIB=scripts/alt_head.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
  echo "== new, checked, whole file"; SEEDS_LIB=scripts/alt_checked_new.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|FAILED|Error" | head -5
  echo "== new, whole file"; timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|FAILED" | head -5
) > gpurun_out/dbg_warm.txt 2>&1
