# k_tile1: full GPU suite, c2/c1 bench lines (k_tile1, unfused seed, k_grid), phase trace
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/t1_pytest.log
( for i in 1 2; do
  echo -n "tile1: "; CFG=c2 bash scripts/gpu_quick.sh
  echo -n "tile1 c1: "; CFG=c1 bash scripts/gpu_quick.sh
  echo -n "unfused seed: "; SEEDS_TILE1_SEED=0 CFG=c2 bash scripts/gpu_quick.sh
  done
  echo -n "k_grid: "; SEEDS_TILE1=0 CFG=c2 bash scripts/gpu_quick.sh ) > gpurun_out/t1_ab.txt 2>&1
SEEDS_LIB=scripts/alt_trace.so timeout 120 python scripts/trace.py c2 grid > gpurun_out/trace_t1.txt 2>&1
