# k_tile1 (fused seed + emit): full GPU suite, then A/B against the relaxed-poll build and the unfused seed
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/t1_pytest.log
( ALTS=scripts/alt_relaxed.so CFGS="c2 c1" bash scripts/gpu_ab.sh
  echo -n "unfused seed: "; SEEDS_TILE1_SEED=0 CFG=c2 bash scripts/gpu_quick.sh
  echo -n "k_grid: "; SEEDS_TILE1=0 CFG=c2 bash scripts/gpu_quick.sh ) > gpurun_out/t1_ab.txt 2>&1
