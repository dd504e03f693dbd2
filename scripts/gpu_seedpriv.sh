# privatised warm seed: warm-start tests, and c4 A/B against SEEDS_SEED_PRIV=0 (global atomics)
cd $GRAFT_REPO_ROOT; O=gpurun_out/sp; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_large.py tests/test_gpu_boundary.py tests/test_gpu_seed.py -x -q -k "warm or c4 or video or host or bad or init or fuzz or seed" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
ENVAB="SEEDS_SEED_PRIV=0" CFGS=c4 STEPS=10 bash scripts/gpu_envab.sh > $O/ab.txt 2>&1
