# k_seed_warm (word-path warm seed): new seed tests, GPU suite, c4 A/B vs SEEDS_WARM_VEC=0, c4 launch list
cd $GRAFT_REPO_ROOT; O=gpurun_out/wv; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_seed.py tests/test_gpu_boundary.py -x -q > $O/pytest_seed.log 2>&1; echo "exit $?" >> $O/pytest_seed.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
ENVAB="SEEDS_WARM_VEC=0" CFGS="c4" STEPS=20 bash scripts/gpu_envab.sh > $O/ab.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --extra none > $O/ncu_launch_c4.log 2>&1
