# k_seed_cells word path (cold, C = 3, W % 4 == 0): GPU suite, A/B vs SEEDS_SEED_VEC=0 on c5 / c4, c5 launch list
cd $GRAFT_REPO_ROOT; O=gpurun_out/sv; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
ENVAB="SEEDS_SEED_VEC=0" CFGS="c5 c4" STEPS=20 bash scripts/gpu_envab.sh > $O/ab.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --extra none > $O/ncu_launch_c5.log 2>&1
