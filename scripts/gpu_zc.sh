# zero-copy single-frame host path: its tests, and the c2 / c1 e2e with it on and off
cd $GRAFT_REPO_ROOT; O=gpurun_out/zc; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for i in 1 2; do for z in 1 0; do for c in c2 c1; do echo -n "zero_copy=$z: "; SEEDS_ZERO_COPY=$z CFG=$c STEPS=30 bash scripts/gpu_quick.sh; done; done; done > $O/ab.txt 2>&1
