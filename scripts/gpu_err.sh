# the host paths with the page-locked error word: their tests (incl. bad warm-start labels) and e2e A/B vs alt_head
cd $GRAFT_REPO_ROOT; O=gpurun_out/err; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_large.py -x -q -k "host or boundary or bad or estate or video" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
ALTS=scripts/alt_head.so CFGS="c2 c1" bash scripts/gpu_ab.sh > $O/ab.txt 2>&1
