# run the GPU tests with $ALT swapped in, then A/B benches
cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
cp $ALT paper_1309_3848_b200/libseeds.so
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -x -k "${TK:-grid or large or c4 or c5 or multi}" 2>&1 | tail -3
cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
CFGS="${CFGS:-c3 c4 c5}" STEPS=5 bash scripts/gpu_ab3.sh
