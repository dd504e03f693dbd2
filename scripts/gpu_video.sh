# seeds_video_host: its parity tests, the host-chunk sweep of c3's e2e, and the c4 / c3 bench lines
cd $GRAFT_REPO_ROOT; O=gpurun_out/video; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "video or host" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python scripts/e2e_chunks.py c3 1,2,4,8,16 > $O/chunks_c3.txt 2>&1
timeout 400 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench_c4.json > $O/bench_c4.log 2>&1
