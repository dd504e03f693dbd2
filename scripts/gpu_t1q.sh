# quick k_tile1 check: c1/c2 parity + fuzz, then c2/c1 bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/t1_pytest.log 2>&1; echo "exit $?" >> gpurun_out/t1_pytest.log
for cfg in c2 c1 c2; do
  rm -f /tmp/b.json
  timeout 120 python bench.py --steps 30 --warmup 5 --config $cfg --no-cpu-baseline --json-out /tmp/b.json > /tmp/b.log 2>&1
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$cfg', round(d['value'],1),'Mpx/s', round(d['ms_per_step'],4),'ms', d.get('kernels',{}))" 2>/dev/null || tail -3 /tmp/b.log
done > gpurun_out/t1_bench.txt 2>&1
