# Checkpoint of the current tree: the whole GPU suite, smoke, the default bench
# line, and ncu (launch list + --set full with source) of c2's k_tile1.
O=gpurun_out/ckpt; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 30 --warmup 5 --json-out $O/bench_c2.json > $O/bench_c2.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_tile1 -s 3 -c 1 -o $O/full_c2_t1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > $O/ncu.log 2>&1
python scripts/ncu_sass_lines.py $O/full_c2_t1.ncu-rep 60 > $O/stall_lines_c2_t1.txt 2>&1
$NCU -i $O/full_c2_t1.ncu-rep --page details --csv > $O/details_c2_t1.csv 2>/dev/null
$NCU -i $O/full_c2_t1.ncu-rep --page raw --csv > $O/raw_c2_t1.csv 2>/dev/null
ls -la $O
