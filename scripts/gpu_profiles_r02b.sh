# Round-2 final evidence (profiles/r02/): the whole GPU suite and smoke, bench lines
# (c2 with its extra map, c3-c5, c5 in 4 bands, the reference arm), the ncu launch list of
# the default bench command, ncu --set full of k_tile1 (c2, with source) and of k_grid
# (c3-c5), summaries, ncu_traffic.json.
O=gpurun_out/prof3; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_default.log 2>&1; echo "exit $?" >> $O/pytest_default.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_tile1 -s 3 -c 1 -o $O/full_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > /dev/null 2>&1
timeout 1200 $NCU --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c3 -f python scripts/run_once.py c3 auto 2 256 > /dev/null 2>&1
timeout 1200 $NCU --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c4 -f python scripts/run_once.py c4 auto 2 8 > /dev/null 2>&1
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c5 -f python scripts/run_once.py c5 auto 2 > /dev/null 2>&1
python scripts/ncu_summary.py $O/full_c2.ncu-rep /tmp/full_c3.ncu-rep /tmp/full_c4.ncu-rep /tmp/full_c5.ncu-rep > $O/ncu_full_summary.json
for c in c2 c3 c4 c5; do
  f=/tmp/full_$c.ncu-rep; [ $c = c2 ] && f=$O/full_c2.ncu-rep
  $NCU -i $f --page details --csv > $O/ncu_full_${c}_details.csv 2>/dev/null
done
python scripts/make_traffic.py c2/grid=$O/full_c2.ncu-rep c3/grid=/tmp/full_c3.ncu-rep c4/grid=/tmp/full_c4.ncu-rep c5/grid=/tmp/full_c5.ncu-rep > $O/traffic.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python scripts/ncu_sass_lines.py $O/full_c2.ncu-rep 40 > $O/ncu_c2_stall_lines.txt 2>&1
python scripts/ncu_sass_lines.py /tmp/full_c5.ncu-rep 40 > $O/ncu_c5_stall_lines.txt 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > /dev/null 2>&1
# bench lines last (they read profiles/ncu_traffic.json, just rebuilt)
timeout 600 python bench.py --steps 30 --warmup 5 --json-out $O/bench_c2.json > $O/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --json-out $O/bench_$c.json > $O/bench_$c.log 2>&1; done
timeout 400 python bench.py --config c5 --bands 4 --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench_c5_bands4.json > $O/bench_c5_bands4.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c2_reference.json 2> $O/bench_c2_reference.log
rm -f $O/full_c2.ncu-rep.bak
ls -la $O
