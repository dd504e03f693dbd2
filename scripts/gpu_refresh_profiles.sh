# Round-end evidence in dependency order: ncu captures first (launch list + one
# --set full capture of k_grid per config), profiles/ncu_traffic.json rebuilt from
# them on the box, then the bench lines (which pair their live timings with it).
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grid -s 3 -c 1 -o gpurun_out/prof/full_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c3 -f python scripts/run_once.py c3 auto 2 256 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c4 -f python scripts/run_once.py c4 auto 2 8 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o /tmp/full_c5 -f python scripts/run_once.py c5 auto 2 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof/full_c2.ncu-rep /tmp/full_c3.ncu-rep /tmp/full_c4.ncu-rep /tmp/full_c5.ncu-rep > gpurun_out/prof/ncu_full_summary.json
python scripts/make_traffic.py c2/grid=gpurun_out/prof/full_c2.ncu-rep c3/grid=/tmp/full_c3.ncu-rep c4/grid=/tmp/full_c4.ncu-rep c5/grid=/tmp/full_c5.ncu-rep
cp profiles/ncu_traffic.json gpurun_out/prof/ncu_traffic.json
for c in c2 c3 c4 c5; do
  f=/tmp/full_$c.ncu-rep; [ $c = c2 ] && f=gpurun_out/prof/full_c2.ncu-rep
  ncu -i $f --page details --csv > gpurun_out/prof/ncu_full_${c}_details.csv 2>/dev/null
done
timeout 300 python bench.py --steps 50 --warmup 5 --json-out gpurun_out/prof/bench_c2.json > gpurun_out/prof/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --json-out gpurun_out/prof/bench_$c.json > gpurun_out/prof/bench_$c.log 2>&1; done
ls -la gpurun_out/prof
