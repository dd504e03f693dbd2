mkdir -p gpurun_out/prof
timeout 300 python bench.py --steps 30 --warmup 5 --json-out gpurun_out/prof/bench_c2.json > gpurun_out/prof/bench_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grid -s 3 -c 1 -o gpurun_out/prof/full_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o gpurun_out/prof/full_c3 -f python scripts/run_once.py c3 auto 2 256 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o gpurun_out/prof/full_c4 -f python scripts/run_once.py c4 auto 2 8 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grid -s 1 -c 1 -o gpurun_out/prof/full_c5 -f python scripts/run_once.py c5 auto 2 > /dev/null 2>&1
ls -la gpurun_out/prof
