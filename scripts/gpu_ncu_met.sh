mkdir -p gpurun_out/metrics
timeout 300 python scripts/metrics_bench.py c5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_met_count -c 1 -o gpurun_out/metrics/met_c5 python scripts/metrics_bench.py c5 > gpurun_out/metrics/ncu.log 2>&1
tail -3 gpurun_out/metrics/ncu.log
