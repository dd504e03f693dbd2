mkdir -p gpurun_out
python scripts/run_once.py c2 resident 2 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_resident -s 1 -c 1 -o gpurun_out/res_c2 -f python scripts/run_once.py c2 resident 2 > gpurun_out/ncu_res.log 2>&1; tail -5 gpurun_out/ncu_res.log
