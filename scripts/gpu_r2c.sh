# round 2: A/B vs the round-1 tree, c2 trace, ncu source-level captures of c2 and c3 (16 frames)
mkdir -p gpurun_out/r2c
for i in 1 2; do
  for c in c2 c3; do
    echo -n "r2 $c: "; CFG=$c STEPS=30 bash scripts/gpu_quick.sh
    (cd scripts/r1tree && cp ../../MEASURED_PEAKS.json . 2>/dev/null; echo -n "r1 $c: "; CFG=$c STEPS=30 bash ../gpu_quick.sh)
  done
done > gpurun_out/r2c/ab_r1.txt 2>&1
python scripts/trace.py c2 grid > gpurun_out/r2c/trace_c2.txt 2>&1
NF=16 python scripts/trace.py c3 grid > gpurun_out/r2c/trace_c3x16.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_grid -c 1 -o gpurun_out/r2c/ncu_c2 python scripts/run_once.py c2 grid 2 1 > gpurun_out/r2c/ncu_c2.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none -k regex:k_grid -c 1 -o gpurun_out/r2c/ncu_c3x16 python scripts/run_once.py c3 grid 2 16 > gpurun_out/r2c/ncu_c3.log 2>&1
ls -la gpurun_out/r2c
