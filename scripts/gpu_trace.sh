mkdir -p gpurun_out
for m in ${MODES:-grid}; do timeout 120 python scripts/trace.py ${CFG:-c2} $m 2>&1 | tail -8; done
