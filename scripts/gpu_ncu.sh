# usage: CFG=c2 MODE=grid KREGEX=k_grid bash scripts/gpu_ncu.sh
mkdir -p gpurun_out
CFG=${CFG:-c2}; MODE=${MODE:-grid}; KREGEX=${KREGEX:-k_grid}; NAME=${NAME:-${MODE}_${CFG}}
python scripts/run_once.py $CFG $MODE 2 ${NFR:-1} > /dev/null && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KREGEX -s ${SKIP:-1} -c 1 -o gpurun_out/$NAME -f python scripts/run_once.py $CFG $MODE 2 ${NFR:-1} > gpurun_out/ncu_$NAME.log 2>&1; tail -3 gpurun_out/ncu_$NAME.log
