# chain trace of k_tile1 (tracing build) on c2 and c1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export SEEDS_LIB=scripts/alt_trace.so
for cfg in c2 c1; do timeout 120 python scripts/trace_t1.py $cfg 2>&1 | tail -12; done > gpurun_out/trace_t1b.txt 2>&1
