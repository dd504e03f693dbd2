# per-phase trace of c2 (all sub-sweeps) and of a 32-frame c3 batch with the tracing build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export SEEDS_LIB=scripts/alt_trace.so
TRACE_S=0,16,48,64,70,99 timeout 120 python scripts/trace.py c2 grid > gpurun_out/trace_c2.txt 2>&1
NF=32 TRACE_S=0,64,70 timeout 120 python scripts/trace.py c3 grid > gpurun_out/trace_c3.txt 2>&1
