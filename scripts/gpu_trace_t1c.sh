cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SEEDS_LIB=scripts/alt_trace.so timeout 120 python scripts/trace_t1.py c2 2>&1 | grep -v Warn | grep -v nanmean > gpurun_out/trace_t1c.txt 2>&1
