# per-phase trace of c2 / c1 with the tracing build: k_tile1 (default) and k_grid (SEEDS_TILE1=0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export SEEDS_LIB=scripts/alt_trace.so
for cfg in c2 c1; do
echo "== $cfg tile1"; TRACE_S=0,16,48,64,70,99 timeout 120 python scripts/trace.py $cfg grid 2>&1 | tail -14
echo "== $cfg grid"; SEEDS_TILE1=0 timeout 120 python scripts/trace.py $cfg grid 2>&1 | tail -7
done > gpurun_out/trace_t1.txt 2>&1
