# a tracing build of libseeds.so (per-CTA clock64 stamps, seeds_debug_trace) at scripts/alt_trace.so;
# use with SEEDS_LIB=scripts/alt_trace.so python scripts/trace.py ...
cp paper_1309_3848_b200/libseeds.so /tmp/lib_keep.so
SEEDS_NVCC_EXTRA="-DSEEDS_TRACE" python -c "from paper_1309_3848_b200 import build; build.build(force=True)"
cp paper_1309_3848_b200/libseeds.so scripts/alt_trace.so
cp /tmp/lib_keep.so paper_1309_3848_b200/libseeds.so
git checkout paper_1309_3848_b200/ptxas_info.txt 2>/dev/null
touch paper_1309_3848_b200/libseeds.so
