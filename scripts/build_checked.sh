# a bounds-checked build of libseeds.so (-DSEEDS_CHECKED: range checks that trap) at scripts/alt_checked.so;
# run the GPU suite with SEEDS_LIB=scripts/alt_checked.so
cp paper_1309_3848_b200/libseeds.so /tmp/lib_keep.so
SEEDS_NVCC_EXTRA="-DSEEDS_CHECKED" python -c "from paper_1309_3848_b200 import build; build.build(force=True)"
cp paper_1309_3848_b200/libseeds.so scripts/alt_checked.so
cp /tmp/lib_keep.so paper_1309_3848_b200/libseeds.so
git checkout paper_1309_3848_b200/ptxas_info.txt 2>/dev/null
touch paper_1309_3848_b200/libseeds.so
