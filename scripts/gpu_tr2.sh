# trace of the current lib and of $ALT (c2 by default)
cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
echo "== cur"; SEEDS_GW_ITERS=${ITERS:-1} timeout 60 python scripts/trace.py ${CFG:-c2} grid 2>&1 | tail -6
cp $ALT paper_1309_3848_b200/libseeds.so
echo "== alt"; timeout 60 python scripts/trace.py ${CFG:-c2} grid 2>&1 | tail -6
cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
