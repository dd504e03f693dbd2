# A/B: the current libseeds.so vs $ALT (same box, alternating)
cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
md5sum paper_1309_3848_b200/libseeds.so $ALT
for i in 1 2; do
  cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so; echo -n "cur: "; bash scripts/gpu_quick.sh
  cp $ALT paper_1309_3848_b200/libseeds.so; echo -n "alt: "; bash scripts/gpu_quick.sh
done
cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
