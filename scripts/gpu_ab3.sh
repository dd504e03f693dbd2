# A/B: current libseeds.so vs $ALT over CFGS (same box, alternating)
cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
for i in 1 2; do
  for c in ${CFGS:-c2}; do
    cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so; echo -n "cur: "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
    cp $ALT paper_1309_3848_b200/libseeds.so; echo -n "alt: "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
  done
done
cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
