# A/B/C: current lib vs $ALTS (space separated) over CFGS, 2 rounds
cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
for i in 1 2; do
  for c in ${CFGS:-c2}; do
    cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so; echo -n "cur: "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
    for a in $ALTS; do cp $a paper_1309_3848_b200/libseeds.so; echo -n "$(basename $a): "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh; done
  done
done
cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
