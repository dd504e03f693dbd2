cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
for i in 1 2; do
  for c in ${CFGS:-c2 c5}; do echo -n "cur: "; CFG=$c STEPS=${STEPS:-10} bash scripts/gpu_quick.sh; done
  for c in ${CFGS:-c2 c5}; do echo -n "min4: "; SEEDS_GW_MIN=4 CFG=$c STEPS=${STEPS:-10} bash scripts/gpu_quick.sh; done
  cp $ALT paper_1309_3848_b200/libseeds.so
  for c in ${CFGS:-c2 c5}; do echo -n "alt: "; CFG=$c STEPS=${STEPS:-10} bash scripts/gpu_quick.sh; done
  cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
done
