cp paper_1309_3848_b200/libseeds.so /tmp/lib_cur.so
for i in 1 2; do
  for it in ${ITERS:-1 2}; do for c in ${CFGS:-c2 c5}; do echo -n "iters $it: "; SEEDS_GW_ITERS=$it CFG=$c STEPS=${STEPS:-10} bash scripts/gpu_quick.sh; done; done
  cp $ALT paper_1309_3848_b200/libseeds.so
  for c in ${CFGS:-c2 c5}; do echo -n "alt: "; CFG=$c STEPS=${STEPS:-10} bash scripts/gpu_quick.sh; done
  cp /tmp/lib_cur.so paper_1309_3848_b200/libseeds.so
done
