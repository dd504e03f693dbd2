# A/B: the in-tree libseeds.so vs each SEEDS_LIB alternative in $ALTS over $CFGS, alternating twice
for i in 1 2; do
  for c in ${CFGS:-c2}; do
    echo -n "cur: "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
    for a in $ALTS; do echo -n "$(basename $a): "; SEEDS_LIB=$a CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh; done
  done
done
