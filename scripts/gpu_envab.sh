# A/B of an environment switch: ENVAB="SEEDS_X=0" CFGS="c2 c3"
for i in 1 2; do for c in ${CFGS:-c2}; do
  echo -n "cur: "; CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
  echo -n "$ENVAB: "; env $ENVAB CFG=$c STEPS=${STEPS:-30} bash scripts/gpu_quick.sh
done; done
