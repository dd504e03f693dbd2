# ncu launch lists (kernel durations) of the c4 and c3 bench commands
cd $GRAFT_REPO_ROOT; O=gpurun_out/ll; mkdir -p $O
for c in c4 c3; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --extra none > $O/ncu_launch_$c.log 2>&1
done
