# ncu --set full (with source) of k_tile1 on c2 and its stall lines
O=gpurun_out/t1prof; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_tile1 -s 3 -c 1 -o $O/full_c2_t1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > $O/ncu.log 2>&1
python scripts/ncu_sass_lines.py $O/full_c2_t1.ncu-rep 60 > $O/stall_lines_c2_t1.txt 2>&1
$NCU -i $O/full_c2_t1.ncu-rep --page details --csv > $O/details_c2_t1.csv 2>/dev/null
