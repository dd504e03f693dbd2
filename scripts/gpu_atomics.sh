# L2 atomic / reduction traffic of one k_grid launch per config ("atomic/L2 throughput")
O=gpurun_out/atom; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum
for spec in "c2 auto 2 1" "c3 auto 2 256" "c4 auto 2 8" "c5 auto 2 1"; do
  set -- $spec
  timeout 900 $NCU --metrics $M --clock-control none -k regex:k_grid -s 1 -c 1 --csv python scripts/run_once.py $spec > $O/atom_$1.csv 2> $O/atom_$1.err
done
ls -la $O
