#!/bin/sh
# Ordering sweep (BASELINE config 5) on every bench graph + SpMV locality counters.
# usage: sh tools/order_sweep_all.sh TAG   -> gpurun_out/sweep_TAG_*.json / *.csv
set -e
tag=${1:-r02}
mkdir -p gpurun_out
for g in "rmat 22" "rmat 24" "rmat 26" "grid 4096"; do
  set -- $g
  python tools/order_sweep.py $1 $2 > gpurun_out/sweep_${tag}_$1_$2.json
  ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum \
      --clock-control none -k regex:k_spmv_merge -s 33 -c 3 --csv \
      --log-file gpurun_out/sweep_${tag}_ncu_$1_$2.csv python tools/order_sweep.py $1 $2 --ncu > /dev/null
done
