#!/bin/bash
# Scatter-add memory-system evidence (north_star): DRAM bytes, L2 reduction
# (red.global.add) sector and hit counts, atomics, per config.  One steady-state k_fuse
# launch per config (the warm-up job's launches are skipped).  Usage: tools/ncu_red.sh OUTDIR
out=${1:-gpurun_out}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,\
lts__t_sectors_op_red.sum,lts__t_sectors_op_red_lookup_hit.sum,lts__t_sector_op_red_hit_rate.pct,\
lts__t_requests_op_atom.sum,lts__t_requests_op_atom_lookup_hit.sum,\
l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum
for cfg in "cfg2 10" "cfg4 10" "cfg5 20"; do
  set -- $cfg
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_fuse -s $2 -c 1 --csv \
    python tools/bench_configs.py $1 > "$out/ncu_red_$1.csv" 2> "$out/ncu_red_$1.err"
  echo "$1 rc=$?"
done
