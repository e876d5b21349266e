# key raw metrics + per-phase instruction/stall split of one kernel in a report
# usage: bash tools/ncu_kern.sh REPORT KERNEL_REGEX
timeout 300 ncu -i $1 --page raw --csv -k regex:$2 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum','lts__t_sectors_op_atom.sum','lts__t_sectors_op_red.sum']
for r in rows[2:]:
  for w in want:
    if w in h: print('  %-62s %s' % (w, r[h.index(w)]))
"
