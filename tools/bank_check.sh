#!/bin/bash
# Shared-memory bank conflicts and time of chosen c64 passes under env variants (run under gpurun).
O=gpurun_out/$1; shift; mkdir -p $O
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread
for v in "$@"; do for p in ${PASSES:-7 10 13}; do
  env ${v/#-/} ncu --metrics $M --clock-control none -k regex:svpass -s $p -c 1 --csv python tools/run_plan.py --reps 2 2>/dev/null | grep -v "^==" | tail -7 | awk -F'","' -v v="$v" -v p=$p '{print v, "launch", p, $(NF-2), $NF}' >> $O/banks.txt
done; done
cat $O/banks.txt
