#!/bin/bash
# DRAM bytes of the pair (4,5) kernel vs block size: does the second pass read from L2?
O=gpurun_out/${1:-pair_l2}
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for w in 0.02 0.1 0.5 1; do
  SV_PAIR_LOOK=1 SV_PAIR_WAVES=$w timeout 300 ncu --metrics $M --clock-control none -k regex:svpass -s 8 -c 1 --csv python tools/run_plan.py --dtype c64 > $O/w$w.csv 2>&1
  echo "waves $w"; grep -E "svpass" $O/w$w.csv | awk -F'","' '{print $(NF-2), $NF}'
done
