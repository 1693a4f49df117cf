#!/bin/bash
# L2 traffic of the a6 kernel by operation (read vs red), hits and misses, and DRAM bytes.
cd "$(dirname "$0")/.."
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_red_lookup_hit.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
for spec in ${SPECS:-1024:1 1024:2}; do
  B=${spec%%:*}; T=${spec##*:}
  timeout 600 ncu --metrics $M --clock-control none -k regex:${KERN:-expert_group} -c 1 --csv \
    python tools/sweep_group.py ${CONFIG:-C3a} $spec > gpurun_out/l2_${B}_${T}.csv 2>/dev/null
  echo "== $spec"; grep -E '"(dram|lts|gpu)__' gpurun_out/l2_${B}_${T}.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
