#!/bin/bash
# per-kernel time, DRAM and L2 traffic of the a6 kernels of one layer forward
#   CONFIG=C3a LAYOUT=sliced KERN='expert_dot|expert_vslice' bash tools/ncu_kernels.sh
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
OUT=gpurun_out/ncu_${CONFIG:-C3a}_${LAYOUT:-sliced}${TAG}.csv
timeout 600 ncu --metrics $M --clock-control none -k "regex:${KERN:-expert_dot|expert_vslice}" -s ${SKIP:-0} -c ${COUNT:-4} --csv \
  python tools/layer_once.py ${CONFIG:-C3a} ${LAYOUT:-sliced} 2 $EXTRA > $OUT 2>/dev/null
python - "$OUT" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ii = hdr.index("ID")
cur = {}
for r in rows[1:]:
    cur.setdefault((r[ii], r[ki][:40]), {})[r[mi]] = r[vi]
for (i, k), m in cur.items():
    print(i, k, " ".join(f"{a.split('__')[1][:28]}={b}" for a, b in m.items()))
PY
