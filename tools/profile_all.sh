#!/bin/bash
# Launch list of one bench step + ncu --set full of each main kernel (one launch each),
# summarised into gpurun_out/*.csv / *.ncu-rep.  KERNELS: regexes; CONFIG: workload.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=${CONFIG:-C3a}
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $ARGS"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}${TAG}.csv $B > /dev/null 2>&1
echo "launches rc=$?"
for k in ${KERNELS:-expert_zdot expert_vslice select_bucket gemm_i8_exact gemm_tc_kernel radix_scatter}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-1} -c 1 -o gpurun_out/full_${k}_${CFG}${TAG} $B > gpurun_out/ncu_${k}.log 2>&1
  echo "$k rc=$?"
done
