#!/bin/bash
# SLICED executor: parity tests, then ncu per-kernel metrics under env knobs ($SWEEP: list of "VAR=val ..." sets)
cd "$(dirname "$0")/.."
# OMNIMOE_* knobs are read only by the measurement build (csrc/tuning.cuh)
python -m paper_2602_05711_b200.build --measure > /dev/null
export OMNIMOE_LIB=$(pwd)/paper_2602_05711_b200/libomnimoe_measure.so
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "sliced or pack_v" > gpurun_out/pytest_sliced.log 2>&1; tail -3 gpurun_out/pytest_sliced.log
IFS=';' read -ra SETS <<< "${SWEEP:-OMNIMOE_V_HINT=1}"
for cfg in "${SETS[@]}"; do
  env $cfg TAG="_$(echo $cfg | tr ' =' '__')" KERN="${KERN:-expert_zdot|expert_vslice}" COUNT=2 bash tools/ncu_kernels.sh > /tmp/o.txt 2>&1
  echo "== $cfg"; cut -c1-900 /tmp/o.txt
done
