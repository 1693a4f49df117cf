cd $GRAFT_REPO_ROOT
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for c in ${CONFIGS:-C5s C3b}; do for v in 0 1; do
OMNIMOE_LIB=$M OMNIMOE_ROUTE_FUSED=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none --csv -k "regex:gemm_i8" -c 1 python tools/layer_once.py $c sliced 1 > gpurun_out/m_${c}_$v.csv 2>/dev/null
python - gpurun_out/m_${c}_$v.csv $c $v <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; mi=h.index("Metric Name"); vi=h.index("Metric Value")
print(sys.argv[2], "fused", sys.argv[3], {r[mi]: r[vi] for r in rows[1:]})
PY
done; done
