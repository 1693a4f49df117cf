cd $GRAFT_REPO_ROOT
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for c in C5s C3b; do for v in 0 1; do
OMNIMOE_LIB=$M OMNIMOE_ROUTE_FUSED=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:gemm_i8|select|limb|exact_dd" python tools/layer_once.py $c sliced 2 > gpurun_out/k_${c}_$v.csv 2>/dev/null
python - gpurun_out/k_${c}_$v.csv $c $v <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
t=collections.defaultdict(float); n=collections.Counter()
for r in rows[1:]:
    k=r[ki].split('(')[0][-40:]; t[k]+=float(r[vi].replace(',','')); n[k]+=1
print(sys.argv[2], "fused", sys.argv[3], {k: round(v/n[k]/1e3,1) for k,v in t.items()})
PY
done; done
