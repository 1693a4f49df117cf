cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
for c in 2 4 8 16; do timeout 600 python bench.py --config C3a --steps 5 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/b.json 2>&1; python -c "
import json; j=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('chunks $c', round(j['ms_per_step'],3), round(j['e2e']['ms_per_step'],3))"; done
python tools/layer_prof.py C5 sliced 3 2>&1 | grep -v -i warn | head -16
