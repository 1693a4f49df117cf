timeout 900 python -m pytest tests -m gpu -q -x -k "dense" 2>&1 | tail -1
for c in C4 C4p; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()})"; done
