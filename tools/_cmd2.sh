set -x
python tools/measure_cert_eps.py C1 C2 C3a C4pp C5 2>&1 | tail -8
timeout 600 python bench.py --config C3a --cert-eps 1e-5 --steps 5 --warmup 3 --cpu-tokens 32 2>&1 | tail -3
timeout 600 python bench.py --config C3b --cert-eps 1e-5 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_c3a.csv python bench.py --config C3a --cert-eps 1e-5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -5 gpurun_out/launches_c3a.csv
