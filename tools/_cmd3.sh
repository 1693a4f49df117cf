./tools/microbench
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expert_warp -s 1 -c 1 -o gpurun_out/prof_expert_v1 python bench.py --config C3a --cert-eps 1e-5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/ncu3.log
