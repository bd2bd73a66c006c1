#!/bin/bash
# Refresh the profiles/ evidence for the current pass kernel (run under gpurun):
# DRAM bytes per W=8 pass, one --set full capture, and the bench launch list.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pass_kernel --csv --log-file gpurun_out/pass_traffic.csv python scripts/one_pass.py 8 128 \
    > gpurun_out/pass_traffic.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 2 -c 1 \
    -o gpurun_out/pass_full -f python scripts/one_pass.py 8 128 > gpurun_out/pass_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out | tail -8
