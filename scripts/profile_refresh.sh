#!/bin/bash
# Refresh the profiles/ evidence for the current pass kernel (run under gpurun):
# DRAM bytes per pass at widths 1 / 9 / 16 (-> profiles/pass_traffic.json via
# scripts/traffic_json.py), one --set full capture, and the bench launch list.
mkdir -p gpurun_out
for w in 1 9 16; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pass_kernel --csv --log-file gpurun_out/pass_traffic_w$w.csv python scripts/one_pass.py $w 128 \
    > gpurun_out/pass_traffic.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 2 -c 1 \
    -o gpurun_out/pass_full -f python scripts/one_pass.py 9 128 > gpurun_out/pass_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out | tail -8
