#!/bin/bash
# ncu evidence for profiles/: per-launch times of one warm pass (W=8) and a full
# capture of the dominant kernel (gate/up GEMM of a middle layer).
set -x
mkdir -p gpurun_out
#ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
#    --csv --log-file gpurun_out/launches_w8.csv python scripts/one_pass.py 8 > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 262 -c 4 \
    -o gpurun_out/gemm_full python scripts/one_pass.py 8 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:attention -s 66 -c 1 \
    -o gpurun_out/attn_full python scripts/one_pass.py 8 > gpurun_out/ncu_attn.log 2>&1
cuobjdump -sass paper_2503_00784_b200/libduodec_b200.so > gpurun_out/sass.txt 2>&1
ls -la gpurun_out
