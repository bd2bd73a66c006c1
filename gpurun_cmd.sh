ncu --set full --clock-control none --import-source on -k regex:gemm_wide -s 130 -c 1 -o gpurun_out/wide_gu2 python scripts/one_pass.py 127 128 > gpurun_out/wide.log 2>&1
tail -1 gpurun_out/wide.log
