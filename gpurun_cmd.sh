mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:attn -s 40 -c 1 -o gpurun_out/attn128_full python scripts/one_pass.py 8 128 > gpurun_out/attn_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn -s 300 -c 1 -o gpurun_out/attn2k_full python scripts/one_pass.py 8 2048 >> gpurun_out/attn_full.log 2>&1
