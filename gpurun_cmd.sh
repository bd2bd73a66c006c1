mkdir -p gpurun_out
# one_pass 127: prefill 128 (1 pass of 128 -> W=128 GEMMs) then 3 W=127 passes; capture the 3rd GEMM (gate/up layer 0) of the 2nd pass
ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 131 -c 1 -o gpurun_out/gemm127 python scripts/one_pass.py 127 128 > gpurun_out/gemm127.log 2>&1
tail -3 gpurun_out/gemm127.log
