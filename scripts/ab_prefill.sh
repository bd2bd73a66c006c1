mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hd128.py tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/t_att.log 2>&1; echo "rc=$?" >> gpurun_out/t_att.log
for r in 1 2; do for v in base lb2 lb3; do echo "$v $(DD_LIB_AB=alt/lib_$v.so timeout 200 python scripts/prefill_2k.py 2048 2>&1 | tail -1)"; done; done > gpurun_out/ab_pf.log 2>&1
tail -2 gpurun_out/t_att.log; cat gpurun_out/ab_pf.log
