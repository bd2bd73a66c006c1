# A/B of the long-prompt prefill (2K tokens, 7B shape) and the GPU tests that
# cover it: bash scripts/ab_prefill.sh   (run under gpurun)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hd128.py tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/t_att.log 2>&1; echo "rc=$?" >> gpurun_out/t_att.log
for r in 1 2; do for v in 0 1; do echo "tc=$v $(DD_ATTN_PREFILL_TC=$v timeout 200 python scripts/prefill_2k.py 1024 2048 2>&1 | tail -2 | tr '\n' ' ')"; done; done > gpurun_out/ab_pf.log 2>&1
tail -3 gpurun_out/t_att.log; cat gpurun_out/ab_pf.log
