timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 120 python scripts/pass_ab.py 17,64,127,128 128
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_wide --csv --log-file gpurun_out/wide_launches.csv python scripts/one_pass.py 127 128 > /dev/null 2>&1
