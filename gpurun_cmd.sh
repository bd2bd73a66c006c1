mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:pass_kernel --csv --log-file gpurun_out/pass_launches.csv python scripts/one_pass.py 8 128 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 2 -c 1 -o gpurun_out/pass_full python scripts/one_pass.py 8 128 > gpurun_out/pass_full.log 2>&1
cuobjdump -sass paper_2503_00784_b200/libduodec_b200.so > gpurun_out/all.sass 2>&1
ls -la gpurun_out
