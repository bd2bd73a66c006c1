mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload config3 --no-cpu-baseline --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
cat gpurun_out/bench.json gpurun_out/bench_c3.json
