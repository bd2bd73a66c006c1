mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:pass_kernel --csv --log-file gpurun_out/pass_launches.csv python scripts/one_pass.py 8 128 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload config3 --no-cpu-baseline --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout -s KILL 120 python scripts/pass_timeline.py 8 128 > gpurun_out/timeline.txt 2>&1
python -c "
import json
for f in ['gpurun_out/bench.json','gpurun_out/bench_c3.json']:
    d=json.load(open(f)); print(f, d['value'], d['ttft_p50_ms'], d['roofline']['frac'], d['roofline']['pass_ms'], d['gpu_baselines'], d.get('cpu_baseline',{}).get('value'))"
