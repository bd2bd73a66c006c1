timeout -s KILL 300 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout -s KILL 120 python scripts/pass_ab.py 32,64,127 128
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ttft_p50_ms'], d['gpu_baselines'], d['roofline']['frac'], d['config']['budget'])"
