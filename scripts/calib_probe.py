"""Draft token time and calibrate() under bench.py's core layout, cold vs warm, caller pinned vs not."""
import os, sys
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import bench
from paper_2503_00784_b200 import DEFAULT_PLANT, SHAPES, Draft, Target, calibrate
print(open("/sys/devices/system/cpu/cpu0/topology/thread_siblings_list").read().strip(), open("/sys/devices/system/cpu/cpu2/topology/thread_siblings_list").read().strip())
tcore, dcores = bench.core_slice(0, 1)
print("tcore", tcore, "dcores", dcores)
os.sched_setaffinity(0, {tcore})
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=1024)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(dcores), cpus=dcores)
for i in range(3):
    print("time_token (caller on tcore)", drf.time_token(20))
    print("calibrate", calibrate(tgt, drf, probe_len=8, trials=12))
    print("pass", tgt.time_pass(8, 12))
os.sched_setaffinity(0, {dcores[0]})
print("time_token (caller on dcores[0])", drf.time_token(20))
d2 = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=12, cpus=list(range(1, 13)))
os.sched_setaffinity(0, set(range(16)))
print("draft cpus 1..12 unpinned caller", d2.time_token(20))
