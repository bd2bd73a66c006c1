"""CPU draft ms/token vs thread count (is the 68M draft memory-bound?)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import SHAPES, DEFAULT_PLANT, Draft  # noqa: E402
for n in (1, 2, 4, 8, 12, 15):
    d = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=n, cpus=list(range(1, 1 + n)))
    print(n, "threads:", round(d.time_token(20), 3), "ms/token", flush=True)
    d.close()
