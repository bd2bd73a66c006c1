"""Config-3 TTFT breakdown: first-iteration record of duo vs vanilla / SpS
(2K prompt, T=1.0, up to 4 sequences)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_00784_b200 import (DEFAULT_PLANT, SHAPES, Draft, EngineConfig, Target,  # noqa: E402
                                   run_generation)

tcore, dcores = bench.core_slice(0, 1)
os.sched_setaffinity(0, {tcore})
tgt = Target(SHAPES["llama2_7b"], weight_seed=1234, plant=DEFAULT_PLANT, max_seq=4096)
drf = Draft(SHAPES["llama_68m"], weight_seed=99, plant=DEFAULT_PLANT, threads=len(dcores), cpus=dcores)
for rep in range(2):
    for mode in ("vanilla", "duo", "sps"):
        cfg = EngineConfig(mode=mode, budget=14, max_sequences=4, max_new_tokens=16, greedy=False,
                           temperature=1.0)
        r = run_generation(tgt, drf if mode != "vanilla" else None,
                           bench.make_prompt(rep + 1, 2048), cfg)
        it = r.iterations[0]
        print(mode, "ttft", round(r.ttft_ms, 2), "dev_ttft", round(r.device_ttft_ms, 2),
              "it0 draft", round(it.draft_ms, 2), "target", round(it.target_ms, 2), "comm",
              round(it.comm_ms, 2), "verify", round(it.verify_ms, 2), "seqs", it.sequence_count,
              flush=True)
