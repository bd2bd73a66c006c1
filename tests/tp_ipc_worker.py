"""One rank of a two-process tensor-parallel group (helper of
tests/test_gpu_tp.py::test_tp_two_processes_ipc, launched by torchrun).

The ranks exchange CUDA IPC handles of their exchange buffers over a gloo
all_gather (the deployment recipe of include/duodec_b200.h), run a prefill
and a scored pass, and save their logits for the test to compare.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_00784_b200 import Target, tp_connect_group  # noqa: E402


def main(out_dir: str, spec: str) -> None:
    import json
    cfg = json.loads(spec)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = Target(cfg["shape"], weight_seed=cfg["seed"], plant=cfg["plant"], max_seq=512,
               device=int(os.environ.get("DD_TP_DEVICE", "0")), tp_rank=rank, tp_size=world)
    tp_connect_group(t)
    t.prefill(cfg["prompt"])
    t.score(cfg["new"])
    np.save(Path(out_dir) / f"logits_r{rank}.npy", t.logits(0, len(cfg["new"])))
    dist.barrier()
    t.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
