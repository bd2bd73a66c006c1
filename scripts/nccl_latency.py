"""NCCL all-reduce latency on this box for the TP reduction's message size
(W x d_model, bf16 and fp32), CUDA-event timed, torch.distributed (backend
nccl) over the ranks of this launch.  On a one-GPU box this is world size 1:
no link traffic, only NCCL's launch + kernel floor, which every one of the
160 per-pass reductions of a 70B TP=8 pass would pay on top of the transfer
(the persistent pass kernel's in-epilogue tile exchange pays no launch).
python scripts/nccl_latency.py [W]   (or under torchrun for N ranks)"""
import json
import os
import sys

import torch
import torch.distributed as dist

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
out = {"world_size": world, "width": w}
for d, dt in ((8192, torch.bfloat16), (8192, torch.float32), (4096, torch.bfloat16)):
    x = torch.randn(w, d, device="cuda").to(dt)
    for _ in range(20):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    s.record()
    for _ in range(n):
        dist.all_reduce(x)
    e.record()
    torch.cuda.synchronize()
    out[f"{w}x{d}_{str(dt).split('.')[-1]}_us"] = round(s.elapsed_time(e) * 1e3 / n, 2)
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
