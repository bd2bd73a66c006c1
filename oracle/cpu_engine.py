"""oracle/cpu_engine.py — TEST INFRASTRUCTURE / CPU BASELINE ONLY.

The reference's decoding loop (proj/src/engine.cpp:273-512, apply_verification
62-106) restated over the CPU Llama oracle (llama_ref.c) for both roles: the
all-CPU path the north star times "beside" the GPU (bench.py cpu_baseline and
--impl reference).  Scored passes are batched ([c] ++ tail, one forward of
width 1 + L) and the KV cache is truncated to |verified| - 1 after each
verification, exactly like the GPU engine; verification and drafting use the
restated protocol functions (oracle/protocol.py).
"""
from __future__ import annotations

import time
from typing import List, Optional

import numpy as np

from . import protocol as P
from .llama import OracleLlama


class CpuDraft:
    """q(ctx) over an OracleLlama with prefix-reusing KV cache."""

    def __init__(self, llama: OracleLlama, temperature: float, greedy: bool):
        self.m, self.T, self.greedy = llama, temperature, greedy
        self.tokens: List[int] = []
        self.forwards = 0

    def __call__(self, ctx) -> np.ndarray:
        ctx = list(ctx)
        keep = 0
        lim = min(len(self.tokens), len(ctx) - 1)
        while keep < lim and self.tokens[keep] == ctx[keep]:
            keep += 1
        self.m.truncate(keep)
        self.tokens = self.tokens[:keep]
        lg = self.m.forward(ctx[keep:], last_only=True)[0]
        self.tokens = ctx
        self.forwards += 1
        return dist(lg, self.T, self.greedy)


def dist(logits: np.ndarray, T: float, greedy: bool) -> np.ndarray:
    if greedy:
        return P.onehot(len(logits), int(np.argmax(logits)))
    return P.softmax64(logits, T)


def run_cpu(mode: str, target: OracleLlama, draft: Optional[OracleLlama], prompt, budget: int,
            max_sequences: int, max_new_tokens: int, greedy: bool = True, temperature: float = 1.0,
            draft_seed: int = 1, verify_seed: int = 2, threaded: bool = True) -> dict:
    """Returns tokens, ttft_ms, total_ms and per-iteration committed counts.

    duo with threaded=True runs the draft in a worker thread concurrently with
    the target pass, one rendezvous per iteration (proj/src/engine.cpp:425-440,
    DuoExecution::threaded); each role owns its RandomStream, so the tokens
    equal the sequential execution's.  The oracle releases the GIL inside its
    forwards (ctypes), and each model runs its own thread count."""
    rd, rv = P.RandomStream(draft_seed), P.RandomStream(verify_seed)
    worker = None
    if mode == "duo" and threaded:
        import queue
        import threading
        req, rep = queue.Queue(), queue.Queue()

        def serve():
            while True:
                z = req.get()
                if z is None:
                    return
                try:
                    rep.put(P.draft_dynamic(drf, z, budget, max_sequences, rd))
                except BaseException as e:  # surfaced on the target thread
                    rep.put(e)
        worker = threading.Thread(target=serve, daemon=True)
    drf = CpuDraft(draft, temperature, greedy) if draft is not None else None
    if worker is not None:
        worker.start()
    verified = list(prompt)
    n_prompt = len(prompt)
    tail: Optional[P.DraftSequence] = None
    iters = []
    recs = []  # IterationRecord (tokens_processed, accepted, sequence_count)
    t0 = time.perf_counter()
    target.truncate(0)
    if n_prompt > 1:
        target.forward(verified[:-1], last_only=True)
    ttft = None
    while len(verified) - n_prompt < max_new_tokens:
        if mode == "vanilla":
            lg = target.forward([verified[-1]])
            verified.append(P.sample(dist(lg[0], temperature, greedy), rv.next_uniform()))
            committed, accepted, n_seq = 1, 0, 0
        elif mode == "sps":
            toks, dists, ctx = [], [], list(verified)
            for _ in range(budget):
                d = drf(ctx)
                t = P.sample(d, rd.next_uniform())
                toks.append(t)
                dists.append(d)
                ctx.append(t)
            lg = target.forward([verified[-1]] + toks)
            p_rows = [dist(r, temperature, greedy) for r in lg]
            acc, nxt = P.sps_verify(toks, dists, p_rows, rv)
            verified += toks[:acc] + [nxt]
            committed, accepted, n_seq = acc + 1, acc, 1
        else:  # duo (threaded: draft of this iteration overlaps the target pass)
            z = list(verified) + (list(tail.tokens) if tail else [])
            tail_tokens = list(tail.tokens) if tail else []
            if worker is not None:
                req.put(z)
                lg = target.forward([verified[-1]] + tail_tokens)
                bundle = rep.get()  # rendezvous
                if isinstance(bundle, BaseException):
                    req.put(None)
                    raise bundle
            else:
                bundle = P.draft_dynamic(drf, z, budget, max_sequences, rd)
                lg = target.forward([verified[-1]] + tail_tokens)
            p_rows = [dist(r, temperature, greedy) for r in lg]
            committed, accepted, usable = 0, 0, True
            n_seq = len(bundle.sequences)
            if tail is not None:
                out = P.verify_prefix(tail.tokens, tail.dists, p_rows[:len(tail.tokens)], rv)
                if out.all_accepted:
                    verified += tail.tokens
                    committed += len(tail.tokens)
                    accepted += len(tail.tokens)
                else:
                    verified += tail.tokens[:out.reject_index] + [out.resample]
                    committed += out.reject_index + 1
                    accepted += out.reject_index
                    usable = False
                tail = None
            if usable:
                bo = P.verify_bundle([s.tokens[0] for s in bundle.sequences], p_rows[-1], rv)
                if bo.accepted:
                    seq = bundle.sequences[bo.seq_index]
                    verified.append(seq.tokens[0])
                    committed += 1
                    accepted += 1
                    if len(seq.tokens) > 1:
                        tail = P.DraftSequence(seq.tokens[1:], seq.dists[1:],
                                               float(seq.dists[1][seq.tokens[1]]))
                else:
                    verified.append(bo.fallback)
                    committed += 1
        target.truncate(len(verified) - 1)
        iters.append(committed)
        recs.append((committed, accepted, n_seq))
        if ttft is None:
            ttft = (time.perf_counter() - t0) * 1e3
    total = (time.perf_counter() - t0) * 1e3
    if worker is not None:
        req.put(None)
        worker.join()
    return dict(tokens=verified[n_prompt:], ttft_ms=ttft, total_ms=total, iterations=iters,
                records=recs)
