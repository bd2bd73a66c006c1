"""oracle/protocol.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

A plain-Python/numpy restatement of the reference DuoDecoding protocol
(reference root /root/reference, paths below relative to it).  Every function
cites the reference lines it restates.  It is pinned against the compiled
reference (oracle/_ref/libduodec_ref.so, tests/test_oracle_vs_ref.py) and
against the committed golden vectors (tests/golden/), and is then used as the
checker for the GPU acceptance kernel at V=32000 and for the engine loop.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

M64 = (1 << 64) - 1
ZERO_MASS = 1e-12  # kZeroMassThreshold, proj/include/duodec/distribution.hpp:17


# ---------------------------------------------------------------- RNG
def splitmix(seed: int, m: int) -> int:
    """Draw m (1-based) of RandomStream(seed): proj/include/duodec/random.hpp:16-21."""
    z = (seed + m * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def derive_seed(base: int, index: int) -> int:
    """random.hpp:38-43."""
    z = (base + (index + 1) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 30)) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class RandomStream:
    """Counter-based uniform stream (random.hpp:11-34)."""

    def __init__(self, seed: int = 0, counter: int = 0):
        self.seed = seed & M64
        self.counter = counter

    def next_u64(self) -> int:
        self.counter += 1
        return splitmix(self.seed, self.counter)

    def next_uniform(self) -> float:
        """random.hpp:24-26: (x >> 11) * 2^-53."""
        return float(self.next_u64() >> 11) * 2.0 ** -53


# ---------------------------------------------------------------- distributions
def seq_sum(v) -> float:
    """Left-to-right fp64 sum, the scalar kernels::sum (proj/src/kernels_scalar.cpp:7-13).
    Tests load the reference with DUODEC_KERNELS=scalar so sums agree bit-for-bit."""
    acc = 0.0
    for x in np.asarray(v, dtype=np.float64).tolist():
        acc += x
    return acc


def sample(p: np.ndarray, u: float) -> int:
    """Inverse CDF: proj/src/distribution.cpp:61-78 (skip p<=0; fallback last support)."""
    acc = 0.0
    last = 0
    for i in np.flatnonzero(p > 0.0):
        acc += float(p[i])
        last = int(i)
        if u < acc:
            return int(i)
    return last


def argmax(p: np.ndarray) -> int:
    """First index of the max: proj/src/kernels_scalar.cpp:40-48."""
    return int(np.argmax(p))


def accept_test(p_tok: float, q_tok: float, r: float) -> bool:
    """proj/src/verify.cpp:25-28: strict r < p/q."""
    return r < p_tok / q_tok


def residual_or_p(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """proj/src/verify.cpp:13-21."""
    buf = np.maximum(p - q, 0.0)
    mass = seq_sum(buf)
    if mass < ZERO_MASS:
        return p
    return buf * (1.0 / mass)


def softmax64(logits: np.ndarray, temperature: float = 1.0) -> np.ndarray:
    """p = softmax(logits / T) in fp64 — the transformer reading of temper()
    (proj/src/model.cpp:54-69: p^(1/T) renormalised == softmax(log p / T))."""
    z = logits.astype(np.float64) * (1.0 / temperature)
    e = np.exp(z - z.max())
    return e / e.sum()


def onehot(v: int, idx: int) -> np.ndarray:
    out = np.zeros(v, dtype=np.float64)
    out[idx] = 1.0
    return out


# ---------------------------------------------------------------- verify
@dataclass
class PrefixOutcome:
    all_accepted: bool
    reject_index: int = -1
    resample: int = -1


def verify_prefix(tokens: Sequence[int], q_rows, p_rows, rng: RandomStream) -> PrefixOutcome:
    """proj/src/verify.cpp:41-61."""
    for j, tok in enumerate(tokens):
        r = rng.next_uniform()
        if not accept_test(float(p_rows[j][tok]), float(q_rows[j][tok]), r):
            res = residual_or_p(np.asarray(p_rows[j]), np.asarray(q_rows[j]))
            return PrefixOutcome(False, j, sample(res, rng.next_uniform()))
    return PrefixOutcome(True)


@dataclass
class BundleOutcome:
    accepted: bool
    seq_index: int = -1
    fallback: int = -1


def verify_bundle(firsts: Sequence[int], p_next: np.ndarray, rng: RandomStream) -> BundleOutcome:
    """proj/src/verify.cpp:63-90: point-mass tests against the running residual."""
    cur = np.array(p_next, dtype=np.float64)
    for i, tok in enumerate(firsts):
        r = rng.next_uniform()
        if accept_test(float(cur[tok]), 1.0, r):
            return BundleOutcome(True, i)
        cur[tok] = 0.0
        mass = seq_sum(cur)
        if mass < ZERO_MASS:
            cur = np.array(p_next, dtype=np.float64)
        else:
            cur = cur * (1.0 / mass)
    return BundleOutcome(False, fallback=sample(cur, rng.next_uniform()))


def sps_verify(tokens: Sequence[int], q_rows, p_rows, rng: RandomStream):
    """proj/src/verify.cpp:92-107 -> (accepted, next_token)."""
    for j, tok in enumerate(tokens):
        r = rng.next_uniform()
        if not accept_test(float(p_rows[j][tok]), float(q_rows[j][tok]), r):
            res = residual_or_p(np.asarray(p_rows[j]), np.asarray(q_rows[j]))
            return j, sample(res, rng.next_uniform())
    return len(tokens), sample(np.asarray(p_rows[len(tokens)]), rng.next_uniform())


# ---------------------------------------------------------------- drafting
def ranked_tokens(p: np.ndarray) -> np.ndarray:
    """proj/src/distribution.cpp:80-87: descending prob, ties ascending id."""
    return np.argsort(-p, kind="stable")


@dataclass
class DraftSequence:
    tokens: List[int]
    dists: List[np.ndarray]
    first_token_prob: float


@dataclass
class DraftBundle:
    sequences: List[DraftSequence]
    threshold: float
    budget_used: int
    forwards_used: int


def draft_dynamic(forward: Callable[[Sequence[int]], np.ndarray], context: Sequence[int],
                  budget: int, max_sequences: int, rng: RandomStream) -> DraftBundle:
    """proj/src/drafting.cpp:71-136 (sampled continuation, probe reuse)."""
    first = forward(list(context))
    ranks = ranked_tokens(first)
    top = int(ranks[0])
    p_top = float(first[top])
    probe = forward(list(context) + [top])
    p_second = float(probe[argmax(probe)])
    threshold = p_top * p_second
    forwards = 2
    s_cap = min(max_sequences, budget)
    firsts = [top]
    for r in ranks[1:]:
        if len(firsts) >= s_cap:
            break
        if not (float(first[r]) > threshold):
            break
        firsts.append(int(r))
    s = len(firsts)
    base_len = budget // s
    rem = budget - base_len * s
    seqs = []
    for i in range(s):
        length = base_len + (rem if i == 0 else 0)
        toks = [firsts[i]]
        dists = [first]
        ctx = list(context) + [firsts[i]]
        for pos in range(1, length):
            if i == 0 and pos == 1:
                d = probe
            else:
                d = forward(ctx)
                forwards += 1
            t = sample(d, rng.next_uniform())
            toks.append(t)
            dists.append(d)
            ctx.append(t)
        seqs.append(DraftSequence(toks, dists, float(first[firsts[i]])))
    return DraftBundle(seqs, threshold, budget, forwards)


# ---------------------------------------------------------------- engine
@dataclass
class Profile:
    """DeviceProfile, proj/include/duodec/simclock.hpp:16-42."""
    draft_per_token_ms: float = 1.0
    target_base_ms: float = 24.0
    target_slope_ms: float = 0.0
    comm_ms: float = 0.2

    def target_pass_ms(self, w: int) -> float:
        return self.target_base_ms + self.target_slope_ms * w

    def draft_ms(self, forwards: int) -> float:
        return self.draft_per_token_ms * forwards

    def verify_ms(self) -> float:
        return 0.01 * self.target_pass_ms(1)


BALANCED24 = Profile(1.0, 24.0, 0.0, 0.2)   # simclock.cpp:58-60
FIGURE1 = Profile(3.0, 20.0, 0.5, 0.2)      # simclock.cpp:62-64


@dataclass
class IterationRecord:
    tokens_processed: int = 0
    sequence_count: int = 0
    accepted: int = 0
    width: int = 0


@dataclass
class GenerationResult:
    tokens: List[int] = field(default_factory=list)
    iterations: List[IterationRecord] = field(default_factory=list)
    ttft_ms: float = 0.0
    total_ms: float = 0.0
    tps: float = 0.0


def scored_with_next(forward, context, candidates) -> List[np.ndarray]:
    """proj/src/engine.cpp:36-43 with forward_scored (proj/src/model.cpp:310-320)."""
    out = []
    ctx = list(context)
    for c in candidates:
        out.append(forward(ctx))
        ctx.append(c)
    out.append(forward(ctx))
    return out


def run_vanilla(target, prompt, max_new_tokens, verify_seed=2, profile=BALANCED24):
    """proj/src/engine.cpp:273-312 on a simulated timeline."""
    rng = RandomStream(verify_seed)
    verified = list(prompt)
    res = GenerationResult()
    now = 0.0
    while len(verified) - len(prompt) < max_new_tokens:
        d = target(verified)
        verified.append(sample(d, rng.next_uniform()))
        now += profile.target_pass_ms(1)
        res.iterations.append(IterationRecord(1, 0, 0, 1))
        if len(res.iterations) == 1:
            res.ttft_ms = now
    res.tokens = verified[len(prompt):]
    res.total_ms = now
    res.tps = len(res.tokens) / (now / 1000.0) if now > 0 else 0.0
    return res


def run_sps(target, draft, prompt, budget, max_new_tokens, draft_seed=1, verify_seed=2,
            profile=BALANCED24):
    """proj/src/engine.cpp:314-393."""
    rd, rv = RandomStream(draft_seed), RandomStream(verify_seed)
    verified = list(prompt)
    res = GenerationResult()
    now = 0.0
    while len(verified) - len(prompt) < max_new_tokens:
        toks, dists = [], []
        ctx = list(verified)
        for _ in range(budget):
            d = draft(ctx)
            t = sample(d, rd.next_uniform())
            toks.append(t)
            dists.append(d)
            ctx.append(t)
        p_rows = scored_with_next(target, verified, toks)
        acc, nxt = sps_verify(toks, dists, p_rows, rv)
        verified += toks[:acc] + [nxt]
        now += profile.draft_ms(budget) + profile.target_pass_ms(budget + 1) + profile.verify_ms()
        res.iterations.append(IterationRecord(acc + 1, 1, acc, budget + 1))
        if len(res.iterations) == 1:
            res.ttft_ms = now
    res.tokens = verified[len(prompt):]
    res.total_ms = now
    res.tps = len(res.tokens) / (now / 1000.0) if now > 0 else 0.0
    return res


def run_duo(target, draft, prompt, budget, max_sequences, max_new_tokens, draft_seed=1,
            verify_seed=2, profile=BALANCED24):
    """proj/src/engine.cpp:395-512 (sequential execution; the threaded path emits
    identical tokens) with apply_verification (engine.cpp:62-106)."""
    rd, rv = RandomStream(draft_seed), RandomStream(verify_seed)
    verified = list(prompt)
    tail: Optional[DraftSequence] = None
    res = GenerationResult()
    now = 0.0
    while len(verified) - len(prompt) < max_new_tokens:
        z = list(verified) + (list(tail.tokens) if tail else [])
        bundle = draft_dynamic(draft, z, budget, max_sequences, rd)
        tail_tokens = list(tail.tokens) if tail else []
        p_rows = scored_with_next(target, verified, tail_tokens)
        committed = accepted = 0
        usable = True
        if tail is not None:
            out = verify_prefix(tail.tokens, tail.dists, p_rows[:len(tail.tokens)], rv)
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
            bo = verify_bundle([s.tokens[0] for s in bundle.sequences], p_rows[-1], rv)
            if bo.accepted:
                seq = bundle.sequences[bo.seq_index]
                verified.append(seq.tokens[0])
                committed += 1
                accepted += 1
                if len(seq.tokens) > 1:  # tail_of, engine.cpp:45-51
                    tail = DraftSequence(seq.tokens[1:], seq.dists[1:],
                                         float(seq.dists[1][seq.tokens[1]]))
            else:
                verified.append(bo.fallback)
                committed += 1
        width = len(tail_tokens) + 1
        now += max(profile.draft_ms(bundle.forwards_used), profile.target_pass_ms(width))
        now += profile.comm_ms + profile.verify_ms()
        res.iterations.append(IterationRecord(committed, len(bundle.sequences), accepted, width))
        if len(res.iterations) == 1:
            res.ttft_ms = now
    res.tokens = verified[len(prompt):]
    res.total_ms = now
    res.tps = len(res.tokens) / (now / 1000.0) if now > 0 else 0.0
    return res


def choose_budget(c: float) -> int:
    """proj/src/engine.cpp:580-582: max(2, round(c)) (std::lround: half away from zero)."""
    return max(2, int(math.floor(c + 0.5)) if c >= 0 else int(math.ceil(c - 0.5)))


def median(v: Sequence[float]) -> float:
    s = sorted(v)
    n = len(s)
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


# ---------------------------------------------------------------- Markov models
class MarkovModel:
    """Backoff Markov table (proj/src/model.cpp:84-320) parsed from the reference's
    text format, with temper() (model.cpp:54-69)."""

    def __init__(self, text: str, temperature: Optional[float] = None):
        self.rows = {}
        self.default = None
        self.vocab = 0
        self.order = 0
        self.temperature = 1.0
        for raw in text.splitlines():
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("vocab"):
                self.vocab = int(line.split()[1])
            elif line.startswith("order"):
                self.order = int(line.split()[1])
            elif line.startswith("temperature"):
                self.temperature = float(line.split()[1])
            elif line.startswith("ctx"):
                head, probs = line[3:].split(":", 1)
                key = tuple(int(t) for t in head.replace(",", " ").split())
                self.rows[key] = np.array([float(x) for x in probs.split()])
            elif line.startswith("default"):
                self.default = np.array([float(x) for x in line.split(":", 1)[1].split()])
        if temperature is not None:
            self.temperature = temperature
        self._t = {k: self._temper(v) for k, v in self.rows.items()}
        self._d = self._temper(self.default)

    def _temper(self, raw: np.ndarray) -> np.ndarray:
        if self.temperature == 1.0:
            return raw.copy()
        inv = 1.0 / self.temperature
        out = np.where(raw > 0.0, np.power(raw, inv), 0.0)
        return out / seq_sum(out)

    def __call__(self, context: Sequence[int]) -> np.ndarray:
        if self.order == 0 or len(context) == 0:
            return self._d
        for k in range(min(self.order, len(context)), 0, -1):
            key = tuple(context[-k:])
            if key in self._t:
                return self._t[key]
        return self._d
