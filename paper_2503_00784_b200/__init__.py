"""B200-native DuoDecoding target path (arXiv 2503.00784).

Host-side mirror of the reference's model / verifier / engine interface
(reference proj/include/duodec/{model,verify,engine}.hpp) over the C ABI in
include/duodec_b200.h.  Everything that computes runs in libduodec_b200.so:
the target forward and the acceptance kernel on the GPU (sm_100a), the draft
model and the decoding loop in native host code.  There is no CPU fallback for
the target path; on a machine without a Blackwell GPU, Target() raises
DeviceError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as _L

__all__ = [
    "StateError",
    "SHAPES", "Target", "Draft", "EngineConfig", "GenerationResult", "IterationRecord",
    "run_generation", "run_vanilla", "run_sps", "run_duo", "calibrate", "choose_budget",
    "tp_connect_group",
    "ConfigError", "DegenerateTiming", "DeviceError", "DuoError",
]

# Model shapes of BASELINE.json's configs.
SHAPES = {
    "llama2_7b": dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128,
                      ffn_dim=11008, vocab=32000, rms_eps=1e-5, rope_theta=1e4),
    "llama_68m": dict(n_layers=2, d_model=768, n_heads=12, n_kv_heads=12, head_dim=64,
                      ffn_dim=3072, vocab=32000, rms_eps=1e-5, rope_theta=1e4),
    "tiny": dict(n_layers=4, d_model=512, n_heads=8, n_kv_heads=8, head_dim=64, ffn_dim=1408,
                 vocab=32000, rms_eps=1e-5, rope_theta=1e4),
    # head_dim-128 parity shapes (the 7B / 70B code paths at oracle-sized
    # widths): MHA like the 7B, and GQA at the 70B's 8:1 q:kv ratio
    "mid128": dict(n_layers=2, d_model=1024, n_heads=8, n_kv_heads=8, head_dim=128,
                   ffn_dim=2816, vocab=32000, rms_eps=1e-5, rope_theta=1e4),
    "gqa128": dict(n_layers=2, d_model=2048, n_heads=16, n_kv_heads=2, head_dim=128,
                   ffn_dim=5632, vocab=32000, rms_eps=1e-5, rope_theta=1e4),
    "llama2_70b": dict(n_layers=80, d_model=8192, n_heads=64, n_kv_heads=8, head_dim=128,
                       ffn_dim=28672, vocab=32000, rms_eps=1e-5, rope_theta=1e4),
}

# Default planted agreement (SURVEY.md §7 hard part 1), recorded beside every number.
DEFAULT_PLANT = dict(plant_seed=7, alpha=0.9, gain=1.0, emb_std=1.0)


class DuoError(RuntimeError):
    """Base of errors raised across the C ABI."""


class ConfigError(DuoError, ValueError):
    """proj/include/duodec/engine.hpp:29-31."""


class DegenerateTiming(DuoError):
    """proj/include/duodec/engine.hpp:32-34."""


class DeviceError(DuoError):
    """CUDA / no-GPU failures (there is no CPU fallback)."""


class StateError(DuoError):
    pass


def _check(rc: int, handle=None):
    if rc == _L.DD_OK:
        return
    msg = (_L.lib().dd_last_error(handle) or b"").decode()
    cls = {_L.DD_E_ARG: ConfigError, _L.DD_E_CUDA: DeviceError, _L.DD_E_STATE: StateError,
           _L.DD_E_CAPACITY: ConfigError}.get(rc, DuoError)
    raise cls(msg or f"duodec_b200 error {rc}")


PRECISIONS = {"bf16": _L.DD_PREC_BF16, "fp32acc": _L.DD_PREC_FP32ACC}


def _desc(shape: dict, max_seq: int, page_size: int = 16, precision: str = "bf16") -> _L.ModelDesc:
    if precision not in PRECISIONS:
        raise ConfigError(f"unknown precision {precision}")
    return _L.ModelDesc(shape["n_layers"], shape["d_model"], shape["n_heads"],
                        shape.get("n_kv_heads", shape["n_heads"]), shape["head_dim"],
                        shape["ffn_dim"], shape["vocab"], shape.get("rms_eps", 1e-5),
                        shape.get("rope_theta", 1e4), max_seq, page_size, PRECISIONS[precision])


def _plant(p: Optional[dict]) -> Optional[_L.PlantDesc]:
    if not p:
        return None
    return _L.PlantDesc(int(p.get("plant_seed", 0)), float(p.get("alpha", 0.0)),
                        float(p.get("gain", 0.0)), float(p.get("emb_std", 0.0)))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class Target:
    """GPU target model: the stateful replacement of ModelSpec on the target
    role (proj/include/duodec/model.hpp:57-65)."""

    def __init__(self, shape: dict, weight_seed: int = 1234, plant: Optional[dict] = None,
                 max_seq: int = 4096, device: int = 0, page_size: int = 16, tp_rank: int = 0,
                 tp_size: int = 1, precision: str = "bf16"):
        """precision: "bf16" (the fast path) or "fp32acc" (split hi + lo
        activations, fp32 KV and attention: the 1e-4 reference mode)."""
        self.shape = dict(shape)
        self.vocab = shape["vocab"]
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.precision = precision
        h = C.c_void_p()
        _check(_L.lib().dd_ctx_create_tp(C.byref(_desc(shape, max_seq, page_size, precision)), device,
                                         tp_rank, tp_size, C.byref(h)))
        self.h = h
        pl = _plant(plant)
        _check(_L.lib().dd_weights_init(self.h, weight_seed, C.byref(pl) if pl else None), self.h)

    # ---- tensor parallelism (include/duodec_b200.h, dd_ctx_create_tp)
    def tp_handle(self) -> bytes:
        """This rank's CUDA IPC handle, to all-gather across the rank processes."""
        buf = C.create_string_buffer(_L.DD_TP_HANDLE_BYTES)
        _check(_L.lib().dd_tp_export(self.h, buf), self.h)
        return buf.raw

    def tp_connect(self, handles: Sequence[bytes]) -> None:
        """Open every rank's exchange buffer (handles in rank order)."""
        blob = b"".join(handles)
        if len(handles) != self.tp_size or len(blob) != self.tp_size * _L.DD_TP_HANDLE_BYTES:
            raise ConfigError("need one IPC handle per rank")
        _check(_L.lib().dd_tp_connect(self.h, blob), self.h)

    @staticmethod
    def tp_connect_local(ranks: Sequence["Target"]) -> None:
        """Connect the ranks of one process (ranks[r] is rank r)."""
        arr = (C.c_void_p * len(ranks))(*[t.h.value for t in ranks])
        _check(_L.lib().dd_tp_connect_local(arr, len(ranks)), ranks[0].h)

    # ---- forward contract
    def prefill(self, tokens: Sequence[int]) -> None:
        t = _i32(tokens)
        _check(_L.lib().dd_prefill(self.h, _i32p(t), len(t)), self.h)

    def score(self, tokens: Sequence[int]) -> None:
        t = _i32(tokens)
        _check(_L.lib().dd_score(self.h, _i32p(t), len(t)), self.h)

    def logits(self, row0: int, rows: int) -> np.ndarray:
        out = np.zeros((rows, self.vocab), dtype=np.float32)
        _check(_L.lib().dd_read_logits(self.h, out.ctypes.data_as(C.POINTER(C.c_float)), row0,
                                       rows), self.h)
        return out

    def kv_len(self) -> int:
        n = C.c_int()
        _check(_L.lib().dd_kv_len(self.h, C.byref(n)), self.h)
        return n.value

    def truncate(self, n_valid: int) -> None:
        _check(_L.lib().dd_kv_truncate(self.h, n_valid), self.h)

    def compact(self, src: Sequence[int], dst: Sequence[int]) -> None:
        s, d = _i32(src), _i32(dst)
        _check(_L.lib().dd_kv_compact(self.h, _i32p(s), _i32p(d), len(s)), self.h)

    # ---- verification
    def upload_q(self, q_rows: np.ndarray) -> None:
        q = np.ascontiguousarray(q_rows, dtype=np.float32)
        _check(_L.lib().dd_upload_q(self.h, q.ctypes.data_as(C.POINTER(C.c_float)), q.shape[0],
                                    q.shape[1]), self.h)

    @staticmethod
    def _args(mode, tail_len, firsts, seed, counter, temperature, greedy, q_onehot):
        a = _L.VerifyArgs()
        a.mode = mode
        a.tail_len = tail_len
        a.n_firsts = len(firsts)
        for i, f in enumerate(firsts):
            a.firsts[i] = int(f)
        a.seed = seed
        a.counter = counter
        a.temperature = temperature
        a.greedy = int(greedy)
        a.q_onehot = int(q_onehot)
        return a

    @staticmethod
    def _out(o: _L.VerifyOut) -> dict:
        return {k: getattr(o, k) for k, _ in _L.VerifyOut._fields_ if k != "pad"}

    def verify(self, mode: int, tail_len: int = 0, firsts: Sequence[int] = (), seed: int = 2,
               counter: int = 0, temperature: float = 1.0, greedy: bool = False,
               q_onehot: bool = False) -> dict:
        a = self._args(mode, tail_len, firsts, seed, counter, temperature, greedy, q_onehot)
        o = _L.VerifyOut()
        _check(_L.lib().dd_verify(self.h, C.byref(a), C.byref(o)), self.h)
        return self._out(o)

    def verify_probs(self, p_rows: np.ndarray, tail: Sequence[int], mode: int,
                     firsts: Sequence[int] = (), seed: int = 2, counter: int = 0,
                     greedy: bool = False, q_onehot: bool = False) -> dict:
        p = np.ascontiguousarray(p_rows, dtype=np.float64)
        t = _i32(tail)
        a = self._args(mode, len(t), firsts, seed, counter, 1.0, greedy, q_onehot)
        o = _L.VerifyOut()
        _check(_L.lib().dd_verify_probs(self.h, p.ctypes.data_as(C.POINTER(C.c_double)),
                                        _i32p(t), p.shape[-1], C.byref(a), C.byref(o)), self.h)
        return self._out(o)

    # ---- measurement
    def time_pass(self, w: int, trials: int = 12) -> float:
        ms = C.c_float()
        _check(_L.lib().dd_time_pass(self.h, w, trials, C.byref(ms)), self.h)
        return ms.value

    def profile_pass(self, w: int) -> dict:
        ms = (C.c_float * 4)()
        _check(_L.lib().dd_profile_pass(self.h, w, ms), self.h)
        return dict(gemm=ms[0], attention=ms[1], epilogue=ms[2], total=ms[3])

    def time_gemms(self, w: int, trials: int = 5):
        """(median ms, launches) of the pass's GEMM launches back to back."""
        ms = C.c_float()
        n = C.c_int()
        _check(_L.lib().dd_time_gemms(self.h, w, trials, C.byref(ms), C.byref(n)), self.h)
        return ms.value, n.value

    def pass_weight_bytes(self) -> int:
        return int(_L.lib().dd_pass_weight_bytes(self.h))

    def read_weights(self, which: int, layer: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint16)
        _check(_L.lib().dd_read_weights(self.h, which, layer,
                                        out.ctypes.data_as(C.POINTER(C.c_uint16)), n), self.h)
        return out

    def close(self):
        if getattr(self, "h", None):
            _L.lib().dd_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_gemm(W_bits: np.ndarray, X_bits: np.ndarray) -> np.ndarray:
    """Y = X . W^T through the tcgen05 GEMM (bf16 bit patterns in, fp32 out)."""
    n_out, k = W_bits.shape
    w = X_bits.shape[0]
    Wc = np.ascontiguousarray(W_bits, dtype=np.uint16)
    Xc = np.ascontiguousarray(X_bits, dtype=np.uint16)
    Y = np.zeros((w, n_out), dtype=np.float32)
    _check(_L.lib().dd_test_gemm(Wc.ctypes.data_as(C.POINTER(C.c_uint16)),
                                 Xc.ctypes.data_as(C.POINTER(C.c_uint16)), n_out, k, w,
                                 Y.ctypes.data_as(C.POINTER(C.c_float))))
    return Y


class Draft:
    """CPU draft model (Llama-68M shape) on pinned host cores."""

    def __init__(self, shape: dict, weight_seed: int = 99, plant: Optional[dict] = None,
                 threads: int = 0, cpus: Optional[Sequence[int]] = None, max_seq: int = 4096):
        self.shape = dict(shape)
        self.vocab = shape["vocab"]
        h = C.c_void_p()
        pl = _plant(plant)
        cp = (C.c_int * len(cpus))(*cpus) if cpus else None
        _check(_L.lib().dd_draft_create(C.byref(_desc(shape, max_seq)), weight_seed,
                                        C.byref(pl) if pl else None, threads, cp,
                                        len(cpus) if cpus else 0, C.byref(h)))
        self.h = h

    def logits(self, context: Sequence[int]) -> np.ndarray:
        t = _i32(context)
        out = np.zeros(self.vocab, dtype=np.float32)
        _check(_L.lib().dd_draft_logits(self.h, _i32p(t), len(t),
                                        out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def dist(self, context: Sequence[int], temperature: float = 1.0, greedy: bool = False):
        """q(. | context) as the engine's drafting sees it -> (q fp32, argmax)."""
        t = _i32(context)
        q = np.zeros(self.vocab, dtype=np.float32)
        am = C.c_int()
        _check(_L.lib().dd_draft_dist(self.h, _i32p(t), len(t), temperature, int(greedy),
                                      q.ctypes.data_as(C.POINTER(C.c_float)), C.byref(am)))
        return q, am.value

    def draft_dynamic(self, context: Sequence[int], budget: int, max_sequences: int,
                      seed: int, counter: int = 0, temperature: float = 1.0,
                      greedy: bool = False) -> dict:
        """The engine's draft_dynamic (proj/src/drafting.cpp:71-136)."""
        t = _i32(context)
        toks = np.zeros(budget, dtype=np.int32)
        lens = np.zeros(max_sequences, dtype=np.int32)
        cnt = C.c_uint64(counter)
        ns, fw = C.c_int(), C.c_int()
        th = C.c_double()
        _check(_L.lib().dd_draft_dynamic(self.h, _i32p(t), len(t), budget, max_sequences,
                                         temperature, int(greedy), seed, C.byref(cnt),
                                         _i32p(toks), _i32p(lens), C.byref(ns), C.byref(th),
                                         C.byref(fw)))
        seqs, k = [], 0
        for i in range(ns.value):
            seqs.append([int(x) for x in toks[k:k + lens[i]]])
            k += int(lens[i])
        return dict(seqs=seqs, threshold=th.value, forwards=fw.value, counter=cnt.value)

    def time_token(self, trials: int = 12) -> float:
        ms = C.c_float()
        _check(_L.lib().dd_draft_time_token(self.h, trials, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "h", None):
            _L.lib().dd_draft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- engine
MODES = {"duo": _L.DD_MODE_DUO, "sps": _L.DD_MODE_SPS, "vanilla": _L.DD_MODE_VANILLA}


@dataclass
class EngineConfig:
    """EngineConfig, proj/include/duodec/engine.hpp:43-60 (+ greedy)."""
    mode: str = "duo"
    budget: int = 24
    max_sequences: int = 8
    max_new_tokens: int = 128
    temperature: float = 1.0
    greedy: bool = False
    draft_seed: int = 1
    verify_seed: int = 2
    budget_policy: str = "fixed"
    budget_hard_cap: int = 256
    calib_probe_len: int = 8
    calib_trials: int = 12
    threaded: bool = True
    # WorkerHooks jitter (engine.hpp:36-41): 0 = off
    jitter_seed: int = 0
    jitter_max_us: int = 0

    def to_c(self) -> _L.EngineConfigC:
        if self.mode not in MODES:
            raise ConfigError(f"unknown mode {self.mode}")
        return _L.EngineConfigC(
            MODES[self.mode], self.budget, self.max_sequences, self.max_new_tokens,
            self.temperature, int(self.greedy), self.draft_seed, self.verify_seed,
            _L.DD_BUDGET_CALIBRATED if self.budget_policy == "calibrated" else _L.DD_BUDGET_FIXED,
            self.budget_hard_cap, self.calib_probe_len, self.calib_trials, int(self.threaded),
            self.jitter_seed, self.jitter_max_us)


@dataclass
class IterationRecord:
    """IterationRecord, proj/include/duodec/engine.hpp:62-70."""
    draft_ms: float
    target_ms: float
    verify_ms: float
    comm_ms: float
    tokens_processed: int
    sequence_count: int
    accepted: int
    width: int


@dataclass
class GenerationResult:
    """GenerationResult, proj/include/duodec/engine.hpp:72-78."""
    tokens: List[int] = field(default_factory=list)
    iterations: List[IterationRecord] = field(default_factory=list)
    ttft_ms: float = 0.0
    total_ms: float = 0.0
    tps: float = 0.0
    prefill_ms: float = 0.0
    budget: int = 0
    device_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    gpu_launches: int = 0
    device_ttft_ms: float = 0.0

    def iteration_lines(self) -> List[dict]:
        """`duodec profile` output (proj/tools/main.cpp:202-207, 332-367):
        one object per iteration with the reference's field names, then the
        summary object."""
        out, hist = [], {}
        for i, it in enumerate(self.iterations):
            out.append({"draft_ms": it.draft_ms, "target_ms": it.target_ms,
                        "verify_ms": it.verify_ms, "comm_ms": it.comm_ms,
                        "tokens_processed": it.tokens_processed, "s": it.sequence_count,
                        "accepted": it.accepted, "iteration": i})
            if it.sequence_count > 0:
                hist[str(it.sequence_count)] = hist.get(str(it.sequence_count), 0) + 1
        out.append({"summary": True, "iterations": len(self.iterations),
                    "sequence_histogram": dict(sorted(hist.items(), key=lambda kv: int(kv[0]))),
                    "tokens": len(self.tokens), "tps": self.tps, "ttft_ms": self.ttft_ms,
                    "total_ms": self.total_ms})
        return out

    def to_json(self, mode: str) -> dict:
        """`duodec generate` output (proj/tools/main.cpp:209-216)."""
        lines = self.iteration_lines()[:-1]
        for ln in lines:
            del ln["iteration"]
        return {"mode": mode, "tokens": list(self.tokens), "tps": self.tps,
                "ttft_ms": self.ttft_ms, "total_ms": self.total_ms, "iterations": lines}


def tp_connect_group(target, group=None) -> None:
    """Connect this process's rank of a tensor-parallel group (one process per
    GPU): all-gather every rank's IPC handle over torch.distributed (any
    backend) and open them in rank order (include/duodec_b200.h dd_tp_connect)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world != target.tp_size or dist.get_rank(group) != target.tp_rank:
        raise ConfigError("process group rank / size must match the target's tp_rank / tp_size")
    handles = [None] * world
    dist.all_gather_object(handles, target.tp_handle(), group=group)
    target.tp_connect(handles)


def run_generation(target, draft: Optional[Draft], prompt: Sequence[int],
                   config: EngineConfig) -> GenerationResult:
    """run_generation (proj/src/engine.cpp:514-532) through dd_engine_run.

    `target` is a Target, or the rank-ordered list of a connected
    tensor-parallel group driven by this process (dd_engine_run_tp)."""
    p = _i32(prompt)
    cap = config.max_new_tokens + config.budget_hard_cap + 8
    toks = np.zeros(cap, dtype=np.int32)
    iters = (_L.IterationRecordC * cap)()
    r = _L.GenerationResultC()
    r.tokens = _i32p(toks)
    r.max_tokens = cap
    r.iterations = iters
    r.max_iterations = cap
    cfg = config.to_c()
    if isinstance(target, (list, tuple)):
        arr = (C.c_void_p * len(target))(*[t.h.value for t in target])
        _check(_L.lib().dd_engine_run_tp(arr, len(target), draft.h if draft else None,
                                         C.byref(cfg), _i32p(p), len(p), C.byref(r)), target[0].h)
    else:
        _check(_L.lib().dd_engine_run(target.h, draft.h if draft else None, C.byref(cfg),
                                      _i32p(p), len(p), C.byref(r)), target.h)
    out = GenerationResult(tokens=[int(x) for x in toks[:r.n_tokens]], ttft_ms=r.ttft_ms,
                           total_ms=r.total_ms, tps=r.tps, prefill_ms=r.prefill_ms,
                           budget=r.budget_used, device_ms=r.device_ms, h2d_bytes=r.h2d_bytes,
                           d2h_bytes=r.d2h_bytes, gpu_launches=r.gpu_launches,
                           device_ttft_ms=r.device_ttft_ms)
    for i in range(r.n_iterations):
        it = iters[i]
        out.iterations.append(IterationRecord(it.draft_ms, it.target_ms, it.verify_ms, it.comm_ms,
                                              it.tokens_processed, it.sequence_count, it.accepted,
                                              it.width))
    return out


def run_vanilla(target, prompt, config):
    return run_generation(target, None, prompt, EngineConfig(**{**config.__dict__, "mode": "vanilla"}))


def run_sps(target, draft, prompt, config):
    return run_generation(target, draft, prompt, EngineConfig(**{**config.__dict__, "mode": "sps"}))


def run_duo(target, draft, prompt, config):
    return run_generation(target, draft, prompt, EngineConfig(**{**config.__dict__, "mode": "duo"}))


def calibrate(target: Target, draft: Draft, probe_len: int = 8, trials: int = 12,
              hard_cap: int = 256):
    """calibrate + choose_budget (proj/src/engine.cpp:534-582) -> (c, budget)."""
    c = C.c_double()
    b = C.c_int()
    _check(_L.lib().dd_calibrate(target.h, draft.h, probe_len, trials, hard_cap, C.byref(c),
                                 C.byref(b)), target.h)
    return c.value, b.value


def choose_budget(c: float) -> int:
    """proj/src/engine.cpp:580-582: max(2, lround(c))."""
    import math
    return max(2, int(math.floor(c + 0.5)))
