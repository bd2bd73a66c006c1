"""ctypes loader for oracle/_ref/libduodec_ref.so — TEST INFRASTRUCTURE ONLY.

The reference library is compiled from /root/reference sources by
oracle/Makefile (this container only).  It is loaded with
DUODEC_KERNELS=scalar so its sums are left-to-right (kernels_scalar.cpp), the
order oracle/protocol.py restates.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libduodec_ref.so"
_lib = None

i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        os.environ["DUODEC_KERNELS"] = "scalar"
        L = C.CDLL(str(LIB_PATH))
        u64, i32, f64, vp = C.c_uint64, C.c_int, C.c_double, C.c_void_p
        ip, dp, up = C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_uint64)
        L.ref_rng_u64.argtypes = [u64, u64, i32, u64p]
        L.ref_rng_uniform.argtypes = [u64, u64, i32, f64p]
        L.ref_derive_seed.argtypes = [u64, u64]
        L.ref_derive_seed.restype = u64
        L.ref_sample.argtypes = [f64p, i32, f64]
        L.ref_argmax.argtypes = [f64p, i32]
        L.ref_accept_test.argtypes = [f64, f64, f64]
        L.ref_residual.argtypes = [f64p, f64p, i32, f64p]
        L.ref_verify_prefix.argtypes = [i32p, f64p, f64p, i32, i32, u64, u64, ip, ip, ip, up]
        L.ref_verify_bundle.argtypes = [i32p, i32, f64p, i32, u64, u64, ip, ip, ip, up]
        L.ref_sps_verify.argtypes = [i32p, f64p, f64p, i32, i32, u64, u64, ip, ip, up]
        L.ref_model_parse.argtypes = [C.c_char_p]
        L.ref_model_parse.restype = vp
        L.ref_model_free.argtypes = [vp]
        L.ref_model_with_temperature.argtypes = [vp, f64]
        L.ref_model_with_temperature.restype = vp
        L.ref_model_forward.argtypes = [vp, i32p, i32, f64p]
        L.ref_draft_dynamic.argtypes = [vp, i32p, i32, i32, i32, u64, u64, i32p, i32p, f64p, dp, ip, up]
        L.ref_run.argtypes = [i32, vp, vp, i32p, i32, i32, i32, i32, f64, u64, u64, i32, i32, f64p, i32,
                              i32p, i32, ip, dp, dp, dp, i32p, i32p, i32p, i32, ip, ip]
        L.ref_calibrate_sim.argtypes = [vp, vp, i32, i32, f64p]
        L.ref_calibrate_sim.restype = f64
        L.ref_choose_budget.argtypes = [f64]
        L.ref_run_fidelity.argtypes = [i32, vp, vp, i32p, i32, i32, i32, f64, i32, i32, f64p]
        L.ref_run_fidelity.restype = f64
        L.ref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _ints(*n):
    return [C.c_int() for _ in range(n[0])]


def rng_u64(seed, skip, n):
    out = np.zeros(n, dtype=np.uint64)
    lib().ref_rng_u64(seed, skip, n, out)
    return [int(x) for x in out]


def rng_uniform(seed, skip, n):
    out = np.zeros(n, dtype=np.float64)
    lib().ref_rng_uniform(seed, skip, n, out)
    return out


def derive_seed(base, index):
    return int(lib().ref_derive_seed(base, index))


def sample(p, u):
    p = np.ascontiguousarray(p, dtype=np.float64)
    return lib().ref_sample(p, len(p), u)


def verify_prefix(tokens, q_rows, p_rows, seed, counter):
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    q = np.ascontiguousarray(q_rows, dtype=np.float64)
    p = np.ascontiguousarray(p_rows, dtype=np.float64)
    a, k, r = C.c_int(), C.c_int(), C.c_int()
    c = C.c_uint64()
    lib().ref_verify_prefix(t, q, p, len(t), q.shape[-1], seed, counter, C.byref(a), C.byref(k),
                            C.byref(r), C.byref(c))
    return bool(a.value), k.value, r.value, c.value


def verify_bundle(firsts, p_next, seed, counter):
    f = np.ascontiguousarray(firsts, dtype=np.int32)
    p = np.ascontiguousarray(p_next, dtype=np.float64)
    a, i, fb = C.c_int(), C.c_int(), C.c_int()
    c = C.c_uint64()
    lib().ref_verify_bundle(f, len(f), p, len(p), seed, counter, C.byref(a), C.byref(i),
                            C.byref(fb), C.byref(c))
    return bool(a.value), i.value, fb.value, c.value


def sps_verify(tokens, q_rows, p_rows, seed, counter):
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    q = np.ascontiguousarray(q_rows, dtype=np.float64).reshape(len(t), -1) if len(t) else \
        np.zeros((0, np.asarray(p_rows).shape[-1]))
    p = np.ascontiguousarray(p_rows, dtype=np.float64)
    a, n = C.c_int(), C.c_int()
    c = C.c_uint64()
    lib().ref_sps_verify(t, np.ascontiguousarray(q), p, len(t), p.shape[-1], seed, counter,
                         C.byref(a), C.byref(n), C.byref(c))
    return a.value, n.value, c.value


class Model:
    def __init__(self, text: str):
        self.h = lib().ref_model_parse(text.encode())
        if not self.h:
            raise ValueError(lib().ref_last_error().decode())
        self.vocab = lib().ref_model_vocab(C.c_void_p(self.h))

    def __call__(self, ctx):
        out = np.zeros(self.vocab, dtype=np.float64)
        c = np.ascontiguousarray(ctx, dtype=np.int32)
        lib().ref_model_forward(self.h, c, len(c), out)
        return out

    def with_temperature(self, t):
        m = Model.__new__(Model)
        m.h = lib().ref_model_with_temperature(self.h, t)
        m.vocab = self.vocab
        return m

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_model_free(self.h)


def draft_dynamic(model: Model, ctx, budget, max_seq, seed, counter):
    c = np.ascontiguousarray(ctx, dtype=np.int32)
    lens = np.zeros(64, dtype=np.int32)
    toks = np.zeros(max(budget, 1) + 8, dtype=np.int32)
    fp = np.zeros(64, dtype=np.float64)
    th = C.c_double()
    fw = C.c_int()
    cnt = C.c_uint64()
    s = lib().ref_draft_dynamic(model.h, c, len(c), budget, max_seq, seed, counter, lens, toks, fp,
                                C.byref(th), C.byref(fw), C.byref(cnt))
    seqs, off = [], 0
    for i in range(s):
        seqs.append([int(x) for x in toks[off:off + lens[i]]])
        off += lens[i]
    return dict(sequences=seqs, first_probs=[float(x) for x in fp[:s]], threshold=th.value,
                forwards=fw.value, counter=cnt.value)


def run(mode, target: Model, draft, prompt, budget=24, max_sequences=8, max_new_tokens=128,
        temperature=1.0, draft_seed=1, verify_seed=2, calibrated=False, threaded=True,
        profile=(1.0, 24.0, 0.0, 0.2), wall=False):
    p = np.ascontiguousarray(prompt, dtype=np.int32)
    cap = max_new_tokens + 512
    out = np.zeros(cap, dtype=np.int32)
    it_tok = np.zeros(cap, dtype=np.int32)
    it_seq = np.zeros(cap, dtype=np.int32)
    it_acc = np.zeros(cap, dtype=np.int32)
    n_out, n_it, bud = C.c_int(), C.c_int(), C.c_int()
    ttft, total, tps = C.c_double(), C.c_double(), C.c_double()
    mode_i = {"vanilla": 0, "sps": 1, "duo": 2}[mode]
    rc = lib().ref_run(mode_i, target.h, draft.h if draft is not None else None, p, len(p), budget,
                       max_sequences, max_new_tokens, temperature, draft_seed, verify_seed,
                       int(calibrated), int(threaded), np.asarray(profile, dtype=np.float64),
                       int(wall), out, cap, C.byref(n_out), C.byref(ttft), C.byref(total),
                       C.byref(tps), it_tok, it_seq, it_acc, cap, C.byref(n_it), C.byref(bud))
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())
    n = n_it.value
    return dict(tokens=[int(x) for x in out[:n_out.value]], ttft_ms=ttft.value,
                total_ms=total.value, tps=tps.value,
                iter_tokens=[int(x) for x in it_tok[:n]], iter_seqs=[int(x) for x in it_seq[:n]],
                iter_accepted=[int(x) for x in it_acc[:n]], budget=bud.value)
