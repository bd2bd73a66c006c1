"""Sampling-mode parity of the GPU engine (-m gpu).

The reference checks its lossless-sampling claim statistically: a Monte-Carlo
run over derive_seed streams against the exact law (proj/src/fidelity.cpp:
43-89; SPEC.md:548-555 criteria 1, 3, 7, 8).  Here the product engine
(dd_engine_run: GPU target + W8A8 CPU draft, draft_dynamic, the fused
acceptance kernel) runs the same 2000 seeded streams as the restated reference
loop over the CPU oracle (oracle/cpu_engine.py: oracle target + the oracle's
W8A8 draft, bit-identical to the product draft's logits), at a temperature and
plant where dynamic drafting admits several sequences in most iterations:

- the two engines emit the identical token stream on >= 95% of the seeds
  (every draw is index-addressed; streams can only diverge where the GPU's
  bf16 logits move a ratio test or an inverse-CDF crossing),
- accepted-length and sequence-count histograms and the first four
  positions' token marginals agree within TV <= 0.02.

Plus the WorkerHooks determinism criterion (engine.hpp:36-41): threaded
execution with scheduling jitter emits the sequential execution's tokens.
"""
import numpy as np
import pytest

from oracle import protocol as P
from oracle.cpu_engine import run_cpu
from oracle.llama import OracleLlama
from paper_2503_00784_b200 import Draft, EngineConfig, Target, run_generation

pytestmark = pytest.mark.gpu

T_SHAPE = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=512,
               vocab=1024, rms_eps=1e-5, rope_theta=1e4)
D_SHAPE = dict(n_layers=1, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=512,
               vocab=1024, rms_eps=1e-5, rope_theta=1e4)
PLANT = dict(plant_seed=5, alpha=0.4, gain=0.6, emb_std=1.0)
TEMP = 1.0
BUDGET, S_MAX, NEW = 6, 4, 12
N_STREAMS = 2000
BASE = 0x5EED


def tv(a, b):
    keys = set(a) | set(b)
    na, nb = sum(a.values()), sum(b.values())
    return 0.5 * sum(abs(a.get(k, 0) / na - b.get(k, 0) / nb) for k in keys)


def hist(xs):
    h = {}
    for x in xs:
        h[x] = h.get(x, 0) + 1
    return h


@pytest.fixture(scope="module")
def models():
    tgt = Target(T_SHAPE, weight_seed=41, plant=PLANT, max_seq=256)
    drf = Draft(D_SHAPE, weight_seed=42, plant=PLANT, threads=4, max_seq=256)
    otg = OracleLlama(T_SHAPE, weight_seed=41, plant=PLANT, max_seq=256, threads=4)
    odr = OracleLlama(D_SHAPE, weight_seed=42, plant=PLANT, max_seq=256, threads=4, w8a8=True)
    yield tgt, drf, otg, odr
    for m in (tgt, drf, otg, odr):
        m.close()


PROMPT = [int(x) for x in np.random.default_rng(2).integers(0, 1024, 16)]


def test_sampled_streams_match_reference_loop(models):
    tgt, drf, otg, odr = models
    g_tok, c_tok, g_rec, c_rec = [], [], [], []
    for i in range(N_STREAMS):
        ds, vs = P.derive_seed(BASE, 2 * i), P.derive_seed(BASE, 2 * i + 1)
        cfg = EngineConfig(mode="duo", budget=BUDGET, max_sequences=S_MAX, max_new_tokens=NEW,
                           greedy=False, temperature=TEMP, draft_seed=ds, verify_seed=vs,
                           threaded=False)
        r = run_generation(tgt, drf, PROMPT, cfg)
        g_tok.append(r.tokens[:NEW])
        g_rec += [(it.tokens_processed, it.accepted, it.sequence_count) for it in r.iterations]
        c = run_cpu("duo", otg, odr, PROMPT, BUDGET, S_MAX, NEW, greedy=False, temperature=TEMP,
                    draft_seed=ds, verify_seed=vs, threaded=False)
        c_tok.append(c["tokens"][:NEW])
        c_rec += c["records"]
    same = np.mean([a == b for a, b in zip(g_tok, c_tok)])
    multi = np.mean([r[2] > 1 for r in c_rec])
    t_acc = tv(hist(r[1] for r in g_rec), hist(r[1] for r in c_rec))
    t_seq = tv(hist(r[2] for r in g_rec), hist(r[2] for r in c_rec))
    t_pos = [tv(hist(t[k] for t in g_tok), hist(t[k] for t in c_tok)) for k in range(4)]
    print(f"identical streams {same:.4f}, multi-sequence iterations {multi:.3f}, TV accepted "
          f"{t_acc:.4f}, TV sequences {t_seq:.4f}, TV positions {np.round(t_pos, 4)}")
    assert multi >= 0.3, f"only {multi:.2f} of the iterations drafted several sequences"
    assert same >= 0.95, f"only {same:.3f} of the streams match"
    assert t_acc <= 0.02 and t_seq <= 0.02 and max(t_pos) <= 0.02


@pytest.mark.parametrize("jitter_seed", [1, 2, 3])
def test_threaded_jitter_equals_sequential(models, jitter_seed):
    """engine.hpp:36-41 WorkerHooks: random delays before each draft step and
    each target step of the threaded execution do not change the output."""
    tgt, drf, _, _ = models
    base = dict(mode="duo", budget=BUDGET, max_sequences=S_MAX, max_new_tokens=40, greedy=False,
                temperature=TEMP, draft_seed=11, verify_seed=12)
    seq = run_generation(tgt, drf, PROMPT, EngineConfig(**base, threaded=False))
    thr = run_generation(tgt, drf, PROMPT, EngineConfig(**base, threaded=True,
                                                        jitter_seed=jitter_seed, jitter_max_us=400))
    assert thr.tokens == seq.tokens
    assert [(i.tokens_processed, i.accepted, i.sequence_count) for i in thr.iterations] == \
           [(i.tokens_processed, i.accepted, i.sequence_count) for i in seq.iterations]
