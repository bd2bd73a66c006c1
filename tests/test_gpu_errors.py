"""Error behaviour of the boundary on the GPU (-m gpu): every misuse returns a
status code (re-raised as the reference's exception classes, engine.hpp:29-34)
and leaves the context usable - no CPU fallback, no silent clamping."""
import pytest

from paper_2503_00784_b200 import (SHAPES, ConfigError, Draft, EngineConfig, StateError, Target,
                                   run_generation)
from paper_2503_00784_b200 import _lib as L

pytestmark = pytest.mark.gpu

TINY = SHAPES["tiny"]
PLANT = dict(plant_seed=7, alpha=0.5, gain=1.0, emb_std=1.0)


@pytest.fixture(scope="module")
def tgt():
    t = Target(TINY, weight_seed=3, plant=PLANT, max_seq=64)
    yield t
    t.close()


def test_pass_width_and_capacity_limits(tgt):
    tgt.truncate(0)
    with pytest.raises(ConfigError):
        tgt.score([])                       # W = 0
    with pytest.raises(ConfigError):
        tgt.score([1] * 257)                # W > 256
    tgt.prefill(list(range(60)))
    with pytest.raises(ConfigError):
        tgt.score([1] * 8)                  # 60 + 8 > max_seq (64)
    assert tgt.kv_len() == 60               # the failed pass appended nothing
    tgt.score([1, 2, 3, 4])                 # exactly at capacity
    assert tgt.kv_len() == 64


def test_bad_tokens_and_truncate(tgt):
    tgt.truncate(0)
    with pytest.raises(ConfigError):
        tgt.score([TINY["vocab"]])          # outside the vocabulary
    with pytest.raises(ConfigError):
        tgt.score([-1])
    tgt.prefill([1, 2, 3])
    with pytest.raises(ConfigError):
        tgt.truncate(4)                     # beyond n_cached
    with pytest.raises(ConfigError):
        tgt.truncate(-1)
    assert tgt.kv_len() == 3


def test_verify_state_errors(tgt):
    tgt.truncate(0)
    tgt.prefill([5, 6, 7])                  # a prefill leaves no scored pass
    with pytest.raises(StateError):
        tgt.verify(L.DD_MODE_VANILLA, greedy=True, q_onehot=True)
    tgt.score([8, 9])
    with pytest.raises(ConfigError):        # tail longer than the scored pass allows
        tgt.verify(L.DD_MODE_DUO, tail_len=2, firsts=[1], greedy=True, q_onehot=True)
    with pytest.raises(ConfigError):        # bundle token outside the vocabulary
        tgt.verify(L.DD_MODE_DUO, tail_len=1, firsts=[TINY["vocab"]], greedy=True, q_onehot=True)
    with pytest.raises(ConfigError):        # non-positive temperature when sampling
        tgt.verify(L.DD_MODE_VANILLA, temperature=0.0)
    out = tgt.verify(L.DD_MODE_DUO, tail_len=1, firsts=[1], greedy=True, q_onehot=True)
    assert out["reject_index"] in (-1, 0)  # still usable after the failures


def test_engine_config_validation(tgt):
    prompt = list(range(10))
    for bad in (dict(budget=1), dict(budget=300), dict(max_sequences=0), dict(max_new_tokens=0),
                dict(greedy=False, temperature=0.0)):
        cfg = EngineConfig(mode="vanilla", **{**dict(budget=4, max_new_tokens=4, greedy=True), **bad})
        with pytest.raises(ConfigError):
            run_generation(tgt, None, prompt, cfg)
    with pytest.raises(ConfigError):        # sps / duo need a draft
        run_generation(tgt, None, prompt, EngineConfig(mode="duo", budget=4, max_new_tokens=4))
    res = run_generation(tgt, None, prompt, EngineConfig(mode="vanilla", budget=4, max_new_tokens=4,
                                                           greedy=True))
    assert len(res.tokens) == 4


def test_tensor_parallel_misuse():
    ranks = [Target(TINY, weight_seed=3, plant=PLANT, max_seq=64, tp_rank=r, tp_size=2)
             for r in range(2)]
    with pytest.raises(StateError):         # no pass before the ranks are connected
        ranks[0].score([1])
    with pytest.raises(ConfigError):        # one handle per rank
        ranks[0].tp_connect([ranks[0].tp_handle()])
    with pytest.raises(ConfigError):        # ranks listed out of order
        Target.tp_connect_local([ranks[1], ranks[0]])
    Target.tp_connect_local(ranks)
    drf = Draft(SHAPES["llama_68m"], weight_seed=4, plant=PLANT, threads=2)
    with pytest.raises(ConfigError):        # calibration times single-rank passes
        run_generation(ranks, drf, list(range(8)),
                       EngineConfig(mode="duo", budget=4, max_new_tokens=4, greedy=True,
                                    budget_policy="calibrated"))
    res = run_generation(ranks, drf, list(range(8)),
                         EngineConfig(mode="duo", budget=4, max_new_tokens=8, greedy=True))
    assert len(res.tokens) >= 8
    drf.close()
    for t in ranks:
        t.close()
    with pytest.raises(ConfigError):        # tp_size must divide the heads
        Target(dict(TINY, n_heads=6, n_kv_heads=6), max_seq=64, tp_rank=0, tp_size=4)
