"""The all-CPU restated reference loop (oracle/cpu_engine.py, the bench's CPU
baseline and --impl reference arm): threaded duo == sequential duo (each role
owns its RandomStream, proj/src/engine.cpp:425-440), and under greedy every
mode emits the target's argmax chain."""
import numpy as np
import pytest

from oracle.cpu_engine import run_cpu
from oracle.llama import OracleLlama

T_SHAPE = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=640,
               vocab=1024, rms_eps=1e-5, rope_theta=1e4)
D_SHAPE = dict(T_SHAPE, n_layers=1, d_model=128, n_heads=2, n_kv_heads=2, ffn_dim=256)
PLANT = dict(plant_seed=3, alpha=0.8, gain=1.0, emb_std=1.0)


@pytest.fixture(scope="module")
def models():
    t = OracleLlama(T_SHAPE, weight_seed=1, plant=PLANT, max_seq=256, threads=2)
    d = OracleLlama(D_SHAPE, weight_seed=2, plant=PLANT, max_seq=256, threads=2)
    yield t, d
    t.close()
    d.close()


@pytest.mark.parametrize("greedy", [True, False])
def test_threaded_duo_equals_sequential(models, greedy):
    t, d = models
    prompt = np.random.default_rng(0).integers(0, 1024, 12).tolist()
    a = run_cpu("duo", t, d, prompt, 6, 4, 40, greedy=greedy, threaded=True)
    b = run_cpu("duo", t, d, prompt, 6, 4, 40, greedy=greedy, threaded=False)
    assert a["tokens"] == b["tokens"]
    assert a["iterations"] == b["iterations"]


def test_greedy_modes_emit_argmax_chain(models):
    t, d = models
    prompt = np.random.default_rng(1).integers(0, 1024, 10).tolist()
    out = {m: run_cpu(m, t, d, prompt, 5, 4, 30, greedy=True)["tokens"][:30]
           for m in ("vanilla", "sps", "duo")}
    assert out["duo"] == out["vanilla"] and out["sps"] == out["vanilla"]
