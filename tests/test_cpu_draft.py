"""The product's CPU draft model (W8A8 VNNI / AMX, 4-bit LM head, host cores) vs the oracle."""
import numpy as np
import pytest

from oracle.llama import OracleLlama
from paper_2503_00784_b200 import Draft

SHAPE = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=640,
             vocab=1024, rms_eps=1e-5, rope_theta=1e4)
PLANT = dict(plant_seed=3, alpha=0.5, gain=1.0, emb_std=1.0)


@pytest.fixture(scope="module")
def draft(native):
    import ctypes
    try:
        d = Draft(SHAPE, weight_seed=31, plant=PLANT, threads=4, max_seq=256)
    except Exception as e:  # host without AVX-512 BF16: single native path
        pytest.skip(str(e))
    yield d
    d.close()


def test_draft_logits_match_oracle(draft):
    orc = OracleLlama(SHAPE, weight_seed=31, plant=PLANT, max_seq=256, threads=4, w8a8=True)
    rng = np.random.default_rng(1)
    ctx = rng.integers(0, SHAPE["vocab"], 50).tolist()
    o = orc.forward(ctx)
    for n in (1, 7, 30, 50):  # prefix reuse, branch forks, re-extension
        g = draft.logits(ctx[:n])
        rel = np.abs(g - o[n - 1]).max() / np.abs(o[n - 1]).max()
        assert rel < 1e-5, (n, rel)  # integer dots are exact; only the fp epilogue order could differ
    # fork: different continuation then back
    g1 = draft.logits(ctx[:20] + [5, 6])
    g2 = draft.logits(ctx[:25])
    assert np.abs(g2 - o[24]).max() / np.abs(o[24]).max() < 1e-5
    orc.close()


def test_draft_time_token(draft):
    assert draft.time_token(10) > 0.0


def test_draft_prefill_bit_exact(draft):
    """Long prefill (token-blocked VNNI matmuls, 16-lane attention and the
    deterministic exp) equals the oracle's W8A8 mode bit for bit."""
    orc = OracleLlama(SHAPE, weight_seed=31, plant=PLANT, max_seq=256, threads=4, w8a8=True)
    ctx = np.random.default_rng(2).integers(0, SHAPE["vocab"], 230).tolist()
    o = orc.forward(ctx)
    for n in (230, 3, 120, 229):
        assert np.array_equal(draft.logits(ctx[:n]), o[n - 1]), n
    orc.close()


def test_draft_prefill_vnni_path_bit_exact(draft, tmp_path):
    """The VNNI prefill path (DD_DRAFT_AMX=0, the fallback when AMX is absent)
    gives the same bits as the oracle too (the AMX path runs above when present)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "from paper_2503_00784_b200 import Draft\n"
        "d = Draft(%r, weight_seed=31, plant=%r, threads=4, max_seq=256)\n"
        "ctx = np.random.default_rng(2).integers(0, %d, 230).tolist()\n"
        "np.save(%r, d.logits(ctx))\n" % (str(root), SHAPE, PLANT, SHAPE["vocab"], str(tmp_path / "g.npy")))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "DD_DRAFT_AMX": "0"},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    orc = OracleLlama(SHAPE, weight_seed=31, plant=PLANT, max_seq=256, threads=4, w8a8=True)
    o = orc.forward(np.random.default_rng(2).integers(0, SHAPE["vocab"], 230).tolist())
    orc.close()
    assert np.array_equal(np.load(tmp_path / "g.npy"), o[-1])


@pytest.mark.parametrize("budget,s_max,temp", [(8, 4, 1.0), (6, 8, 1.0), (5, 2, 0.7),
                                               (12, 4, 1.5), (3, 4, 1.0), (16, 16, 2.0)])
def test_engine_draft_dynamic_matches_reference(draft, budget, s_max, temp):
    """The engine's C++ draft_dynamic (csrc/engine.cpp) vs the restated
    reference drafting (oracle/protocol.py draft_dynamic, pinned to the
    compiled reference by test_golden / test_oracle_vs_ref), with the same q
    rows: sequence count, admission order, even split with the remainder on
    the top sequence, sampled continuations in sequence-major draw order,
    probe reuse (forward count), theta, and the draft stream's counter
    (proj/src/drafting.cpp:71-136)."""
    from oracle import protocol as P
    rng = np.random.default_rng(budget * 100 + s_max)
    multi = 0
    for trial in range(12):
        ctx = rng.integers(0, SHAPE["vocab"], int(rng.integers(3, 40))).tolist()
        seed, counter = int(rng.integers(1, 2**63)), int(rng.integers(0, 1000))
        got = draft.draft_dynamic(ctx, budget, s_max, seed, counter, temperature=temp)

        def fwd(c):
            return draft.dist(c, temperature=temp)[0].astype(np.float64)
        rs = P.RandomStream(seed, counter)
        want = P.draft_dynamic(fwd, ctx, budget, s_max, rs)
        assert got["seqs"] == [list(s.tokens) for s in want.sequences], trial
        assert got["threshold"] == want.threshold
        assert got["forwards"] == want.forwards_used
        assert got["counter"] == rs.counter
        assert sum(map(len, got["seqs"])) == budget
        multi += len(got["seqs"]) > 1
    if s_max > 1 and budget > 1:
        assert multi > 0, "no multi-sequence bundle exercised"


def test_engine_draft_dynamic_greedy(draft):
    """Greedy drafting: one sequence, the draft's argmax chain, no draws."""
    ctx = [5, 17, 300, 2]
    got = draft.draft_dynamic(ctx, 6, 4, seed=1, counter=3, greedy=True)
    assert len(got["seqs"]) == 1 and got["counter"] == 3 + 5
    chain, c = [], list(ctx)
    for _ in range(6):
        t = int(np.argmax(draft.logits(c)))
        chain.append(t)
        c.append(t)
    assert got["seqs"][0] == chain
