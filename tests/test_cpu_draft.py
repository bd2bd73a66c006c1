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
