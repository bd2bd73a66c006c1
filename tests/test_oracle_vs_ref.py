"""The restated protocol vs the compiled reference library, randomized
(needs oracle/_ref/libduodec_ref.so, built from /root/reference by oracle/Makefile)."""
import numpy as np
import pytest

from oracle import protocol as P
from oracle import refdll

pytestmark = pytest.mark.skipif(not refdll.available(), reason="reference library not built")


def rand_dist(rng, V, conc=0.4):
    p = rng.gamma(conc, size=V)
    return p / p.sum()


def test_verify_randomized():
    rng = np.random.default_rng(7)
    for _ in range(1500):
        V = int(rng.integers(2, 40))
        L = int(rng.integers(0, 7))
        p = np.stack([rand_dist(rng, V) for _ in range(L + 1)])
        q = np.stack([rand_dist(rng, V) for _ in range(L)]) if L else np.zeros((0, V))
        toks = [int(rng.choice(V, p=q[j])) for j in range(L)]
        seed, cnt = int(rng.integers(1, 2 ** 62)), int(rng.integers(0, 10))
        if L:
            rs = P.RandomStream(seed, cnt)
            o = P.verify_prefix(toks, q, p[:L], rs)
            assert refdll.verify_prefix(toks, q, p[:L], seed, cnt) == (
                o.all_accepted, o.reject_index, o.resample, rs.counter)
        firsts = [int(x) for x in rng.choice(V, size=min(V, int(rng.integers(1, 9))), replace=False)]
        rs = P.RandomStream(seed, cnt)
        b = P.verify_bundle(firsts, p[L], rs)
        assert refdll.verify_bundle(firsts, p[L], seed, cnt) == (b.accepted, b.seq_index, b.fallback,
                                                                rs.counter)
        rs = P.RandomStream(seed, cnt)
        a, n = P.sps_verify(toks, q, p, rs)
        assert refdll.sps_verify(toks, q, p, seed, cnt) == (a, n, rs.counter)


def test_zero_mass_paths():
    # residual zero mass -> p; bundle removing all mass -> reset to p_next
    p = np.array([1.0, 0.0, 0.0])
    for seed in range(1, 50):
        assert refdll.verify_bundle([0], p, seed, 0)[:3] == (True, 0, -1)
        rs = P.RandomStream(seed)
        o = P.verify_bundle([1, 2], p, rs)
        assert refdll.verify_bundle([1, 2], p, seed, 0) == (o.accepted, o.seq_index, o.fallback,
                                                            rs.counter)


def random_markov(rng, V, order):
    lines = [f"vocab {V}", f"order {order}"]
    for ctx in range(V):
        row = rand_dist(rng, V, 0.6)
        lines.append(f"ctx {ctx} : " + " ".join(f"{x:.17g}" for x in row))
    d = rand_dist(rng, V, 0.6)
    lines.append("default : " + " ".join(f"{x:.17g}" for x in d))
    return "\n".join(lines)


@pytest.mark.parametrize("seed", range(6))
def test_engine_randomized_models(seed):
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(3, 9))
    t_txt, d_txt = random_markov(rng, V, 1), random_markov(rng, V, 1)
    T, D = refdll.Model(t_txt), refdll.Model(d_txt)
    temp = [1.0, 0.6, 1.3][seed % 3]
    pt, pd = P.MarkovModel(t_txt, temp), P.MarkovModel(d_txt, temp)
    for mode in ("vanilla", "sps", "duo"):
        budget, smax = int(rng.integers(2, 12)), int(rng.integers(1, 6))
        r = refdll.run(mode, T, D if mode != "vanilla" else None, [0, 1], budget=budget,
                       max_sequences=smax, max_new_tokens=40, temperature=temp, draft_seed=seed + 1,
                       verify_seed=seed + 7, threaded=(seed % 2 == 0))
        if mode == "vanilla":
            o = P.run_vanilla(pt, [0, 1], 40, verify_seed=seed + 7)
        elif mode == "sps":
            o = P.run_sps(pt, pd, [0, 1], budget, 40, seed + 1, seed + 7)
        else:
            o = P.run_duo(pt, pd, [0, 1], budget, smax, 40, seed + 1, seed + 7)
        assert o.tokens == r["tokens"], mode
        assert [it.tokens_processed for it in o.iterations] == r["iter_tokens"]
        assert o.total_ms == pytest.approx(r["total_ms"], rel=1e-12)


def test_onehot_target_gives_argmax_chain():
    """SURVEY.md §4 probe: a one-hot target reduces every mode to its argmax chain."""
    rng = np.random.default_rng(3)
    V = 6
    rows = []
    for ctx in range(V):
        r = np.zeros(V)
        r[int(rng.integers(0, V))] = 1.0
        rows.append(f"ctx {ctx} : " + " ".join(str(x) for x in r))
    t_txt = f"vocab {V}\norder 1\n" + "\n".join(rows) + "\ndefault : " + " ".join(
        ["1"] + ["0"] * (V - 1))
    d_txt = random_markov(rng, V, 1)
    T, D = refdll.Model(t_txt), refdll.Model(d_txt)
    chain, c = [], 0
    pt = P.MarkovModel(t_txt)
    ctx = [0]
    for _ in range(20):
        c = int(np.argmax(pt(ctx)))
        chain.append(c)
        ctx.append(c)
    for mode in ("vanilla", "sps", "duo"):
        for g in (2, 8, 24):
            for s in range(1, 4):
                r = refdll.run(mode, T, D if mode != "vanilla" else None, [0], budget=g,
                               max_new_tokens=20, draft_seed=s, verify_seed=s + 10)
                assert r["tokens"][:20] == chain


def test_fidelity_duo_small():
    """SPEC acceptance criterion (fidelity): duo's token law equals the target's."""
    import ctypes as C
    t_txt = open("/root/reference/proj/data/models/target_demo.model").read() \
        if refdll.available() else None
    d_txt = open("/root/reference/proj/data/models/draft_demo.model").read()
    T, D = refdll.Model(t_txt), refdll.Model(d_txt)
    tv = np.zeros(3)
    mx = refdll.lib().ref_run_fidelity(2, T.h, D.h, np.array([0, 1, 2], dtype=np.int32), 3, 8, 4,
                                       1.0, 20000, 3, tv)
    assert mx <= 0.01
