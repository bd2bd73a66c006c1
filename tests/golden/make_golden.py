"""Generate tests/golden/*.json from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libduodec_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile):  python tests/golden/make_golden.py
The fixtures let tests/test_golden.py pin the oracle restatement without the
reference (e.g. on the GPU box).
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import refdll  # noqa: E402

OUT = Path(__file__).resolve().parent
MODELS = Path("/root/reference/proj/data/models")


def rand_dist(rng, V):
    p = rng.gamma(0.4, size=V)
    return p / p.sum()


def main():
    g = {}
    g["rng"] = {str(s): {"u64": [str(x) for x in refdll.rng_u64(s, 0, 8)],
                         "uniform": refdll.rng_uniform(s, 0, 8).tolist()} for s in (1, 2, 12345)}
    g["derive_seed"] = [[b, i, str(refdll.derive_seed(b, i))] for b in (1, 2, 99) for i in (0, 1, 7)]
    rng = np.random.default_rng(2024)
    cases = []
    for k in range(120):
        V = int(rng.integers(2, 24))
        L = int(rng.integers(1, 6))
        p = np.stack([rand_dist(rng, V) for _ in range(L + 1)])
        q = np.stack([rand_dist(rng, V) for _ in range(L)])
        toks = [int(rng.choice(V, p=q[j])) for j in range(L)]
        firsts = [int(x) for x in rng.choice(V, size=min(V, int(rng.integers(1, 5))), replace=False)]
        seed, counter = int(rng.integers(1, 2 ** 62)), int(rng.integers(0, 20))
        vp = refdll.verify_prefix(toks, q, p[:L], seed, counter)
        vb = refdll.verify_bundle(firsts, p[L], seed, counter)
        sp = refdll.sps_verify(toks, q, p, seed, counter)
        cases.append({"V": V, "p": p.tolist(), "q": q.tolist(), "tokens": toks, "firsts": firsts,
                      "seed": str(seed), "counter": counter,
                      "verify_prefix": [int(vp[0]), vp[1], vp[2], str(vp[3])],
                      "verify_bundle": [int(vb[0]), vb[1], vb[2], str(vb[3])],
                      "sps_verify": [sp[0], sp[1], str(sp[2])]})
    g["verify_cases"] = cases
    t_txt = (MODELS / "target_demo.model").read_text()
    d_txt = (MODELS / "draft_demo.model").read_text()
    g["models"] = {"target_demo": t_txt, "draft_demo": d_txt}
    T, D = refdll.Model(t_txt), refdll.Model(d_txt)
    runs = []
    for mode in ("vanilla", "sps", "duo"):
        for budget, smax, prof, temp, seeds in [(8, 4, (3.0, 20.0, 0.5, 0.2), 1.0, (1, 2)),
                                                (24, 8, (1.0, 24.0, 0.0, 0.2), 1.0, (1, 2)),
                                                (5, 2, (3.0, 20.0, 0.5, 0.2), 0.7, (11, 12)),
                                                (12, 4, (1.0, 24.0, 0.0, 0.2), 1.5, (5, 9))]:
            r = refdll.run(mode, T, D if mode != "vanilla" else None, [0, 1, 2], budget=budget,
                           max_sequences=smax, max_new_tokens=32, temperature=temp,
                           draft_seed=seeds[0], verify_seed=seeds[1], profile=prof)
            runs.append({"mode": mode, "budget": budget, "max_sequences": smax, "profile": prof,
                         "temperature": temp, "seeds": list(seeds), **r})
    g["engine_runs"] = runs
    drafts = []
    for ctx in ([0], [5, 6], [1, 2, 3], [6], [7, 7]):
        for budget, smax in ((8, 4), (2, 8), (24, 8), (5, 1)):
            drafts.append({"ctx": ctx, "budget": budget, "max_sequences": smax,
                           **refdll.draft_dynamic(D, ctx, budget, smax, 1, 0)})
    g["draft_dynamic"] = drafts
    g["calibrate"] = {"balanced24": refdll.lib().ref_calibrate_sim(T.h, D.h, 8, 12, np.array([1.0, 24.0, 0.0, 0.2])),
                      "figure1": refdll.lib().ref_calibrate_sim(T.h, D.h, 8, 12, np.array([3.0, 20.0, 0.5, 0.2]))}
    g["choose_budget"] = [[c, refdll.lib().ref_choose_budget(c)] for c in (24.0, 5.4, 0.3, 2.5, 7.49, 7.5)]
    (OUT / "reference_golden.json").write_text(json.dumps(g))
    print("wrote", OUT / "reference_golden.json")


if __name__ == "__main__":
    main()
