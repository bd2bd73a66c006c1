"""The CPU Llama oracle (oracle/llama_ref.c) vs transformers' LlamaForCausalLM
(fp32, same weights): pins the forward-contract math the reference leaves
abstract (RoPE convention, RMSNorm, SwiGLU, causal attention, KV cache)."""
import numpy as np
import pytest

from oracle.llama import OracleLlama

SHAPE = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=640,
             vocab=512, rms_eps=1e-5, rope_theta=1e4)
GQA = dict(SHAPE, n_heads=8, n_kv_heads=2, head_dim=32)
PLANT = dict(plant_seed=3, alpha=0.5, gain=1.0, emb_std=1.0)


def bits_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def hf_model(orc, shape):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    d, V, F = shape["d_model"], shape["vocab"], shape["ffn_dim"]
    H, Hk, hd = shape["n_heads"], shape["n_kv_heads"], shape["head_dim"]
    cfg = tr.LlamaConfig(vocab_size=V, hidden_size=d, intermediate_size=F,
                         num_hidden_layers=shape["n_layers"], num_attention_heads=H,
                         num_key_value_heads=Hk, head_dim=hd, rms_norm_eps=shape["rms_eps"],
                         rope_theta=shape["rope_theta"], max_position_embeddings=256,
                         tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    m = tr.LlamaForCausalLM(cfg).float().eval()
    sd = {}
    T = lambda a: torch.from_numpy(bits_f32(a).copy())  # noqa: E731
    sd["model.embed_tokens.weight"] = T(orc.tensor(0, 0, V * d)).view(V, d)
    sd["lm_head.weight"] = T(orc.tensor(1, 0, V * d)).view(V, d)
    qd, kvd = H * hd, Hk * hd
    for l in range(shape["n_layers"]):
        qkv = T(orc.tensor(2, l, (qd + 2 * kvd) * d)).view(qd + 2 * kvd, d)
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = qkv[:qd]
        sd[p + "self_attn.k_proj.weight"] = qkv[qd:qd + kvd]
        sd[p + "self_attn.v_proj.weight"] = qkv[qd + kvd:]
        sd[p + "self_attn.o_proj.weight"] = T(orc.tensor(3, l, d * qd)).view(d, qd)
        gu = T(orc.tensor(4, l, 2 * F * d)).view(2 * F, d)
        sd[p + "mlp.gate_proj.weight"] = gu[:F]
        sd[p + "mlp.up_proj.weight"] = gu[F:]
        sd[p + "mlp.down_proj.weight"] = T(orc.tensor(5, l, d * F)).view(d, F)
        sd[p + "input_layernorm.weight"] = torch.ones(d)
        sd[p + "post_attention_layernorm.weight"] = torch.ones(d)
    sd["model.norm.weight"] = torch.ones(d)
    m.load_state_dict(sd, strict=False)
    return m, torch


@pytest.mark.parametrize("shape", [SHAPE, GQA], ids=["mha", "gqa"])
def test_oracle_matches_transformers(shape):
    orc = OracleLlama(shape, weight_seed=17, plant=PLANT, max_seq=256, threads=4)
    m, torch = hf_model(orc, shape)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, shape["vocab"], 40).tolist()
    # oracle: prefill 30 then a scored pass of 10 (KV-cache path)
    orc.forward(toks[:30])
    o = orc.forward(toks[30:])
    with torch.no_grad():
        h = m(torch.tensor([toks])).logits[0, 30:].numpy()
    rel = np.abs(o - h).max() / np.abs(h).max()
    assert rel < 3e-2, rel  # oracle rounds activations to bf16 like the GPU; HF is fp32
    assert (o.argmax(-1) == h.argmax(-1)).mean() >= 0.9
    cc = np.corrcoef(o.ravel(), h.ravel())[0, 1]
    assert cc > 0.999


@pytest.mark.parametrize("shape", [SHAPE, GQA], ids=["mha", "gqa"])
def test_oracle_fp32_mode_matches_transformers(shape):
    """fp32 mode (no bf16 activation / KV rounding) vs transformers fp32 at
    the north star's fp32-accumulate bar (1e-4 of max |logit|): pins the
    forward math itself, not just its bf16 approximation."""
    orc = OracleLlama(shape, weight_seed=17, plant=PLANT, max_seq=256, threads=4, fp32=True)
    m, torch = hf_model(orc, shape)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, shape["vocab"], 40).tolist()
    orc.forward(toks[:30])
    o = orc.forward(toks[30:])
    with torch.no_grad():
        h = m(torch.tensor([toks])).logits[0, 30:].numpy()
    rel = np.abs(o - h).max() / np.abs(h).max()
    assert rel < 1e-4, rel
    assert (o.argmax(-1) == h.argmax(-1)).all()


def test_oracle_scored_pass_equals_sequential():
    """forward_scored contract (model.hpp:61-65): a W-token pass == W one-token passes."""
    orc = OracleLlama(SHAPE, weight_seed=5, max_seq=128, threads=4)
    toks = list(range(3, 20))
    a = orc.forward(toks)
    orc.truncate(0)
    rows = [orc.forward([t])[0] for t in toks]
    assert np.allclose(a, np.stack(rows), rtol=0, atol=1e-5)


def test_plant_makes_bigram_argmax():
    """A planted token t predicts pi(t) in any model sharing the plant."""
    big = dict(SHAPE, d_model=512, ffn_dim=1024, vocab=1024, n_heads=8)
    orc = OracleLlama(big, weight_seed=9, plant=dict(plant_seed=4, alpha=1.0, gain=1.0,
                                                     emb_std=1.0), max_seq=64, threads=4)
    src = orc.plant_src()
    pi = {int(t): v for v, t in enumerate(src) if t >= 0}
    hits = 0
    for t in range(0, 1024, 37):
        orc.truncate(0)
        lg = orc.forward([5, t])[-1]
        hits += int(np.argmax(lg) == pi[t])
    assert hits >= 26  # 28 probes
