// Drives integration/gpu_target.hpp with the reference's own types: on a
// machine without an sm_100 GPU the constructor must throw the reference's
// ConfigError (no CPU fallback); with one, a prompt, a scored pass, a greedy
// duo verification and a rollback run through the adapter.
#include <cstdio>

#include "gpu_target.hpp"

int main() {
    dd_model_desc d{};
    d.n_layers = 2; d.d_model = 512; d.n_heads = 8; d.n_kv_heads = 8; d.head_dim = 64;
    d.ffn_dim = 1408; d.vocab = 1024; d.rms_eps = 1e-5f; d.rope_theta = 1e4f;
    d.max_seq = 256; d.page_size = 16; d.precision = DD_PREC_BF16;
    try {
        duodec_b200::GpuTarget tgt(d, 5);
        duodec::GenerationState s{};
        s.verified = {1, 2, 3, 4, 5, 6, 7, 8};
        tgt.prefill(s.verified);
        duodec::DraftSequence tail;
        tail.tokens = {9, 10};
        std::vector<double> u(1024, 1.0 / 1024);
        tail.dists = {duodec::Distribution::from_probs(u), duodec::Distribution::from_probs(u)};
        s.unverified = tail;
        tgt.upload_tail_q(tail);
        tgt.target_step(s);
        duodec::DraftBundle b;
        duodec::DraftSequence b0;
        b0.tokens = {11};
        b.sequences = {b0};
        duodec::RandomStream rng(2);
        const dd_verify_out o = tgt.verify_duo(s, b, rng, 1.0, true);
        s.verified.push_back(9);
        tgt.rollback(s);
        std::printf("GPU ok: prefix_all_accepted=%d draws=%d counter=%llu\n", o.prefix_all_accepted,
                    o.n_draws, static_cast<unsigned long long>(rng.counter()));
    } catch (const duodec::ConfigError& e) {
        std::printf("ConfigError: %s\n", e.what());
    }
    return 0;
}
