// Standalone timing harness for attn_split_kernel (scripts/micro; not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_00784_b200/csrc
//   scripts/micro/attn_bench.cu paper_2503_00784_b200/csrc/attention.cu -o attn_bench -lcuda
#include <cstdio>
#include <vector>
#include <algorithm>
#include "model.h"
namespace dd { void attention_set_trace(unsigned long long* p); }
using namespace dd;
int main(int argc, char** argv) {
    ModelDims m{32, 4096, 32, 32, 128, 11008, 32000, 1e-5f, 1e4f};
    const int max_seq = 4096, ps_sz = 16, n_pages = max_seq / ps_sz;
    size_t kv_elems = (size_t)n_pages * m.n_layers * 2 * m.n_kv_heads * ps_sz * m.head_dim;
    __nv_bfloat16* kv; cudaMalloc(&kv, kv_elems * 2); cudaMemset(kv, 0, kv_elems * 2);
    int32_t* pt; cudaMalloc(&pt, 4 * n_pages);
    std::vector<int32_t> hpt(n_pages); for (int i = 0; i < n_pages; ++i) hpt[i] = i;
    cudaMemcpy(pt, hpt.data(), 4 * n_pages, cudaMemcpyHostToDevice);
    float* q; cudaMalloc(&q, 256 * 4096 * 4); cudaMemset(q, 0, 256 * 4096 * 4);
    __nv_bfloat16* o; cudaMalloc(&o, 256 * 4096 * 2);
    PassState* dps; cudaMalloc(&dps, sizeof(PassState));
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int cases[][2] = {{128, 8}, {2048, 8}, {128, 32}, {2048, 32}, {128, 128}, {1792, 256}};
    for (auto& cs : cases) {
        PassState hps{}; hps.n_cached = cs[0]; hps.w = cs[1];
        cudaMemcpy(dps, &hps, sizeof(hps), cudaMemcpyHostToDevice);
        for (int i = 0; i < 5; ++i) launch_attention(dps, cs[1], m, q, kv, pt, ps_sz, i % 32, o, s);
        cudaEventRecord(a, s);
        const int reps = 64;
        for (int i = 0; i < reps; ++i) launch_attention(dps, cs[1], m, q, kv, pt, ps_sz, i % 32, o, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("n=%d W=%d: %.2f us/launch  (%s)\n", cs[0], cs[1], ms * 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
        unsigned long long* tr; cudaMalloc(&tr, 4096 * 16 * 8); cudaMemset(tr, 0, 4096 * 16 * 8);
        attention_set_trace(tr);
        launch_attention(dps, cs[1], m, q, kv, pt, ps_sz, 3, o, s);
        cudaStreamSynchronize(s);
        attention_set_trace(nullptr);
        std::vector<unsigned long long> h(4096 * 16); cudaMemcpy(h.data(), tr, 4096 * 16 * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, tmax = 0;
        for (int c = 0; c < 4096; ++c) if (h[c * 16]) { t0 = std::min(t0, h[c * 16]); }
        double avg[8] = {0}, mx[8] = {0}; int cnt_[8] = {0};
        for (int c = 0; c < 4096; ++c) for (int k = 0; k < 8; ++k) if (h[c * 16 + k]) { double v = (h[c * 16 + k] - t0) / 1e3; avg[k] += v; mx[k] = std::max(mx[k], v); cnt_[k]++; tmax = std::max(tmax, h[c*16+k]); }
        printf("   stamps avg/max us:");
        for (int k = 0; k < 8; ++k) printf(" %d:%.2f/%.2f(%d)", k, cnt_[k] ? avg[k] / cnt_[k] : -1.0, mx[k], cnt_[k]);
        printf("  span %.2f\n", (tmax - t0) / 1e3);
        cudaFree(tr);

    }
    return 0;
}
