// Micro-check (scripts/micro; not product): decode attention on tcgen05.
// S = Q K^T (A = Q [M query rows (16 real)] x 128 dims K-major SW128, B = K
// [64 keys] x 128 dims K-major SW128), then O = P V with B = V [64 keys][128
// dims] in the MN-major SW128 layout a 2-D TMA box {64 dims, 64 keys} writes
// (two 64-dim halves).  Checks the TMEM row layout of M = 64 and M = 128 and
// the MN-major descriptor against a host reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_00784_b200/csrc
//   scripts/micro/attn_tc.cu -o scripts/micro/attn_tc_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "common.cuh"
using namespace dd;

__host__ __device__ constexpr uint32_t idesc_mn(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((addr & 0x3FFFF) >> 4);
    d |= uint64_t(lbo >> 4) << 16;
    d |= uint64_t(sbo >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

// smem: Q [2 halves][M rows][128 B], K [2 halves][64 keys][128 B], V [2 halves][64 keys][128 B],
// P [M rows][128 B] (64 keys), all SW128 (16-byte chunk c of row r at c ^ (r % 8))
__device__ bool wait_bounded(uint64_t* bar, uint32_t ph) {
    const long long t0 = clock64();
    while (clock64() - t0 < 2000000000LL)
        if (mbar_test_wait(bar, ph)) return true;
    return false;
}
__global__ void k(const uint16_t* q, const uint16_t* kk, const uint16_t* vv, float* s_out, float* o_out, int M) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* sQ = sm;                   // 2 * 128 * 128 = 32 KiB
    uint8_t* sK = sQ + 2 * 128 * 128;   // 16 KiB
    uint8_t* sV = sK + 2 * 64 * 128;    // 16 KiB
    uint8_t* sP = sV + 2 * 64 * 128;    // 16 KiB
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc<512>(&slot);
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    auto put = [&](uint8_t* base, int row, int col, uint16_t v) {  // col in elements within 64
        const int chunk = (col >> 3) ^ (row & 7);
        *reinterpret_cast<uint16_t*>(base + row * 128 + chunk * 16 + (col & 7) * 2) = v;
    };
    for (int i = tid; i < 2 * 128 * 64; i += blockDim.x) {  // Q, zero rows >= 16
        const int h = i / (128 * 64), r = (i / 64) % 128, c = i % 64;
        put(sQ + h * 128 * 128, r, c, r < 16 ? q[r * 128 + h * 64 + c] : (r < M ? q[(r % 16) * 128 + ((h * 64 + c + r) % 128)] : 0));
    }
    for (int i = tid; i < 2 * 64 * 64; i += blockDim.x) {
        const int h = i / (64 * 64), r = (i / 64) % 64, c = i % 64;
        put(sK + h * 64 * 128, r, c, kk[r * 128 + h * 64 + c]);
        put(sV + h * 64 * 128, r, c, vv[r * 128 + h * 64 + c]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t tS = tmem, tO = tmem + 64;
    if (tid == 0) {
        const uint32_t id = idesc_mn(M, 64, 0, 0);
        for (int ks = 0; ks < 8; ++ks) {  // K = 128 dims in 16-dim steps
            const int h = ks >> 2, kin = ks & 3;
            const uint64_t a = desc_sw128(smem_u32(sQ + h * 128 * 128), 16, 1024) + 2 * kin;
            const uint64_t b = desc_sw128(smem_u32(sK + h * 64 * 128), 16, 1024) + 2 * kin;
            umma_bf16(tS, a, b, id, ks ? 1u : 0u);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    if (!wait_bounded(&bar, 0)) { if (tid == 0) printf("S MMA timed out\n"); return; }
    tc_fence_after();
    // dump S: every lane of every warp (4 warps x 32 lanes), 64 columns
    {
        float v[16];
        for (int c0 = 0; c0 < 64; c0 += 16) {
            tmem_ld16(tS + (uint32_t(warp * 32) << 16) + c0, v);
            for (int j = 0; j < 16; ++j) s_out[(warp * 32 + lane) * 64 + c0 + j] = v[j];
        }
    }
    // P = bf16(S / 64) for rows 0..15 (lanes of warp 0 hold rows 0..31 for M=128)
    if (warp == 0) {  // tcgen05.ld is warp-collective: every lane loads, lanes < 16 write P
        float v[16];
        for (int c0 = 0; c0 < 64; c0 += 16) {
            tmem_ld16(tS + c0, v);
            for (int j = 0; j < 16; ++j) {
                const float p = v[j] / 64.f;
                uint32_t u;
                memcpy(&u, &p, 4);
                u += 0x7fff + ((u >> 16) & 1);
                if (lane < 16) put(sP, lane, c0 + j, uint16_t(u >> 16));
            }
        }
    }
    for (int i = tid; i < 112 * 64; i += blockDim.x) put(sP, 16 + i / 64, i % 64, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        // O[M x 128] = P[M x 64 keys] V[64 keys x 128 dims]; B = V MN-major:
        // 64-dim halves LBO = 8 KiB apart, 8-key groups SBO = 1 KiB apart
        const uint32_t id = idesc_mn(M, 128, 0, 1);
        for (int ks = 0; ks < 4; ++ks) {  // 16 keys per step
            const uint64_t a = desc_sw128(smem_u32(sP), 16, 1024) + 2 * ks;
            const uint64_t b = desc_sw128(smem_u32(sV + ks * 16 * 128), 64 * 128, 1024);
            umma_bf16(tO, a, b, id, ks ? 1u : 0u);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    if (!wait_bounded(&bar, 1)) { if (tid == 0) printf("PV MMA timed out\n"); return; }
    tc_fence_after();
    {
        float v[16];
        for (int c0 = 0; c0 < 128; c0 += 16) {
            tmem_ld16(tO + (uint32_t(warp * 32) << 16) + c0, v);
            for (int j = 0; j < 16; ++j) o_out[(warp * 32 + lane) * 128 + c0 + j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7fff + ((u >> 16) & 1); return u >> 16; }
static float bf2f(uint16_t b) { uint32_t u = uint32_t(b) << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    std::vector<uint16_t> q(16 * 128), kk(64 * 128), vv(64 * 128);
    srand(3);
    auto rnd = [] { return (rand() / float(RAND_MAX)) * 2 - 1; };
    for (auto& x : q) x = f2bf(rnd());
    for (auto& x : kk) x = f2bf(rnd());
    for (auto& x : vv) x = f2bf(rnd());
    uint16_t *dq, *dk, *dv;
    float *ds, *dO;
    cudaMalloc(&dq, q.size() * 2); cudaMalloc(&dk, kk.size() * 2); cudaMalloc(&dv, vv.size() * 2);
    cudaMalloc(&ds, 128 * 64 * 4); cudaMalloc(&dO, 128 * 128 * 4);
    cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, kk.data(), kk.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, vv.data(), vv.size() * 2, cudaMemcpyHostToDevice);
    printf("start\n");
    const int smem = 32768 + 16384 * 3 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // host reference
    std::vector<float> S(16 * 64), O(16 * 128, 0.f);
    for (int r = 0; r < 16; ++r)
        for (int j = 0; j < 64; ++j) {
            double a = 0;
            for (int d = 0; d < 128; ++d) a += double(bf2f(q[r * 128 + d])) * bf2f(kk[j * 128 + d]);
            S[r * 64 + j] = float(a);
        }
    for (int r = 0; r < 16; ++r)
        for (int d = 0; d < 128; ++d) {
            double a = 0;
            for (int j = 0; j < 64; ++j) a += double(bf2f(f2bf(S[r * 64 + j] / 64.f))) * bf2f(vv[j * 128 + d]);
            O[r * 128 + d] = float(a);
        }
    for (int M : {128, 64}) {
        cudaMemset(ds, 0, 128 * 64 * 4); cudaMemset(dO, 0, 128 * 128 * 4);
        printf("launch M=%d\n", M);
        k<<<1, 128, smem>>>(dq, dk, dv, ds, dO, M);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> s(128 * 64), o(128 * 128);
        cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
        // which TMEM lanes hold query rows 0..15?
        printf("M=%d (%s)\n  lanes matching S rows:", M, cudaGetErrorString(e));
        for (int r = 0; r < 16; ++r) {
            int found = -1;
            for (int l = 0; l < 128 && found < 0; ++l) {
                double err = 0;
                for (int j = 0; j < 64; ++j) err = std::max(err, (double)std::fabs(s[l * 64 + j] - S[r * 64 + j]));
                if (err < 1e-3) found = l;
            }
            printf(" %d", found);
        }
        // all M rows: row r >= 16 uses q[(r%16)][(d + r) % 128]
        printf("\n  all rows -> lane:");
        for (int r = 0; r < M; ++r) {
            int found = -1;
            for (int l = 0; l < 128 && found < 0; ++l) {
                double err = 0;
                for (int j = 0; j < 64; ++j) {
                    double a = 0;
                    for (int d = 0; d < 128; ++d) {
                        const uint16_t qv = r < 16 ? q[r * 128 + d] : q[(r % 16) * 128 + ((d + r) % 128)];
                        a += double(bf2f(qv)) * bf2f(kk[j * 128 + d]);
                    }
                    err = std::max(err, std::fabs(s[l * 64 + j] - a));
                }
                if (err < 1e-3) found = l;
            }
            printf(" %d", found);
        }
        double eo = 0;
        for (int r = 0; r < 16; ++r)
            for (int d = 0; d < 128; ++d) eo = std::max(eo, (double)std::fabs(o[r * 128 + d] - O[r * 128 + d]));
        printf("\n  O rows 0..15 at lanes 0..15: max abs err %.3g (|O| ~ %.3g)\n", eo, std::fabs(O[5]));
    }
    return 0;
}
