// Host interface of the skinny tcgen05 GEMM (see gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dd {

struct GemmArgs {
    int n_out;         // weight rows (output features), multiple of 128
    int k;             // reduction length, multiple of 64
    int w;             // valid tokens (columns stored)
    int nt;            // padded token count: multiple of 16, <= 256
    int kb_per_split;  // 64-wide k-blocks per split
    int splits;
    int stages;        // smem ring depth
    float* ws;         // [splits][w][n_out] fp32 partial sums
};

struct GemmPlan {
    int tiles;
    int splits;
    int kb_per_split;
    int stages;
    int smem_bytes;
};

// Row-major [rows, cols] bf16 tensor map with 64-column boxes, 128B swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_rows);

GemmPlan plan_gemm(int n_out, int k, int nt);

cudaError_t launch_gemm(const CUtensorMap* map_w, const CUtensorMap* map_x, int n_out, int k,
                        int w, int nt, const GemmPlan& plan, float* ws, cudaStream_t stream);

}  // namespace dd
