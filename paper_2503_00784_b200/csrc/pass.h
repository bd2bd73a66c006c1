// Persistent whole-pass kernel (pass.cu): one launch runs the embedding, every
// layer's QKV / attention / O / gate-up / down and the LM head of a scored
// pass, with tile-level dataflow flags instead of kernel boundaries.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "model.h"
#include "tp.h"

namespace dd {

enum PassPhaseType { kPhEmbed = 0, kPhGemm = 1, kPhAttn = 2 };
// where a GEMM phase's activation k-block comes from
enum PassXSrc {
    kXNormed = 0,  // h (embedding / residual producer): flag of tile kb / 2
    kXAttn = 1,    // o (attention): flags of head kb * 64 / head_dim, every query tile
    kXSwiglu = 2,  // a (SwiGLU): flag of gate/up tile kb
};

struct PassPhase {
    int type;
    int x_map;     // 0 = h, 1 = o, 2 = a
    int x_src;
    int x_flag;    // flag base of the producing phase
    int out_flag;  // flag base of this phase's outputs
    int layer;
    int qkv_flag;  // attention: flag base of the layer's QKV tiles
    // GEMM sub-phases: the (tile, k-block) grid is cut into kg k-groups x tg
    // tile groups, run in the order (k-group 0: tile groups 0..tg-1), (k-group
    // 1: ...), each a stream-K over every CTA.  A tile group is complete after
    // its last k-group, so outputs are published progressively (tile group 0
    // first) and a consumer's k-group i needs only its producer's tile group i.
    int kg;
    int tg;
    const __nv_bfloat16* w;  // pre-tiled weights (GEMM)
    const int* begins;       // [149] stream-K range starts by rank (weighted), or nullptr
    GemmArgs a;              // GEMM shape + fused epilogue
};

struct PassParams {
    const PassPhase* phases;
    int n_phases;
    int stages;
    int nt;
    int tmem_buf;
    int prefetch;  // L2 prefetch distance (k-blocks) beyond the shared-memory ring
    int attn_cpg;     // attention: kAttnChunk-key chunks per group of a split item
    int attn_single;  // attention: items of at most this many chunks are not split
    int nodep;     // timing experiments only (wrong numerics): skip waits, bit 1 activation producer, 2 epilogue inputs, 4 attention inputs, 8 stream-K reducer
    const int* rank_of_smid;  // [1024] partition rank of each SM, or nullptr (rank = blockIdx)
    const int* attn_rank;     // [nctas] position of each partition rank in the attention item order, or nullptr
    TpPeers tp;               // tensor parallelism (tp.size > 1): O / down tile exchange (W <= 16)
    unsigned long long* trace;  // debug: [CTA][phase][12] globaltimer stamps, or nullptr

    const PassState* ps;
    int* flags;
    // embedding
    const __nv_bfloat16* emb;
    const float* gain;
    float* x;
    __nv_bfloat16* h;
    float* ss;
    // attention
    ModelDims m;
    const float* q;
    const __nv_bfloat16* kv_pool;
    const int32_t* page_table;
    int page_size;
    float scale_log2;
    __nv_bfloat16* o;
    float* attn_part;
    int* attn_cnt;
};

constexpr int kPassThreads = 256;
constexpr int kAttnChunk = 32;    // keys staged per attention step
#ifndef DD_ATTN_BUFS_128
#define DD_ATTN_BUFS_128 3
#endif
// K/V chunk buffers of a decode attention item (all staged ahead, each refilled
// after use).  head_dim 128 keeps 3 (16 KiB each): the smem they free buys the
// weight ring a ninth stage (W=9: 3.006 -> 2.983 ms, 2K context -0.02 ms).
__host__ __device__ constexpr int attn_bufs(int hd) { return hd == 128 ? DD_ATTN_BUFS_128 : 4; }
static_assert(DD_ATTN_BUFS_128 >= 2 && DD_ATTN_BUFS_128 <= 4, "attn_item's cp.async wait ladder handles 2..4 buffers");
constexpr int kAttnGroups = 4;    // chunk groups per (head, query tile)
constexpr int kCounterStride = 32;  // ints: one 128-byte line per stream-K tile counter
constexpr int kFlagStride = 32;   // ints: one 128-byte line per flag replica
constexpr int kFlagReplicas = 8;  // every flag is published to 8 lines; CTA c polls replica c % 8
                                  // (148 pollers on one line serialise in its L2 slice)

void* pass_debug_enable(int on);  // mapped host int[148][8] progress words
size_t pass_attn_part_floats(const ModelDims& m);
size_t pass_attn_cnt_ints(const ModelDims& m);
int pass_smem_bytes(const ModelDims& m, int nt, int* stages);

cudaError_t launch_pass_kernel(const CUtensorMap& map_h, const CUtensorMap& map_o,
                               const CUtensorMap& map_a, const PassParams& p, int smem_bytes,
                               int nctas, cudaStream_t s);

}  // namespace dd
