// tk_kernels.h -- internal launchers shared by the runtime (runtime.cu) and
// the raw C-ABI entry points.  All take device pointers and a stream.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tetri.h"

namespace tk {

// Count of kernels launched by the library (tk_launch_count).
void note_launch();

enum Epi : int {
  EPI_BF16 = 0,            // C bf16 = acc
  EPI_BF16_BIAS = 1,       // C bf16 = acc + bias
  EPI_BF16_BIAS_RELU = 2,  // C bf16 = relu(acc + bias)
  EPI_F32_BIAS_RESID = 3,  // C fp32 += acc + bias (residual stream, in place)
  EPI_F32 = 4,             // C fp32 = acc (logits)
  EPI_QKV_PAGED = 5,       // fused QKV (+bias): Q columns -> C bf16, K/V columns -> KV pages
};

// Page-major KV pool geometry: [page][layer][head][K|V][page_tokens][head_dim] bf16.
// K and V of one (page, layer, head) are adjacent 4 KB blocks (head_dim 128),
// so one 5-D TMA box brings both into shared memory.
struct KvGeom {
  int n_layers, n_heads, head_dim, page_tokens;
  __host__ __device__ size_t page_elems() const {
    return static_cast<size_t>(n_layers) * 2 * n_heads * page_tokens * head_dim;
  }
  // element offset of (page, layer, kv, head, slot, 0)
  __host__ __device__ size_t offset(int page, int layer, int kv, int head, int slot) const {
    return (((static_cast<size_t>(page) * n_layers + layer) * n_heads + head) * 2 + kv) *
               static_cast<size_t>(page_tokens) * head_dim +
           static_cast<size_t>(slot) * head_dim;
  }
};

// Per-token row metadata of a chunk, built on the host from tk_slice[]:
// position in its request, and the page / slot its K/V goes to.
struct TokenMeta {
  int32_t pos;
  int32_t page;
  int32_t slot;
  int32_t slice;
};

// EPI_QKV_PAGED target: token rows' K/V go straight from the GEMM epilogue to
// their pages (the separate kv_write pass and its 2x10 MB of traffic per
// OPT-13B chunk layer disappear).  No rotary embedding (OPT).
struct QkvScatter {
  const TokenMeta* meta;
  __nv_bfloat16* pool;
  KvGeom g;
  int layer;
};

int gemm_bf16(const void* A, const void* B, void* C, const void* bias, int M, int N, int K,
              int epi, void* workspace, int64_t ws_bytes, cudaStream_t stream, int max_ctas = 0,
              const QkvScatter* scatter = nullptr);
int64_t gemm_workspace_bytes(int M, int N, int K);
// true when gemm_bf16 takes the swap-AB weight-streaming path for this M
// (that path has no EPI_QKV_PAGED epilogue)
bool gemm_is_skinny(int M);

int launch_embed_opt(const int32_t* ids, const TokenMeta* meta, int n, const __nv_bfloat16* tok_emb,
                     const __nv_bfloat16* pos_emb, float* resid, int hidden, cudaStream_t s);
int launch_embed_llama(const int32_t* ids, int n, const __nv_bfloat16* tok_emb, float* resid,
                       int hidden, cudaStream_t s);
int launch_layernorm(const float* x, const __nv_bfloat16* w, const __nv_bfloat16* b,
                     __nv_bfloat16* y, int rows, int cols, float eps, cudaStream_t s);
int launch_rmsnorm(const float* x, const __nv_bfloat16* w, __nv_bfloat16* y, int rows, int cols,
                   float eps, cudaStream_t s);
// out[i] = x[rows[i]] (+ delta[rows[i]] when given: the residual's pending bf16 update)
int launch_gather_rows_f32(const float* x, const int32_t* rows, int n, int cols, float* out,
                           cudaStream_t s, const __nv_bfloat16* delta = nullptr);
// x += delta (written back), then y = LayerNorm / RMSNorm(x); delta may be null.
int launch_add_norm(float* x, const __nv_bfloat16* delta, const __nv_bfloat16* w,
                    const __nv_bfloat16* b, __nv_bfloat16* y, int rows, int cols, float eps,
                    bool rms, cudaStream_t s);
// qkv [n, 3*H*D] bf16 (q scaled in place by q_scale) -> K,V into pages.
int launch_kv_write(__nv_bfloat16* qkv, const TokenMeta* meta, int n, __nv_bfloat16* pool,
                    KvGeom g, int layer, float q_scale, int rope, float rope_theta,
                    cudaStream_t s);
// Chunk attention work decomposition (host-built, staged to the device).
constexpr int kAttnMaxSplitSlots = 64;   // split partial buffers per launch
constexpr int kAttnMinSplitBlocks = 8;   // >= 512 keys per KV split
struct AttnQBlock {
  int32_t slice;
  int32_t row0;        // chunk row of the first query of this <=128-row block
  int32_t nrows;
  int32_t pos0;        // position of that query in its request
  int32_t n_splits;    // KV splits of this block (1: written directly)
  int32_t first_slot;  // partial slot of split 0 when n_splits > 1
};
struct AttnWork {
  int32_t qblock;
  int32_t kb0, kb1;    // 64-key blocks [kb0, kb1)
  int32_t slot;        // partial slot (-1: unsplit)
};
int build_attn_work(const tk_slice* slices, int n_slices, int n_heads, AttnQBlock* qbs, int qcap,
                    AttnWork* items, int icap, int* n_qblocks, int block_keys);
int launch_attn_combine(__nv_bfloat16* o, const AttnQBlock* qblocks, int n_qblocks, int n_heads,
                        int head_dim, float* partial, cudaStream_t s);
// tcgen05 / TMEM chunk attention (head_dim 128): persistent CTAs over a
// stream-K split of (head, query-tile pair, 128-key block) space.
constexpr int kFaMaxPieces = 2 * 148;  // split pieces per launch (<= 2 per CTA boundary)
struct FaPair {                        // two 128-row query tiles of one slice
  int32_t slice, row0, pos0;           // chunk row / request position of tile 0's first row
  int32_t nrows0, nrows1;              // rows in tile 0 / tile 1 (0: lone tile)
  int32_t nblk;                        // 128-key blocks up to tile 1's (or lone tile's) last row
};
struct FaUnit {
  int32_t pair, head, kb0, kb1;        // key blocks [kb0, kb1) of this (pair, head)
  int32_t piece;                       // partial slot (-1: the whole (pair, head), written directly)
};
struct FaGroup {                       // a (pair, head) computed as several pieces
  int32_t first_piece, n_pieces, pair, head;
};
struct FaPlan {
  int n_pairs, n_units, n_ctas, n_pieces, n_groups;
  int span;  // query rows per record: 256 (pairs, one CTA per unit) / 512 (quads, CTA pairs)
};
// Host-side plan; arrays are caller-provided with capacities.  0 / -1 (overflow).
int build_fa_plan(const tk_slice* slices, int n_slices, int n_heads, int max_ctas, FaPlan* plan,
                  FaPair* pairs, int pcap, FaUnit* units, int ucap, FaGroup* groups, int gcap,
                  int32_t* cta_off, int ocap, int span = 256);
// Record span the attention launch for this head_dim uses (512: CTA-pair kernel).
int fa_span(int head_dim);
int64_t fa_partial_bytes();
int gemm_debug_trace(unsigned long long* host, int n);
int gemm_debug_cta_trace(unsigned long long* host, int n);
int fa_debug_trace(unsigned long long* host, int n);  // TK_FA_VARIANT=7 timing stamps
int launch_chunk_attention_fa(const __nv_bfloat16* qkv, int q_rows, int q_stride,
                              __nv_bfloat16* o, const __nv_bfloat16* pool, int pool_pages,
                              KvGeom g, int layer, const FaPlan& plan, const FaPair* pairs_dev,
                              const FaUnit* units_dev, const FaGroup* groups_dev,
                              const int32_t* cta_off_dev, const tk_slice* slices_dev,
                              const int32_t* bt_dev, float scale, float* partial,
                              cudaStream_t s);
// true: use the tcgen05 attention for this head_dim (TK_ATTN_MMA_SYNC=1 forces mma.sync)
bool use_tc_attention(int head_dim);
int64_t attn_partial_bytes(int n_heads, int head_dim);
int launch_chunk_attention_work(const __nv_bfloat16* q, int q_stride, __nv_bfloat16* o,
                                const __nv_bfloat16* pool, KvGeom g, int layer,
                                const AttnWork* work, int n_work, const AttnQBlock* qblocks,
                                int n_qblocks, bool any_split, const tk_slice* slices_dev,
                                const int32_t* bt_dev, float scale, float* partial,
                                cudaStream_t s);
int64_t decode_attention_workspace_bytes(int batch, int n_heads, int head_dim, int max_ctx);
int launch_decode_attention(const __nv_bfloat16* q, int q_stride, __nv_bfloat16* o,
                            const __nv_bfloat16* pool,
                            KvGeom g, int layer, const int32_t* block_tables, int bt_stride,
                            const int32_t* ctx_lens, int batch, int max_ctx, float scale,
                            void* workspace, int64_t ws_bytes, cudaStream_t s);
int launch_argmax_strided(const float* logits, int rows, int cols, int stride, int32_t* out,
                          cudaStream_t s);
int launch_init_normal(__nv_bfloat16* w, int64_t n, uint64_t seed, float std, cudaStream_t s);
int launch_fill(__nv_bfloat16* w, int64_t n, float value, cudaStream_t s);
int launch_swiglu(const __nv_bfloat16* gate_up, __nv_bfloat16* out, int n, int ffn,
                  cudaStream_t s);

// KV page copy (handoff): pages src_pages[i] of src_pool -> dst_pages[i] of dst_pool,
// one launch per kCopyMaxPages pages; dst_pool may live on a peer device.
constexpr int kCopyThreads = 512;
constexpr int kCopyCtasPerSm = 4;
constexpr int kCopyMaxPages = 1024;
struct PageCopyList {
  int32_t n, parts;
  int64_t page_vec;  // page bytes / 16
  int32_t src[kCopyMaxPages];
  int32_t dst[kCopyMaxPages];
};
int launch_kv_copy_pages(const void* src_pool, void* dst_pool, int64_t page_bytes,
                         const int32_t* src_pages, const int32_t* dst_pages, int n, int n_sms,
                         cudaStream_t s);

}  // namespace tk
