/*
 * tetri.h -- C ABI of libtetri.so, the B200 (sm_100a) device path of the
 * TetriInfer serving data path.
 *
 * The reference (pdsim) has no FFI: its device work is four pure-Python
 * cost-model stand-ins called from the instance actors.  Each entry point
 * below is what replaces one of them:
 *
 *   tk_prefill_chunk   <- costs.chunk_cost          pdsim/costs.py:142-152,
 *                         called at pdsim/prefill.py:353
 *   tk_decode_step     <- costs.decode_iter_latency pdsim/costs.py:104-109,
 *                         called at pdsim/decode.py:255-258
 *   tk_kv_send         <- costs.transfer_latency    pdsim/costs.py:130-139,
 *                         called at pdsim/prefill.py:420-424, control.py:341
 *   tk_predict         <- PredictorModel.predict    pdsim/prefill.py:99-109
 *                         (+ costs.sequential_predictor_cost :155-161)
 *   tk_swap_out/in     <- swap_penalty_us_per_page  pdsim/decode.py:257-258
 *
 * Conventions
 *   - Every function returns int status: 0 ok, <0 error (TK_E*).  The
 *     thread-local message is tk_last_error().
 *   - Plain pointers and sizes only.  Host arrays passed in are borrowed for
 *     the duration of the call (copied to pinned staging before return);
 *     host output arrays are written when the returned event completes
 *     (tk_event_wait, or tk_event_query returning 1).
 *   - Launches are asynchronous on the instance's streams.  Instance
 *     handles are not thread-safe; one host thread drives them.
 *   - "raw" entry points (tk_gemm_bf16, ...) take DEVICE pointers and a
 *     cudaStream_t passed as void*; they exist for kernel-level parity tests
 *     and microbenchmarks.
 */
#ifndef TETRI_H
#define TETRI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_OK 0
#define TK_EINVAL (-1)   /* bad argument / shape                        */
#define TK_ECUDA (-2)    /* CUDA runtime or driver error                */
#define TK_ENOMEM (-3)   /* device / pinned allocation failed           */
#define TK_ECAPACITY (-4)/* KV page id out of the instance's pool       */
#define TK_EUNSUPPORTED (-5)

#define TK_ARCH_OPT 0    /* pre-LN, learned positions (+2), ReLU FFN, biases, tied head */
#define TK_ARCH_LLAMA 1  /* RMSNorm, RoPE, SwiGLU, no biases, untied head               */

typedef struct tk_model_desc {
  int32_t arch;          /* TK_ARCH_*                                            */
  int32_t n_layers;
  int32_t hidden;        /* = n_heads * head_dim                                 */
  int32_t n_heads;
  int32_t head_dim;      /* 64 or 128                                            */
  int32_t ffn;
  int32_t vocab;
  int32_t max_positions; /* learned-position rows (OPT; +2 offset rows added)    */
  int32_t n_labels;      /* >0: sequence-classification head (length predictor) */
  float init_std;        /* weights ~ N(0, init_std^2); norms weight 1 bias 0    */
  float norm_eps;
  float rope_theta;
} tk_model_desc;

/* One contiguous run of prompt tokens of one request inside a chunk
 * (a slice of pdsim Chunk.slices: (request, start, len)).                    */
typedef struct tk_slice {
  int32_t start;         /* position of the first token of the slice           */
  int32_t len;           /* tokens of this slice in the chunk                  */
  int32_t bt_offset;     /* offset of this request's page list in block_tables */
  int32_t n_pages;       /* pages in that list (must cover start+len tokens)   */
  int32_t emit;          /* 1: slice ends the prompt -> produce first token    */
} tk_slice;

typedef struct tk_instance tk_instance;
typedef struct tk_event tk_event;

/* --- errors, versions, devices ------------------------------------------ */
const char* tk_last_error(void);
int tk_version(void);
int tk_device_count(int32_t* n);
/* Free / total HBM of a device (sizes the decode KV capacity from real free
 * memory in B200 mode; replaces the constant pdsim/costs.py:46).            */
int tk_device_memory(int32_t device, int64_t* free_bytes, int64_t* total_bytes);

/* --- instances ------------------------------------------------------------
 * An instance = model weights (shared by every instance of the same model
 * and seed on one device) + a KV page pool of kv_pages pages of page_tokens
 * tokens in page-major layout [page][layer][head][K|V][page_tokens][head_dim]
 * bf16 + streams (compute, copy, predictor) + pinned staging.
 * max_chunk bounds tokens per tk_prefill_chunk / rows per tk_decode_step.   */
int tk_instance_create(int32_t device, const tk_model_desc* model, uint64_t seed,
                       int32_t kv_pages, int32_t page_tokens, int32_t max_chunk,
                       tk_instance** out);
int tk_instance_destroy(tk_instance* inst);
int tk_instance_info(tk_instance* inst, int64_t* weight_bytes, int64_t* page_bytes,
                     int64_t* kv_pool_bytes);
/* Parameter access for parity tests: tensor `name` (e.g. "layers.3.fc1.weight",
 * "embed_tokens.weight"), bf16 data copied to/from a host buffer.            */
int tk_weight_numel(tk_instance* inst, const char* name, int64_t* numel);
int tk_weight_read(tk_instance* inst, const char* name, uint16_t* host_bf16, int64_t numel);
int tk_weight_write(tk_instance* inst, const char* name, const uint16_t* host_bf16,
                    int64_t numel);
/* KV page access (bf16, one page = page_bytes) for parity tests.            */
int tk_kv_read(tk_instance* inst, int32_t page, uint16_t* host_bf16);

/* --- the data path --------------------------------------------------------
 * Chunked-prefill forward of one chunk: n_tokens packed slice tokens (the
 * padded tail of a pdsim Chunk is not executed).  Writes K/V of every token
 * into its request's pages; attention is causal within the request over its
 * accumulated prefix.  For slices with emit=1, first_tokens_out[i] receives
 * the greedy first token (argmax of the LM head on the slice's last token);
 * other entries are -1.  If logits_out is non-NULL it receives fp32 logits
 * [n_emit, vocab] for the emitting slices, in slice order.                  */
int tk_prefill_chunk(tk_instance* inst, int32_t n_tokens, const int32_t* token_ids,
                     const tk_slice* slices, int32_t n_slices, const int32_t* block_tables,
                     int32_t n_block_entries, int32_t* first_tokens_out, float* logits_out,
                     tk_event** ev);
/* One continuous-batching decode iteration over B rows (pdsim running order).
 * Row b: input token last_tokens[b] at position ctx_lens[b] (tokens already in
 * KV); its K/V is appended into page block_tables[b*bt_stride + ctx/pt].
 * next_tokens_out[b] receives the greedy next token.  Without logits_out the
 * step runs as a CUDA graph recorded once per (batch bucket, 1024-token context
 * bucket) of the instance (TK_NO_DECODE_GRAPH=1: eager launches); the result is
 * the same computation.                                                        */
int tk_decode_step(tk_instance* inst, int32_t batch, const int32_t* last_tokens,
                   const int32_t* ctx_lens, const int32_t* block_tables, int32_t bt_stride,
                   int32_t* next_tokens_out, float* logits_out, tk_event** ev);
/* Prefill->decode KV handoff: n_pages whole pages src_pages[i] of src into
 * dst_pages[i] of dst (P2P over NVLink between devices, D2D on one device),
 * on src's copy stream, ordered after all work already issued on src.        */
int tk_kv_send(tk_instance* src, const int32_t* src_pages, tk_instance* dst,
               const int32_t* dst_pages, int32_t n_pages, tk_event** ev);
/* Same handoff with an explicit engine: TK_SEND_AUTO (= tk_kv_send: the SM
 * page-copy kernel when src and dst share a device, the copy engines across
 * devices -- the NVLink transfer then leaves the SMs to the next chunk),
 * TK_SEND_SM (kernel on src's SMs: peer stores over NVLink / device copy),
 * TK_SEND_CE (copy engines: one async copy per run of consecutive pages;
 * leaves the SMs to the next chunk).  Replaces the same stand-in,
 * pdsim/costs.py:130-139 (called from pdsim/prefill.py:420-424).             */
enum { TK_SEND_AUTO = 0, TK_SEND_SM = 1, TK_SEND_CE = 2 };
int tk_kv_send_ex(tk_instance* src, const int32_t* src_pages, tk_instance* dst,
                  const int32_t* dst_pages, int32_t n_pages, int32_t engine, tk_event** ev);
/* Length predictor: sequence classification over n prompts (ids packed,
 * lens[i] each, truncated to max_len), on the predictor stream.  bucket_out[i]
 * = argmax over the instance's n_labels classes.                             */
int tk_predict(tk_instance* inst, const int32_t* token_ids, const int32_t* lens, int32_t n,
               int32_t max_len, int32_t* bucket_out, tk_event** ev);
/* Same classification, also returning the fp32 class scores [n, n_labels]
 * (row-major; the call waits for them).  Parity tests compare these with the
 * oracle's logits instead of the argmax alone.                               */
int tk_predict_scores(tk_instance* inst, const int32_t* token_ids, const int32_t* lens,
                      int32_t n, int32_t max_len, int32_t* bucket_out, float* scores_out,
                      tk_event** ev);
/* Swap whole requests' pages to / from pinned host memory (page_bytes each). */
int tk_swap_out(tk_instance* inst, const int32_t* pages, int32_t n, void* pinned_host,
                tk_event** ev);
int tk_swap_in(tk_instance* inst, const int32_t* pages, int32_t n, const void* pinned_host,
               tk_event** ev);
int tk_host_alloc(int64_t bytes, void** out);
int tk_host_free(void* p);

/* --- events ----------------------------------------------------------------
 * tk_event_query: 1 done (host outputs written), 0 pending.  elapsed_ns is
 * the device time between the event's start and end markers.
 * tk_event_release: the handle is no longer used; if the work has not been
 * observed complete yet, its host outputs are abandoned (never written).     */
int tk_event_query(tk_event* ev, int64_t* elapsed_ns);
int tk_event_wait(tk_event* ev, int64_t* elapsed_ns);
int tk_event_release(tk_event* ev);
int tk_instance_sync(tk_instance* inst);
/* Device time between the start marker of `a` and the end marker of `b`
 * (both done; same device).                                                 */
int tk_event_elapsed(tk_event* a, tk_event* b, int64_t* elapsed_ns);
/* A completed marker on `device`, recorded and synchronized inside the call:
 * the host reads its own clock on return, and tk_event_elapsed(anchor, ev)
 * then maps any later event of that device to host time (completion stamps
 * of TTFT/JCT, pdsim/control.py:334-352, are device times, not poll times). */
int tk_event_anchor(int32_t device, tk_event** anchor);

/* --- instrumentation --------------------------------------------------------
 * Kernels launched by this library since load (all instances).             */
int tk_launch_count(int64_t* n);
/* Bytes the last data-path call on `inst` staged host->device and will copy
 * device->host (metadata + ids in, tokens out).                             */
int tk_last_staged_bytes(tk_instance* inst, int64_t* h2d, int64_t* d2h);
/* Per-kernel-class timing with CUDA events on the launching stream.  Kinds:
 * 0 QKV GEMM, 1 O GEMM, 2 FC1/gate-up GEMM, 3 FC2/down GEMM, 4 attention,
 * 5 head (LM/score GEMM), 6 other (norms, embed, KV write, argmax).
 * tk_profile_read synchronizes, returns the totals since the last read for
 * one kind (algorithmic FLOPs and bytes as defined in DESIGN.md) and resets. */
int tk_profile_enable(tk_instance* inst, int32_t on);
int tk_profile_read(tk_instance* inst, int32_t kind, int64_t* launches, double* total_ms,
                    double* flops, double* bytes);

/* --- raw kernels on device pointers (parity tests / microbenchmarks) -------
 * C[M,N] = A[M,K] . B[N,K]^T (+ bias[N]) (relu) (+ residual) ; A,B bf16 K-major.
 * epilogue: 0 bf16 out; 1 bf16 out + bias; 2 bf16 + bias + relu;
 *           3 fp32 out (residual in/out: C += acc + bias); 4 fp32 out = acc.  */
int tk_gemm_bf16(const void* A, const void* B, void* C, const void* bias, int32_t M,
                 int32_t N, int32_t K, int32_t epilogue, void* workspace,
                 int64_t workspace_bytes, void* stream);
int tk_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int64_t* bytes);
/* LayerNorm over fp32 rows -> bf16: y = (x-mean)/sqrt(var+eps)*w + b.       */
/* Greedy argmax per row of fp32 logits [rows, row_stride], over the first
 * cols columns; ties -> lowest index (torch.argmax).                         */
int tk_argmax(const float* logits, int32_t rows, int32_t cols, int32_t row_stride, int32_t* out,
              void* stream);
int tk_layernorm(const float* x, const void* w, const void* b, void* y, int32_t rows,
                 int32_t cols, float eps, void* stream);
/* Paged decode attention for one layer: q bf16 [B, H, D] -> o bf16 [B, H, D]
 * over ctx_lens[b] tokens of the pages in block_tables (layout as above).    */
int tk_paged_decode_attention(const void* q, void* o, const void* kv_pool, int32_t layer,
                              int32_t n_layers, int32_t n_heads, int32_t head_dim,
                              int32_t page_tokens, const int32_t* block_tables,
                              int32_t bt_stride, const int32_t* ctx_lens, int32_t batch,
                              float scale, void* workspace, int64_t workspace_bytes,
                              void* stream);
/* Chunk (prefill) attention for one layer: q rows of the chunk (bf16, row
 * stride q_stride elements) attend causally to their request's pages.
 * slices/block_tables are HOST arrays (staged synchronously); q/o/kv_pool are
 * device pointers.  o is [n_tokens, n_heads*head_dim].                       */
int tk_chunk_attention(const void* q, int32_t q_stride, void* o, const void* kv_pool,
                       int32_t layer, int32_t n_layers, int32_t n_heads, int32_t head_dim,
                       int32_t page_tokens, const tk_slice* slices, int32_t n_slices,
                       const int32_t* block_tables, int32_t n_tokens, float scale,
                       void* stream);
/* Microbenchmark form of tk_chunk_attention: stages once, launches iters
 * times back to back and reports the mean device time of launches 2..iters
 * (CUDA events on `stream`) in *avg_us.                                      */
int tk_chunk_attention_timed(const void* q, int32_t q_stride, void* o, const void* kv_pool,
                             int32_t layer, int32_t n_layers, int32_t n_heads, int32_t head_dim,
                             int32_t page_tokens, const tk_slice* slices, int32_t n_slices,
                             const int32_t* block_tables, int32_t n_tokens, float scale,
                             void* stream, int32_t iters, float* avg_us);

/* The chunk-attention work plan for a chunk's slices (host only, no device):
 * counts = {pairs, units, ctas, pieces, split groups}; pairs[i*6..] = (slice,
 * row0, pos0, nrows0, nrows1, key blocks); units[i*5..] = (pair, head, kb0,
 * kb1, piece); cta_off[c] = first unit of CTA c (n_ctas + 1 entries).
 * span 256: records are pairs of 128-row tiles, one CTA per unit; span 512:
 * quads of the CTA-pair kernel (nrows0 = the quad's rows, nrows1 = 0), one
 * 2-CTA cluster per unit -- max_ctas / ctas then count clusters.            */
int tk_fa_plan(const tk_slice* slices, int32_t n_slices, int32_t n_heads, int32_t max_ctas,
               int32_t* counts, int32_t* pairs, int32_t pair_cap, int32_t* units,
               int32_t unit_cap, int32_t* cta_off, int32_t cta_cap, int32_t span);
/* Debug: clock64 stamps of the chunk-attention pipeline of CTA 0, recorded
 * only when TK_FA_VARIANT=7 (scripts/attn_trace.py).                       */
int tk_debug_fa_trace(uint64_t* host, int32_t n);
/* GEMM pipeline stamps (TK_GEMM_TRACE=1 runs): 6 kinds x 1024 k-blocks of CTA 0. */
int tk_debug_gemm_trace(uint64_t* host, int32_t n);
/* Per-CTA globaltimer stamps of the last traced GEMM: 5 kinds x 256 CTAs. */
int tk_debug_gemm_cta_trace(uint64_t* host, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* TETRI_H */
