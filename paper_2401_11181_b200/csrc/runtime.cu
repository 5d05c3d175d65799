// runtime.cu -- native runtime behind include/tetri.h.
//
// Owns, per device: model weights (one bf16 blob per (device, model, seed),
// shared by every instance that asks for it, e.g. a co-located prefill and
// decode instance), per instance: a page-major KV pool, three streams
// (compute / copy / predictor), device scratch sized for max_chunk rows, an
// fp32 residual stream, GEMM + attention workspaces and a ring of pinned +
// device staging slots through which each call's host metadata travels in a
// single H2D copy.  Every data-path call is asynchronous and returns a
// tk_event whose completion also publishes the call's small host outputs.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "tk_common.cuh"
#include "tk_kernels.h"

namespace tk {

static thread_local std::string g_err;

bool use_tc_attention(int head_dim) {
  static const bool forced_off = getenv("TK_ATTN_MMA_SYNC") != nullptr;
  return (head_dim == 128 || head_dim == 64) && !forced_off;
}
static std::atomic<int64_t> g_launches{0};

bool pdl_enabled() {
  static const bool on = getenv("TK_NO_PDL") == nullptr;
  return on;
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
          std::to_string(line) + ")";
  return e == cudaErrorMemoryAllocation ? TK_ENOMEM : TK_ECUDA;
}

// ------------------------------------------------------------------ weights
struct Tensor {
  __nv_bfloat16* ptr = nullptr;
  int64_t numel = 0;
};

struct LayerW {
  __nv_bfloat16 *ln1_w, *ln1_b, *qkv_w, *qkv_b, *o_w, *o_b, *ln2_w, *ln2_b, *fc1_w, *fc1_b, *fc2_w,
      *fc2_b;
};

struct Weights {
  int device = 0;
  tk_model_desc md{};
  uint64_t seed = 0;
  int refs = 0;
  void* blob = nullptr;
  int64_t bytes = 0;
  std::map<std::string, Tensor> named;
  std::vector<LayerW> layers;
  __nv_bfloat16 *embed = nullptr, *pos = nullptr, *fln_w = nullptr, *fln_b = nullptr,
                *head = nullptr;  // LM head [vocab, h] or score [labels_pad, h]
  int head_rows = 0;              // GEMM N of the head (vocab, or labels padded to 8)
};

static std::mutex g_mu;
static std::map<std::string, Weights*> g_weights;

static std::string weight_key(int device, const tk_model_desc& md, uint64_t seed) {
  std::string k(reinterpret_cast<const char*>(&md), sizeof(md));
  return std::to_string(device) + ":" + std::to_string(seed) + ":" + k;
}

struct Spec {
  std::string name;
  int64_t numel;
  int kind;  // 0 normal(std), 1 ones, 2 zeros
};

static std::vector<Spec> weight_specs(const tk_model_desc& m) {
  std::vector<Spec> s;
  const int64_t h = m.hidden, f = m.ffn;
  const bool opt = m.arch == TK_ARCH_OPT;
  s.push_back({"embed_tokens.weight", static_cast<int64_t>(m.vocab) * h, 0});
  if (opt) s.push_back({"embed_positions.weight", (m.max_positions + 2) * h, 0});
  for (int l = 0; l < m.n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    if (opt) {
      s.push_back({p + "self_attn_layer_norm.weight", h, 1});
      s.push_back({p + "self_attn_layer_norm.bias", h, 2});
      s.push_back({p + "self_attn.qkv_proj.weight", 3 * h * h, 0});
      s.push_back({p + "self_attn.qkv_proj.bias", 3 * h, 2});
      s.push_back({p + "self_attn.out_proj.weight", h * h, 0});
      s.push_back({p + "self_attn.out_proj.bias", h, 2});
      s.push_back({p + "final_layer_norm.weight", h, 1});
      s.push_back({p + "final_layer_norm.bias", h, 2});
      s.push_back({p + "fc1.weight", f * h, 0});
      s.push_back({p + "fc1.bias", f, 2});
      s.push_back({p + "fc2.weight", h * f, 0});
      s.push_back({p + "fc2.bias", h, 2});
    } else {
      s.push_back({p + "input_layernorm.weight", h, 1});
      s.push_back({p + "self_attn.qkv_proj.weight", 3 * h * h, 0});
      s.push_back({p + "self_attn.o_proj.weight", h * h, 0});
      s.push_back({p + "post_attention_layernorm.weight", h, 1});
      s.push_back({p + "mlp.gate_up_proj.weight", 2 * f * h, 0});
      s.push_back({p + "mlp.down_proj.weight", h * f, 0});
    }
  }
  if (opt) {
    s.push_back({"final_layer_norm.weight", h, 1});
    s.push_back({"final_layer_norm.bias", h, 2});
  } else {
    s.push_back({"norm.weight", h, 1});
  }
  if (m.n_labels > 0) {
    const int64_t rows = (m.n_labels + 7) / 8 * 8;
    s.push_back({"score.weight", rows * h, 0});
  } else if (!opt) {
    s.push_back({"lm_head.weight", static_cast<int64_t>(m.vocab) * h, 0});
  }
  return s;
}

static int validate_desc(const tk_model_desc& m) {
  TK_CHECK(m.arch == TK_ARCH_OPT || m.arch == TK_ARCH_LLAMA, TK_EINVAL, "model: unknown arch");
  TK_CHECK(m.n_layers > 0 && m.hidden > 0 && m.n_heads > 0 && m.ffn > 0 && m.vocab > 0,
           TK_EINVAL, "model: sizes must be positive");
  TK_CHECK(m.n_heads * m.head_dim == m.hidden, TK_EINVAL, "model: hidden != n_heads*head_dim");
  TK_CHECK(m.head_dim == 128 || m.head_dim == 64, TK_EUNSUPPORTED, "model: head_dim 64 or 128");
  TK_CHECK(m.hidden % 64 == 0 && m.ffn % 64 == 0, TK_EINVAL,
           "model: hidden and ffn must be multiples of 64");
  TK_CHECK(m.vocab % 8 == 0, TK_EINVAL, "model: vocab must be a multiple of 8");
  TK_CHECK(m.arch != TK_ARCH_OPT || m.max_positions > 0, TK_EINVAL, "model: max_positions");
  return TK_OK;
}

static int acquire_weights(int device, const tk_model_desc& md, uint64_t seed, Weights** out) {
  std::lock_guard<std::mutex> lock(g_mu);
  const std::string key = weight_key(device, md, seed);
  auto it = g_weights.find(key);
  if (it != g_weights.end()) {
    it->second->refs++;
    *out = it->second;
    return TK_OK;
  }
  auto specs = weight_specs(md);
  int64_t total = 0;
  for (auto& s : specs) total += (s.numel * 2 + 255) / 256 * 256;
  std::unique_ptr<Weights> w(new Weights());
  w->device = device;
  w->md = md;
  w->seed = seed;
  w->bytes = total;
  TK_CUDA(cudaMalloc(&w->blob, total));
  int64_t off = 0;
  uint64_t tix = 0;
  for (auto& s : specs) {
    Tensor t;
    t.ptr = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(w->blob) + off);
    t.numel = s.numel;
    off += (s.numel * 2 + 255) / 256 * 256;
    w->named[s.name] = t;
    const uint64_t tseed = seed * 0x9E3779B97F4A7C15ull + (++tix) * 0xC2B2AE3D27D4EB4Full;
    int rc = s.kind == 0   ? launch_init_normal(t.ptr, t.numel, tseed, md.init_std, 0)
             : s.kind == 1 ? launch_fill(t.ptr, t.numel, 1.f, 0)
                           : launch_fill(t.ptr, t.numel, 0.f, 0);
    if (rc) {
      cudaFree(w->blob);
      return rc;
    }
  }
  TK_CUDA(cudaDeviceSynchronize());
  auto P = [&](const std::string& n) { return w->named[n].ptr; };
  const bool opt = md.arch == TK_ARCH_OPT;
  w->embed = P("embed_tokens.weight");
  if (opt) w->pos = P("embed_positions.weight");
  for (int l = 0; l < md.n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    LayerW L{};
    if (opt) {
      L.ln1_w = P(p + "self_attn_layer_norm.weight");
      L.ln1_b = P(p + "self_attn_layer_norm.bias");
      L.qkv_w = P(p + "self_attn.qkv_proj.weight");
      L.qkv_b = P(p + "self_attn.qkv_proj.bias");
      L.o_w = P(p + "self_attn.out_proj.weight");
      L.o_b = P(p + "self_attn.out_proj.bias");
      L.ln2_w = P(p + "final_layer_norm.weight");
      L.ln2_b = P(p + "final_layer_norm.bias");
      L.fc1_w = P(p + "fc1.weight");
      L.fc1_b = P(p + "fc1.bias");
      L.fc2_w = P(p + "fc2.weight");
      L.fc2_b = P(p + "fc2.bias");
    } else {
      L.ln1_w = P(p + "input_layernorm.weight");
      L.qkv_w = P(p + "self_attn.qkv_proj.weight");
      L.o_w = P(p + "self_attn.o_proj.weight");
      L.ln2_w = P(p + "post_attention_layernorm.weight");
      L.fc1_w = P(p + "mlp.gate_up_proj.weight");
      L.fc2_w = P(p + "mlp.down_proj.weight");
    }
    w->layers.push_back(L);
  }
  if (opt) {
    w->fln_w = P("final_layer_norm.weight");
    w->fln_b = P("final_layer_norm.bias");
  } else {
    w->fln_w = P("norm.weight");
  }
  if (md.n_labels > 0) {
    w->head = P("score.weight");
    w->head_rows = (md.n_labels + 7) / 8 * 8;
  } else {
    w->head = opt ? w->embed : P("lm_head.weight");  // OPT ties lm_head to embed_tokens
    w->head_rows = md.vocab;
  }
  w->refs = 1;
  *out = w.get();
  g_weights[key] = w.release();
  return TK_OK;
}

static void release_weights(Weights* w) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (--w->refs > 0) return;
  for (auto it = g_weights.begin(); it != g_weights.end(); ++it) {
    if (it->second == w) {
      g_weights.erase(it);
      break;
    }
  }
  cudaSetDevice(w->device);
  cudaFree(w->blob);
  delete w;
}

// ------------------------------------------------------------------ staging ring
constexpr int kRingSlots = 8;
constexpr int64_t kSlotBytes = 4 << 20;

struct Slot {
  uint8_t* host = nullptr;  // pinned
  uint8_t* dev = nullptr;
  cudaEvent_t done = nullptr;  // last use finished on device
  tk_event* owner = nullptr;   // event whose outputs live in this slot
};

}  // namespace tk

struct tk_event {
  int device = 0;
  cudaEvent_t start = nullptr, end = nullptr;
  bool finished = false;
  // host output publication on completion: dst[i] = src[i] (i < n_out), or
  // with remap: dst[i] = remap[i] >= 0 ? src[remap[i]] : -1.
  const int32_t* out_src = nullptr;
  int32_t* out_dst = nullptr;
  const int32_t* remap = nullptr;
  int n_out = 0;
  tk::Slot* slot = nullptr;
  bool released = false;
};

struct tk_instance {
  int device = 0;
  tk::Weights* w = nullptr;
  tk::KvGeom geom{};
  int kv_pages = 0;
  __nv_bfloat16* pool = nullptr;
  int64_t page_bytes = 0;
  int max_chunk = 0;
  cudaStream_t s_compute = nullptr, s_copy = nullptr, s_pred = nullptr;
  // scratch
  float* resid = nullptr;
  __nv_bfloat16* delta = nullptr;  // pending bf16 residual update (O-proj / FC2 output)
  __nv_bfloat16 *xn = nullptr, *qkv = nullptr, *attn = nullptr, *ffn = nullptr;
  float* logits = nullptr;
  int max_emit = 0;
  void* gemm_ws = nullptr;
  int64_t gemm_ws_bytes = 0;
  void* dec_ws = nullptr;
  int64_t dec_ws_bytes = 0;
  float* attn_partial = nullptr;
  int dec_max_ctx = 0;
  tk::Slot ring[tk::kRingSlots];
  int ring_next = 0;
  int64_t last_h2d = 0, last_d2h = 0;
  // profiling (tk_profile_*)
  bool prof = false;
  struct ProfRec {
    int kind;
    double flops, bytes;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  // Decode steps as CUDA graphs (tk_decode_step): one graph per (padded batch, context
  // bucket); every per-step input lives at fixed device addresses (dec_fixed), padding
  // rows attend to a scratch page past the pool (page kv_pages).
  struct DecGraph {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // kernels in the graph (tk_launch_count)
    int seen = 0;
    bool failed = false;
  };
  std::map<uint64_t, DecGraph> dec_graphs;
  uint8_t* dec_fixed = nullptr;
  int64_t dec_fixed_bytes = 0;
};

namespace tk {

static int finalize_event(tk_event* ev) {
  if (ev->finished) return TK_OK;
  TK_CUDA(cudaEventSynchronize(ev->end));
  // a released event abandons its host outputs (the caller's buffer may be gone)
  if (ev->out_dst && !ev->released) {
    for (int i = 0; i < ev->n_out; ++i)
      ev->out_dst[i] = ev->remap ? (ev->remap[i] >= 0 ? ev->out_src[ev->remap[i]] : -1)
                                 : ev->out_src[i];
  }
  ev->finished = true;
  if (ev->slot && ev->slot->owner == ev) ev->slot->owner = nullptr;
  return TK_OK;
}

static void maybe_free_event(tk_event* ev) {
  if (ev->released && ev->finished) {
    cudaEventDestroy(ev->start);
    cudaEventDestroy(ev->end);
    delete ev;
  }
}

// Take the next ring slot, finishing whatever call last used it.
static int take_slot(tk_instance* inst, Slot** out) {
  Slot* s = &inst->ring[inst->ring_next];
  inst->ring_next = (inst->ring_next + 1) % kRingSlots;
  if (s->owner) {
    tk_event* prev = s->owner;
    int rc = finalize_event(prev);
    if (rc) return rc;
    maybe_free_event(prev);
  }
  TK_CUDA(cudaEventSynchronize(s->done));
  *out = s;
  return TK_OK;
}

// Released events whose device work had not finished yet (handoff / swap
// events own no staging slot).  Releasing must not block the host -- a
// streamed handoff drops each part's handle while the copy still runs behind
// the next chunk -- so they are parked here and freed once complete.
static std::mutex g_zombie_mu;
static std::vector<tk_event*> g_zombies;

static void sweep_zombies() {
  std::lock_guard<std::mutex> lock(g_zombie_mu);
  size_t keep = 0;
  for (tk_event* ev : g_zombies) {
    if (cudaEventQuery(ev->end) == cudaSuccess) {
      ev->finished = true;
      maybe_free_event(ev);
    } else {
      g_zombies[keep++] = ev;
    }
  }
  cudaGetLastError();  // a not-ready query is not an error
  g_zombies.resize(keep);
}

static int new_event(tk_instance* inst, cudaStream_t s, tk_event** out) {
  if (!g_zombies.empty()) sweep_zombies();
  tk_event* ev = new tk_event();
  ev->device = inst->device;
  TK_CUDA(cudaEventCreate(&ev->start));
  TK_CUDA(cudaEventCreate(&ev->end));
  TK_CUDA(cudaEventRecord(ev->start, s));
  *out = ev;
  return TK_OK;
}

// Bump allocator inside a slot (host and device views at equal offsets).
struct Packer {
  Slot* slot;
  int64_t off = 0;
  template <typename T>
  T* put(const T* src, int64_t n, T** dev) {
    off = (off + 15) / 16 * 16;
    T* h = reinterpret_cast<T*>(slot->host + off);
    if (src && n) memcpy(h, src, n * sizeof(T));
    *dev = reinterpret_cast<T*>(slot->dev + off);
    off += n * sizeof(T);
    return h;
  }
  bool ok() const { return off <= kSlotBytes; }
};

static float attn_scale(const tk_model_desc& m) { return 1.f / sqrtf(static_cast<float>(m.head_dim)); }

enum ProfKind { PK_QKV = 0, PK_O = 1, PK_FC1 = 2, PK_FC2 = 3, PK_ATTN = 4, PK_HEAD = 5, PK_OTHER = 6 };

static cudaEvent_t pool_event(tk_instance* inst) {
  if (!inst->ev_pool.empty()) {
    cudaEvent_t e = inst->ev_pool.back();
    inst->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Run `op` bracketed by CUDA events on `s` when profiling is on.
template <typename Op>
static int profiled(tk_instance* inst, cudaStream_t s, int kind, double flops, double bytes,
                    Op&& op) {
  if (!inst->prof) return op();
  cudaEvent_t a = pool_event(inst), b = pool_event(inst);
  TK_CUDA(cudaEventRecord(a, s));
  int rc = op();
  TK_CUDA(cudaEventRecord(b, s));
  inst->recs.push_back({kind, flops, bytes, a, b});
  return rc;
}

// One transformer layer over `n` rows whose metadata lives on the device.
// attention_fn performs the attention step writing inst->attn; attn_flops /
// attn_bytes are its algorithmic work.
template <typename AttnFn>
static int run_layer(tk_instance* inst, int layer, int n, const TokenMeta* meta_dev,
                     cudaStream_t s, double attn_flops, double attn_bytes, AttnFn&& attention_fn) {
  const tk_model_desc& m = inst->w->md;
  const LayerW& L = inst->w->layers[layer];
  const double h = m.hidden, f = m.ffn, nn = n;
  const bool opt = m.arch == TK_ARCH_OPT;
  const int hi = m.hidden;
  int rc;
  // The residual stream is fp32; O-proj and FC2 store their bf16 output
  // (bias included) in inst->delta and the next norm adds it in.
  const __nv_bfloat16* pending = layer > 0 ? inst->delta : nullptr;
  rc = profiled(inst, s, PK_OTHER, 0, nn * h * (pending ? 12 : 6), [&] {
    return launch_add_norm(inst->resid, pending, L.ln1_w, opt ? L.ln1_b : nullptr, inst->xn, n,
                           hi, m.norm_eps, !opt, s);
  });
  if (rc) return rc;
  // OPT (no rotary embedding) above the skinny range: the QKV epilogue writes K/V
  // straight into the pages; otherwise a kv_write pass (RoPE for Llama).  The
  // decode-size (skinny) GEMM can scatter K/V too (TK_FUSED_DECODE_KV=1), but its
  // per-row 2-byte page stores made the QKV GEMM slower than the kv_write launch it
  // saves (B=32: equal, B=128: -2%; profiles/r02_experiments.md).
  static const bool fused_decode_kv = getenv("TK_FUSED_DECODE_KV") != nullptr;
  static const bool no_fused_kv = getenv("TK_NO_FUSED_KV") != nullptr;  // experiments
  const bool fused_kv = opt && !no_fused_kv && (fused_decode_kv || !gemm_is_skinny(n));
  const QkvScatter scatter{meta_dev, inst->pool, inst->geom, layer};
  rc = profiled(inst, s, PK_QKV, 2 * nn * 3 * h * h, (3 * h * h + nn * 4 * h) * 2, [&] {
    return gemm_bf16(inst->xn, L.qkv_w, inst->qkv, L.qkv_b, n, 3 * hi, hi,
                     fused_kv ? EPI_QKV_PAGED : (opt ? EPI_BF16_BIAS : EPI_BF16), inst->gemm_ws,
                     inst->gemm_ws_bytes, s, 0, fused_kv ? &scatter : nullptr);
  });
  if (rc) return rc;
  if (!fused_kv) {
    rc = profiled(inst, s, PK_OTHER, 0, nn * h * 8, [&] {
      return launch_kv_write(inst->qkv, meta_dev, n, inst->pool, inst->geom, layer, 1.f,
                             opt ? 0 : 1, m.rope_theta, s);
    });
    if (rc) return rc;
  }
  rc = profiled(inst, s, PK_ATTN, attn_flops, attn_bytes, attention_fn);
  if (rc) return rc;
  rc = profiled(inst, s, PK_O, 2 * nn * h * h, (h * h + nn * h) * 2 + nn * h * 2, [&] {
    return gemm_bf16(inst->attn, L.o_w, inst->delta, L.o_b, n, hi, hi, EPI_BF16_BIAS,
                     inst->gemm_ws, inst->gemm_ws_bytes, s);
  });
  if (rc) return rc;
  rc = profiled(inst, s, PK_OTHER, 0, nn * h * 12, [&] {
    return launch_add_norm(inst->resid, inst->delta, L.ln2_w, opt ? L.ln2_b : nullptr, inst->xn,
                           n, hi, m.norm_eps, !opt, s);
  });
  if (rc) return rc;
  const double up = opt ? f : 2 * f;
  rc = profiled(inst, s, PK_FC1, 2 * nn * up * h, (up * h + nn * h + nn * up) * 2, [&] {
    return opt ? gemm_bf16(inst->xn, L.fc1_w, inst->ffn, L.fc1_b, n, m.ffn, hi, EPI_BF16_BIAS_RELU,
                           inst->gemm_ws, inst->gemm_ws_bytes, s)
               : gemm_bf16(inst->xn, L.fc1_w, inst->ffn, nullptr, n, 2 * m.ffn, hi, EPI_BF16,
                           inst->gemm_ws, inst->gemm_ws_bytes, s);
  });
  if (rc) return rc;
  if (!opt) {
    rc = profiled(inst, s, PK_OTHER, 0, nn * f * 6, [&] {
      return launch_swiglu(inst->ffn, inst->ffn + static_cast<size_t>(n) * 2 * m.ffn, n, m.ffn, s);
    });
    if (rc) return rc;
  }
  const __nv_bfloat16* ffn_act =
      opt ? inst->ffn : inst->ffn + static_cast<size_t>(n) * 2 * m.ffn;
  rc = profiled(inst, s, PK_FC2, 2 * nn * h * f, (h * f + nn * f) * 2 + nn * h * 2, [&] {
    return gemm_bf16(ffn_act, L.fc2_w, inst->delta, L.fc2_b, n, hi, m.ffn, EPI_BF16_BIAS,
                     inst->gemm_ws, inst->gemm_ws_bytes, s);
  });
  return rc;
}

// Final norm + head over `n_rows` gathered residual rows -> logits / argmax.
static int run_head(tk_instance* inst, int n_rows, const int32_t* rows_dev, int32_t* tokens_dev,
                    cudaStream_t s) {
  const tk_model_desc& m = inst->w->md;
  Weights* w = inst->w;
  int rc;
  float* gathered = reinterpret_cast<float*>(inst->qkv);  // qkv scratch is free here
  // the last layer's FC2 output is still pending in inst->delta
  rc = launch_gather_rows_f32(inst->resid, rows_dev, n_rows, m.hidden, gathered, s,
                              m.n_layers > 0 ? inst->delta : nullptr);
  if (rc) return rc;
  rc = m.arch == TK_ARCH_OPT
           ? launch_layernorm(gathered, w->fln_w, w->fln_b, inst->xn, n_rows, m.hidden, m.norm_eps, s)
           : launch_rmsnorm(gathered, w->fln_w, inst->xn, n_rows, m.hidden, m.norm_eps, s);
  if (rc) return rc;
  rc = profiled(inst, s, PK_HEAD, 2.0 * n_rows * w->head_rows * m.hidden,
                (static_cast<double>(w->head_rows) * m.hidden + n_rows * m.hidden) * 2 +
                    static_cast<double>(n_rows) * w->head_rows * 4,
                [&] {
                  return gemm_bf16(inst->xn, w->head, inst->logits, nullptr, n_rows, w->head_rows,
                                   m.hidden, EPI_F32, inst->gemm_ws, inst->gemm_ws_bytes, s);
                });
  if (rc) return rc;
  const int cols = m.n_labels > 0 ? m.n_labels : m.vocab;
  return launch_argmax_strided(inst->logits, n_rows, cols, w->head_rows, tokens_dev, s);
}

}  // namespace tk

using namespace tk;

// ================================================================== C ABI
extern "C" {

const char* tk_last_error(void) { return g_err.c_str(); }

int tk_version(void) { return 10000; }

int tk_device_count(int32_t* n) {
  int c = 0;
  TK_CUDA(cudaGetDeviceCount(&c));
  *n = c;
  return TK_OK;
}

int tk_instance_create(int32_t device, const tk_model_desc* model, uint64_t seed,
                       int32_t kv_pages, int32_t page_tokens, int32_t max_chunk,
                       tk_instance** out) {
  TK_CHECK(model && out, TK_EINVAL, "tk_instance_create: null argument");
  int rc = validate_desc(*model);
  if (rc) return rc;
  TK_CHECK(kv_pages >= 0 && page_tokens > 0 && max_chunk > 0, TK_EINVAL,
           "tk_instance_create: kv_pages/page_tokens/max_chunk");
  TK_CUDA(cudaSetDevice(device));
  {
    // peer access to every other device (NVLink P2P for the KV handoff)
    int nd = 0;
    cudaGetDeviceCount(&nd);
    for (int d = 0; d < nd; ++d) {
      if (d == device) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, device, d);
      if (can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "peer", __FILE__, __LINE__);
        cudaGetLastError();
      }
    }
  }
  std::unique_ptr<tk_instance> inst(new tk_instance());
  inst->device = device;
  rc = acquire_weights(device, *model, seed, &inst->w);
  if (rc) return rc;
  const tk_model_desc& m = *model;
  inst->geom = KvGeom{m.n_layers, m.n_heads, m.head_dim, page_tokens};
  inst->kv_pages = kv_pages;
  inst->page_bytes = static_cast<int64_t>(inst->geom.page_elems()) * 2;
  inst->max_chunk = max_chunk;
  if (kv_pages > 0) {
    // one page past the pool: the K/V of padding rows of graph decode steps
    TK_CUDA(cudaMalloc(&inst->pool, inst->page_bytes * (kv_pages + 1)));
    // stale slots are read (and masked) by whole-page loads: keep them finite
    TK_CUDA(cudaMemset(inst->pool, 0, inst->page_bytes * (kv_pages + 1)));
  }
  TK_CUDA(cudaStreamCreateWithFlags(&inst->s_compute, cudaStreamNonBlocking));
  TK_CUDA(cudaStreamCreateWithFlags(&inst->s_copy, cudaStreamNonBlocking));
  TK_CUDA(cudaStreamCreateWithFlags(&inst->s_pred, cudaStreamNonBlocking));
  const int64_t rows = max_chunk;
  const int ffn_cols = m.arch == TK_ARCH_OPT ? m.ffn : 3 * m.ffn;
  // The fp32 residual stream and the pending bf16 update are one allocation;
  // TK_L2_PERSIST=1 keeps it in a persisting L2 window on the compute stream (the
  // add+norm re-reads both after the weight stream and the KV pages went through
  // L2).  Off by default: in situ the norms gain <1% (they are bound by their
  // launch ramp and tail, not by DRAM; profiles/r02_experiments.md).
  TK_CUDA(cudaMalloc(&inst->resid, rows * m.hidden * 6));
  inst->delta = reinterpret_cast<__nv_bfloat16*>(inst->resid + rows * m.hidden);
  {
    static const bool persist = getenv("TK_L2_PERSIST") && atoi(getenv("TK_L2_PERSIST")) != 0;
    cudaDeviceProp prop{};
    TK_CUDA(cudaGetDeviceProperties(&prop, device));
    const size_t want = static_cast<size_t>(rows) * m.hidden * 6;
    if (persist && prop.persistingL2CacheMaxSize > 0 && prop.accessPolicyMaxWindowSize > 0) {
      size_t cur = 0;
      TK_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
      const size_t lim = std::min<size_t>(prop.persistingL2CacheMaxSize, cur + want);
      TK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim));
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = inst->resid;
      attr.accessPolicyWindow.num_bytes = std::min<size_t>(want, prop.accessPolicyMaxWindowSize);
      attr.accessPolicyWindow.hitRatio = 1.0f;
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      TK_CUDA(cudaStreamSetAttribute(inst->s_compute, cudaStreamAttributeAccessPolicyWindow, &attr));
    }
  }
  TK_CUDA(cudaMalloc(&inst->xn, rows * m.hidden * 2));
  // qkv scratch doubles as the fp32 gather buffer of the head
  TK_CUDA(cudaMalloc(&inst->qkv, rows * std::max<int64_t>(3 * m.hidden * 2, m.hidden * 4)));
  TK_CUDA(cudaMalloc(&inst->attn, rows * m.hidden * 2));
  TK_CUDA(cudaMalloc(&inst->ffn, rows * ffn_cols * 2));
  inst->max_emit = max_chunk;
  TK_CUDA(cudaMalloc(&inst->logits, rows * static_cast<int64_t>(inst->w->head_rows) * 4));
  // The stream-K plan depends on M only through ceil(M/128): size the shared
  // workspace for every row count a call may use.
  int64_t ws = 0;
  const int gate_up = m.arch == TK_ARCH_OPT ? m.ffn : 2 * m.ffn;
  for (int rows_m = 128; rows_m < max_chunk + 128; rows_m += 128) {
    const int mm = std::min(rows_m, max_chunk);
    ws = std::max(ws, gemm_workspace_bytes(mm, 3 * m.hidden, m.hidden));
    ws = std::max(ws, gemm_workspace_bytes(mm, m.hidden, m.hidden));
    ws = std::max(ws, gemm_workspace_bytes(mm, gate_up, m.hidden));
    ws = std::max(ws, gemm_workspace_bytes(mm, m.hidden, m.ffn));
    ws = std::max(ws, gemm_workspace_bytes(mm, inst->w->head_rows, m.hidden));
  }
  inst->gemm_ws_bytes = ws;
  TK_CUDA(cudaMalloc(&inst->gemm_ws, ws));
  TK_CUDA(cudaMemset(inst->gemm_ws, 0, ws));
  inst->dec_max_ctx = std::max(1, kv_pages) * page_tokens;
  inst->dec_ws_bytes = decode_attention_workspace_bytes(max_chunk, m.n_heads, m.head_dim,
                                                        std::min(inst->dec_max_ctx, 1 << 16));
  TK_CUDA(cudaMalloc(&inst->dec_ws, inst->dec_ws_bytes));
  inst->dec_fixed_bytes = kSlotBytes;
  TK_CUDA(cudaMalloc(&inst->dec_fixed, inst->dec_fixed_bytes));
  TK_CUDA(cudaMalloc(&inst->attn_partial, attn_partial_bytes(m.n_heads, m.head_dim)));
  // zeroed once: the attention kernel's per-group arrival counters live at its end
  TK_CUDA(cudaMemset(inst->attn_partial, 0, attn_partial_bytes(m.n_heads, m.head_dim)));
  for (auto& s : inst->ring) {
    TK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.host), kSlotBytes, cudaHostAllocDefault));
    TK_CUDA(cudaMalloc(&s.dev, kSlotBytes));
    TK_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    TK_CUDA(cudaEventRecord(s.done, inst->s_compute));
  }
  TK_CUDA(cudaDeviceSynchronize());
  *out = inst.release();
  return TK_OK;
}

int tk_instance_destroy(tk_instance* inst) {
  if (!inst) return TK_OK;
  cudaSetDevice(inst->device);
  cudaDeviceSynchronize();
  for (auto& s : inst->ring) {
    if (tk_event* ev = s.owner) {
      finalize_event(ev);  // clears s.owner
      ev->slot = nullptr;
      maybe_free_event(ev);
    }
    cudaFreeHost(s.host);
    cudaFree(s.dev);
    cudaEventDestroy(s.done);
  }
  for (auto& kv : inst->dec_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  cudaFree(inst->dec_fixed);
  cudaFree(inst->pool);
  cudaFree(inst->resid);  // (delta lives in the same allocation)
  cudaFree(inst->xn);
  cudaFree(inst->qkv);
  cudaFree(inst->attn);
  cudaFree(inst->ffn);
  cudaFree(inst->logits);
  cudaFree(inst->gemm_ws);
  cudaFree(inst->dec_ws);
  cudaFree(inst->attn_partial);
  cudaStreamDestroy(inst->s_compute);
  cudaStreamDestroy(inst->s_copy);
  cudaStreamDestroy(inst->s_pred);
  release_weights(inst->w);
  delete inst;
  return TK_OK;
}

int tk_instance_info(tk_instance* inst, int64_t* weight_bytes, int64_t* page_bytes,
                     int64_t* kv_pool_bytes) {
  TK_CHECK(inst, TK_EINVAL, "null instance");
  if (weight_bytes) *weight_bytes = inst->w->bytes;
  if (page_bytes) *page_bytes = inst->page_bytes;
  if (kv_pool_bytes) *kv_pool_bytes = inst->page_bytes * inst->kv_pages;
  return TK_OK;
}

int tk_weight_numel(tk_instance* inst, const char* name, int64_t* numel) {
  TK_CHECK(inst && name && numel, TK_EINVAL, "null argument");
  auto it = inst->w->named.find(name);
  TK_CHECK(it != inst->w->named.end(), TK_EINVAL, std::string("unknown tensor ") + name);
  *numel = it->second.numel;
  return TK_OK;
}

int tk_weight_read(tk_instance* inst, const char* name, uint16_t* host, int64_t numel) {
  int64_t n;
  int rc = tk_weight_numel(inst, name, &n);
  if (rc) return rc;
  TK_CHECK(n == numel, TK_EINVAL, "tk_weight_read: numel mismatch");
  TK_CUDA(cudaSetDevice(inst->device));
  TK_CUDA(cudaDeviceSynchronize());
  TK_CUDA(cudaMemcpy(host, inst->w->named[name].ptr, n * 2, cudaMemcpyDeviceToHost));
  return TK_OK;
}

int tk_weight_write(tk_instance* inst, const char* name, const uint16_t* host, int64_t numel) {
  int64_t n;
  int rc = tk_weight_numel(inst, name, &n);
  if (rc) return rc;
  TK_CHECK(n == numel, TK_EINVAL, "tk_weight_write: numel mismatch");
  TK_CUDA(cudaSetDevice(inst->device));
  TK_CUDA(cudaDeviceSynchronize());
  TK_CUDA(cudaMemcpy(inst->w->named[name].ptr, host, n * 2, cudaMemcpyHostToDevice));
  return TK_OK;
}

int tk_kv_read(tk_instance* inst, int32_t page, uint16_t* host) {
  TK_CHECK(inst && host, TK_EINVAL, "null argument");
  TK_CHECK(page >= 0 && page < inst->kv_pages, TK_ECAPACITY, "tk_kv_read: page out of pool");
  TK_CUDA(cudaSetDevice(inst->device));
  TK_CUDA(cudaDeviceSynchronize());
  TK_CUDA(cudaMemcpy(host, reinterpret_cast<uint8_t*>(inst->pool) + page * inst->page_bytes,
                     inst->page_bytes, cudaMemcpyDeviceToHost));
  return TK_OK;
}

// ------------------------------------------------------------------ prefill chunk
static int prefill_impl(tk_instance* inst, cudaStream_t s, int32_t n_tokens,
                        const int32_t* token_ids, const tk_slice* slices, int32_t n_slices,
                        const int32_t* block_tables, int32_t n_bt, int32_t* tokens_out,
                        float* logits_out, tk_event** ev_out, bool classify_only) {
  const tk_model_desc& m = inst->w->md;
  TK_CHECK(n_tokens > 0 && n_tokens <= inst->max_chunk, TK_EINVAL,
           "prefill: n_tokens must be in [1, max_chunk]");
  TK_CHECK(n_slices > 0 && slices && token_ids && block_tables, TK_EINVAL,
           "prefill: slices, ids and block tables required");
  TK_CUDA(cudaSetDevice(inst->device));
  Slot* slot;
  int rc = take_slot(inst, &slot);
  if (rc) return rc;
  Packer pk{slot};
  int32_t* ids_d;
  pk.put(token_ids, n_tokens, &ids_d);
  TokenMeta* meta_d;
  TokenMeta* meta = pk.put<TokenMeta>(nullptr, n_tokens, &meta_d);
  tk_slice* sl_d;
  pk.put(slices, n_slices, &sl_d);
  int32_t* bt_d;
  pk.put(block_tables, n_bt, &bt_d);
  const int pt = inst->geom.page_tokens;
  std::vector<int32_t> emit_rows;
  int row = 0;
  for (int i = 0; i < n_slices; ++i) {
    const tk_slice& sl = slices[i];
    TK_CHECK(sl.len > 0 && sl.start >= 0, TK_EINVAL, "prefill: slice len/start");
    TK_CHECK(sl.bt_offset >= 0 && sl.bt_offset + sl.n_pages <= n_bt, TK_EINVAL,
             "prefill: slice block-table range");
    TK_CHECK(static_cast<int64_t>(sl.n_pages) * pt >= sl.start + sl.len, TK_EINVAL,
             "prefill: slice pages do not cover start+len");
    TK_CHECK(m.arch != TK_ARCH_OPT || sl.start + sl.len <= m.max_positions, TK_EINVAL,
             "prefill: position beyond max_positions");
    TK_CHECK(row + sl.len <= n_tokens, TK_EINVAL, "prefill: slices exceed n_tokens");
    for (int t = 0; t < sl.len; ++t) {
      const int pos = sl.start + t;
      const int page = block_tables[sl.bt_offset + pos / pt];
      TK_CHECK(page >= 0 && page < inst->kv_pages, TK_ECAPACITY, "prefill: page id out of pool");
      meta[row + t] = TokenMeta{pos, page, pos % pt, i};
    }
    row += sl.len;
    if (sl.emit) emit_rows.push_back(row - 1);
  }
  TK_CHECK(row == n_tokens, TK_EINVAL, "prefill: slice lengths must sum to n_tokens");
  for (int t = 0; t < n_tokens; ++t)
    TK_CHECK(token_ids[t] >= 0 && token_ids[t] < m.vocab, TK_EINVAL, "prefill: token id");
  const int n_emit = static_cast<int>(emit_rows.size());
  int32_t* emit_d;
  pk.put(emit_rows.data(), n_emit, &emit_d);
  const bool tc_attn = use_tc_attention(m.head_dim);
  AttnQBlock* qb_d = nullptr;
  AttnWork* work_d = nullptr;
  int n_qb = 0, n_work = 0;
  bool any_split = false;
  FaPlan fa{};
  FaPair* fa_pairs_d = nullptr;
  FaUnit* fa_units_d = nullptr;
  FaGroup* fa_groups_d = nullptr;
  int32_t* fa_off_d = nullptr;
  if (tc_attn) {
    const int pcap = n_slices + n_tokens / 256 + 1;
    const int ucap = pcap * m.n_heads + kNumSMs + 1;
    FaPair* pairs = pk.put<FaPair>(nullptr, pcap, &fa_pairs_d);
    FaUnit* units = pk.put<FaUnit>(nullptr, ucap, &fa_units_d);
    FaGroup* groups = pk.put<FaGroup>(nullptr, pcap * m.n_heads, &fa_groups_d);
    int32_t* off = pk.put<int32_t>(nullptr, kNumSMs + 1, &fa_off_d);
    TK_CHECK(pk.ok(), TK_EINVAL, "prefill: metadata exceeds staging slot");
    // attention CTAs (TK_FA_CTAS caps them, experiments)
    static const int fa_ctas = getenv("TK_FA_CTAS") ? std::max(1, std::min(kNumSMs, atoi(getenv("TK_FA_CTAS"))))
                                                    : kNumSMs;
    const int span = fa_span(m.head_dim);
    TK_CHECK(build_fa_plan(slices, n_slices, m.n_heads, span > 256 ? fa_ctas / 2 : fa_ctas, &fa,
                           pairs, pcap, units, ucap, groups, pcap * m.n_heads, off, kNumSMs + 1,
                           span) == 0,
             TK_EINVAL, "prefill: attention plan overflow");
  } else {
    const int qcap = n_slices + n_tokens / 128 + 1;
    AttnQBlock* qbs = pk.put<AttnQBlock>(nullptr, qcap, &qb_d);
    AttnWork* work = pk.put<AttnWork>(nullptr, qcap + kAttnMaxSplitSlots, &work_d);
    TK_CHECK(pk.ok(), TK_EINVAL, "prefill: metadata exceeds staging slot");
    n_work = build_attn_work(slices, n_slices, m.n_heads, qbs, qcap, work,
                             qcap + kAttnMaxSplitSlots, &n_qb, 64);
    TK_CHECK(n_work >= 0, TK_EINVAL, "prefill: attention work list overflow");
    for (int k = 0; k < n_qb; ++k) any_split |= qbs[k].n_splits > 1;
  }
  int32_t* out_d;
  int32_t* out_h = pk.put<int32_t>(nullptr, std::max(1, n_slices), &out_d);
  int32_t* tok_d;
  pk.put<int32_t>(nullptr, std::max(1, n_emit), &tok_d);
  TK_CHECK(pk.ok(), TK_EINVAL, "prefill: metadata exceeds staging slot");

  tk_event* ev;
  rc = new_event(inst, s, &ev);
  if (rc) return rc;
  TK_CUDA(cudaMemcpyAsync(slot->dev, slot->host, pk.off, cudaMemcpyHostToDevice, s));
  inst->last_h2d = pk.off;
  inst->last_d2h = static_cast<int64_t>(n_emit) * 4;
  const int h = m.hidden;
  rc = m.arch == TK_ARCH_OPT
           ? launch_embed_opt(ids_d, meta_d, n_tokens, inst->w->embed, inst->w->pos, inst->resid, h, s)
           : launch_embed_llama(ids_d, n_tokens, inst->w->embed, inst->resid, h, s);
  if (rc) return rc;
  const float scale = attn_scale(m);
  double ctx_sum = 0;  // sum over query rows of keys attended (pos + 1)
  for (int t = 0; t < n_tokens; ++t) ctx_sum += meta[t].pos + 1;
  const double attn_flops = 4.0 * m.head_dim * m.n_heads * ctx_sum;
  int64_t prefix_tokens = 0;
  for (int i = 0; i < n_slices; ++i) prefix_tokens += slices[i].start + slices[i].len;
  const double attn_bytes = 2.0 * m.hidden * 2 * prefix_tokens + 2.0 * n_tokens * m.hidden * 2;
  for (int l = 0; l < m.n_layers; ++l) {
    rc = run_layer(inst, l, n_tokens, meta_d, s, attn_flops, attn_bytes, [&]() {
      if (tc_attn)
        return launch_chunk_attention_fa(inst->qkv, inst->max_chunk, 3 * h, inst->attn, inst->pool,
                                         inst->kv_pages, inst->geom, l, fa, fa_pairs_d, fa_units_d,
                                         fa_groups_d, fa_off_d, sl_d, bt_d, scale,
                                         inst->attn_partial, s);
      return launch_chunk_attention_work(inst->qkv, 3 * h, inst->attn, inst->pool, inst->geom, l,
                                         work_d, n_work, qb_d, n_qb, any_split, sl_d, bt_d, scale,
                                         inst->attn_partial, s);
    });
    if (rc) return rc;
  }
  if (n_emit > 0) {
    rc = run_head(inst, n_emit, emit_d, tok_d, s);
    if (rc) return rc;
  }
  int32_t* map_d;
  int32_t* map_h = pk.put<int32_t>(nullptr, n_slices, &map_d);
  TK_CHECK(pk.ok(), TK_EINVAL, "prefill: metadata exceeds staging slot");
  for (int i = 0, e = 0; i < n_slices; ++i) map_h[i] = slices[i].emit ? e++ : -1;
  if (n_emit > 0)
    TK_CUDA(cudaMemcpyAsync(out_h, tok_d, n_emit * 4, cudaMemcpyDeviceToHost, s));
  TK_CUDA(cudaEventRecord(ev->end, s));
  TK_CUDA(cudaEventRecord(slot->done, s));
  ev->slot = slot;
  slot->owner = ev;
  if (tokens_out) {
    ev->out_src = out_h;
    ev->out_dst = tokens_out;
    ev->remap = classify_only ? nullptr : map_h;
    ev->n_out = classify_only ? n_emit : n_slices;
  }
  if (logits_out && n_emit > 0) {
    TK_CUDA(cudaStreamSynchronize(s));
    const int cols = m.n_labels > 0 ? m.n_labels : m.vocab;
    TK_CUDA(cudaMemcpy2D(logits_out, cols * 4, inst->logits, inst->w->head_rows * 4, cols * 4,
                         n_emit, cudaMemcpyDeviceToHost));
  }
  *ev_out = ev;
  return TK_OK;
}

int tk_prefill_chunk(tk_instance* inst, int32_t n_tokens, const int32_t* token_ids,
                     const tk_slice* slices, int32_t n_slices, const int32_t* block_tables,
                     int32_t n_block_entries, int32_t* first_tokens_out, float* logits_out,
                     tk_event** ev) {
  TK_CHECK(inst && ev, TK_EINVAL, "tk_prefill_chunk: null argument");
  TK_CHECK(inst->pool != nullptr, TK_ECAPACITY, "tk_prefill_chunk: instance has no KV pool");
  return prefill_impl(inst, inst->s_compute, n_tokens, token_ids, slices, n_slices, block_tables,
                      n_block_entries, first_tokens_out, logits_out, ev, false);
}

// ------------------------------------------------------------------ decode step
// The device work of one decode step over `batch` rows whose inputs sit at the given
// device addresses: embed, every layer (KV append, split-KV paged attention, GEMMs),
// head + argmax.  Run eagerly, or recorded once per shape bucket into a CUDA graph.
static int decode_body(tk_instance* inst, cudaStream_t s, int batch, const int32_t* ids_d,
                       const TokenMeta* meta_d, const int32_t* lens_d, const int32_t* bt_d,
                       int bt_stride, const int32_t* rows_d, int32_t* out_d, int max_ctx,
                       double attn_flops, double attn_bytes) {
  const tk_model_desc& m = inst->w->md;
  const int h = m.hidden;
  int rc = m.arch == TK_ARCH_OPT
               ? launch_embed_opt(ids_d, meta_d, batch, inst->w->embed, inst->w->pos, inst->resid, h, s)
               : launch_embed_llama(ids_d, batch, inst->w->embed, inst->resid, h, s);
  if (rc) return rc;
  const float scale = attn_scale(m);
  for (int l = 0; l < m.n_layers; ++l) {
    rc = run_layer(inst, l, batch, meta_d, s, attn_flops, attn_bytes, [&]() {
      return launch_decode_attention(inst->qkv, 3 * h, inst->attn, inst->pool, inst->geom, l, bt_d,
                                     bt_stride, lens_d, batch, max_ctx, scale, inst->dec_ws,
                                     inst->dec_ws_bytes, s);
    });
    if (rc) return rc;
  }
  return run_head(inst, batch, rows_d, out_d, s);
}

static bool decode_graphs_on() {
  static const bool on = getenv("TK_NO_DECODE_GRAPH") == nullptr;
  return on;
}

// Graph batch bucket: the skinny GEMM's batch widths (16/32/64/128), then steps of 32.
static int decode_batch_bucket(int batch, int cap) {
  int b = 16;
  while (b < batch && b < 128) b *= 2;
  if (batch > 128) b = (batch + 31) / 32 * 32;
  return std::min(std::max(b, batch), cap);
}

int tk_decode_step(tk_instance* inst, int32_t batch, const int32_t* last_tokens,
                   const int32_t* ctx_lens, const int32_t* block_tables, int32_t bt_stride,
                   int32_t* next_tokens_out, float* logits_out, tk_event** ev_out) {
  TK_CHECK(inst && ev_out && last_tokens && ctx_lens && block_tables, TK_EINVAL,
           "tk_decode_step: null argument");
  TK_CHECK(batch > 0 && batch <= inst->max_chunk, TK_EINVAL, "tk_decode_step: batch");
  const tk_model_desc& m = inst->w->md;
  TK_CHECK(m.n_labels == 0, TK_EUNSUPPORTED, "tk_decode_step: classifier instance");
  TK_CUDA(cudaSetDevice(inst->device));
  cudaStream_t s = inst->s_compute;
  const int pt = inst->geom.page_tokens;
  int max_ctx = 0;
  double kv_sum = 0;
  for (int b = 0; b < batch; ++b) {
    const int ctx = ctx_lens[b];
    TK_CHECK(ctx >= 0 && (ctx / pt) < bt_stride, TK_EINVAL, "tk_decode_step: ctx beyond block table");
    TK_CHECK(m.arch != TK_ARCH_OPT || ctx < m.max_positions, TK_EINVAL,
             "tk_decode_step: position beyond max_positions");
    TK_CHECK(last_tokens[b] >= 0 && last_tokens[b] < m.vocab, TK_EINVAL, "tk_decode_step: token");
    const int page = block_tables[static_cast<int64_t>(b) * bt_stride + ctx / pt];
    TK_CHECK(page >= 0 && page < inst->kv_pages, TK_ECAPACITY, "tk_decode_step: page out of pool");
    max_ctx = std::max(max_ctx, ctx + 1);
    kv_sum += ctx + 1;
  }
  TK_CHECK(decode_attention_workspace_bytes(batch, m.n_heads, m.head_dim, max_ctx) <=
               inst->dec_ws_bytes,
           TK_EINVAL, "tk_decode_step: context exceeds attention workspace");
  const double attn_flops = 4.0 * m.head_dim * m.n_heads * kv_sum;
  // K and V of every attended token read once, Q read, O written (one layer)
  const double attn_bytes = kv_sum * 2.0 * m.hidden * 2 + 2.0 * batch * m.hidden * 2;

  // Graph mode: the step padded to a batch bucket and a context bucket (1024 tokens),
  // inputs copied to fixed device addresses; padding rows are token 0 at position 0
  // whose K/V go to the scratch page and whose outputs are dropped.
  bool graph = decode_graphs_on() && !inst->prof && logits_out == nullptr && inst->kv_pages > 0;
  int rows_p = batch, ctx_p = max_ctx, stride_p = bt_stride;
  if (graph) {
    rows_p = decode_batch_bucket(batch, inst->max_chunk);
    ctx_p = std::max(max_ctx, std::min((max_ctx + 1023) / 1024 * 1024, inst->dec_max_ctx));
    if (decode_attention_workspace_bytes(rows_p, m.n_heads, m.head_dim, ctx_p) > inst->dec_ws_bytes)
      ctx_p = max_ctx;
    stride_p = (ctx_p + pt - 1) / pt;
    graph = decode_attention_workspace_bytes(rows_p, m.n_heads, m.head_dim, ctx_p) <=
            inst->dec_ws_bytes;
  }
  if (!graph) {
    rows_p = batch;
    ctx_p = max_ctx;
    stride_p = bt_stride;
  }
  Slot* slot;
  int rc = take_slot(inst, &slot);
  if (rc) return rc;
  Packer pk{slot};
  int32_t* ids_d;
  int32_t* ids = pk.put<int32_t>(nullptr, rows_p, &ids_d);
  TokenMeta* meta_d;
  TokenMeta* meta = pk.put<TokenMeta>(nullptr, rows_p, &meta_d);
  int32_t* lens_d;
  int32_t* lens = pk.put<int32_t>(nullptr, rows_p, &lens_d);
  int32_t* rows_d;
  int32_t* rows = pk.put<int32_t>(nullptr, rows_p, &rows_d);
  int32_t* bt_d;
  int32_t* bt = pk.put<int32_t>(nullptr, static_cast<int64_t>(rows_p) * stride_p, &bt_d);
  const int64_t in_bytes = pk.off;
  int32_t* out_d;
  int32_t* out_h = pk.put<int32_t>(nullptr, rows_p, &out_d);
  TK_CHECK(pk.ok() && pk.off <= inst->dec_fixed_bytes, TK_EINVAL,
           "tk_decode_step: metadata exceeds staging slot");
  const int trash = inst->kv_pages;  // the page past the pool (graph padding rows)
  for (int b = 0; b < rows_p; ++b) {
    int32_t* row_bt = bt + static_cast<int64_t>(b) * stride_p;
    if (b < batch) {
      const int ctx = ctx_lens[b];
      const int32_t* src = block_tables + static_cast<int64_t>(b) * bt_stride;
      const int ncopy = std::min(bt_stride, stride_p);
      memcpy(row_bt, src, static_cast<size_t>(ncopy) * 4);
      for (int j = ncopy; j < stride_p; ++j) row_bt[j] = src[0];  // never read (ctx bound)
      ids[b] = last_tokens[b];
      meta[b] = TokenMeta{ctx, src[ctx / pt], ctx % pt, b};
      lens[b] = ctx + 1;
    } else {
      for (int j = 0; j < stride_p; ++j) row_bt[j] = trash;
      ids[b] = 0;
      meta[b] = TokenMeta{0, trash, 0, b};
      lens[b] = 1;
    }
    rows[b] = b;
  }
  tk_event* ev;
  rc = new_event(inst, s, &ev);
  if (rc) return rc;
  inst->last_h2d = in_bytes;
  inst->last_d2h = static_cast<int64_t>(batch) * 4;
  if (!graph) {
    TK_CUDA(cudaMemcpyAsync(slot->dev, slot->host, in_bytes, cudaMemcpyHostToDevice, s));
    rc = decode_body(inst, s, batch, ids_d, meta_d, lens_d, bt_d, stride_p, rows_d, out_d,
                     max_ctx, attn_flops, attn_bytes);
    if (rc) return rc;
  } else {
    auto fixed = [&](auto* p) {
      return reinterpret_cast<decltype(p)>(inst->dec_fixed +
                                           (reinterpret_cast<uint8_t*>(p) - slot->dev));
    };
    TK_CUDA(cudaMemcpyAsync(inst->dec_fixed, slot->host, in_bytes, cudaMemcpyHostToDevice, s));
    const int32_t* fids = fixed(ids_d);
    const TokenMeta* fmeta = fixed(meta_d);
    const int32_t* flens = fixed(lens_d);
    const int32_t* frows = fixed(rows_d);
    const int32_t* fbt = fixed(bt_d);
    out_d = fixed(out_d);
    auto body = [&]() {
      return decode_body(inst, s, rows_p, fids, fmeta, flens, fbt, stride_p, frows, out_d, ctx_p,
                         attn_flops, attn_bytes);
    };
    const uint64_t key = (static_cast<uint64_t>(rows_p) << 32) | static_cast<uint32_t>(ctx_p);
    auto& g = inst->dec_graphs[key];
    if (g.exec) {
      TK_CUDA(cudaGraphLaunch(g.exec, s));
      g_launches.fetch_add(g.launches, std::memory_order_relaxed);
    } else if (g.failed || g.seen++ == 0) {
      // first use of a shape: eager (sets kernel attributes, plans, tensor maps)
      rc = body();
      if (rc) return rc;
    } else {
      const int64_t l0 = g_launches.load();
      TK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      rc = body();
      cudaGraph_t cg = nullptr;
      const cudaError_t e = cudaStreamEndCapture(s, &cg);
      const int64_t n = g_launches.load() - l0;
      g_launches.fetch_sub(n, std::memory_order_relaxed);  // recorded, not run
      cudaError_t ie = cudaErrorUnknown;
      if (rc == TK_OK && e == cudaSuccess && cg) ie = cudaGraphInstantiate(&g.exec, cg, 0);
      if (cg) cudaGraphDestroy(cg);
      if (ie != cudaSuccess) {
        cudaGetLastError();
        g.exec = nullptr;
        g.failed = true;  // this shape stays eager
        rc = body();
        if (rc) return rc;
      } else {
        g.launches = n;
        TK_CUDA(cudaGraphLaunch(g.exec, s));
        g_launches.fetch_add(n, std::memory_order_relaxed);
      }
    }
  }
  TK_CUDA(cudaMemcpyAsync(out_h, out_d, batch * 4, cudaMemcpyDeviceToHost, s));
  TK_CUDA(cudaEventRecord(ev->end, s));
  TK_CUDA(cudaEventRecord(slot->done, s));
  ev->slot = slot;
  slot->owner = ev;
  if (next_tokens_out) {
    ev->out_src = out_h;
    ev->out_dst = next_tokens_out;
    ev->n_out = batch;
  }
  if (logits_out) {
    TK_CUDA(cudaStreamSynchronize(s));
    TK_CUDA(cudaMemcpy2D(logits_out, m.vocab * 4, inst->logits, inst->w->head_rows * 4,
                         m.vocab * 4, batch, cudaMemcpyDeviceToHost));
  }
  *ev_out = ev;
  return TK_OK;
}

// ------------------------------------------------------------------ KV handoff
int tk_kv_send(tk_instance* src, const int32_t* src_pages, tk_instance* dst,
               const int32_t* dst_pages, int32_t n_pages, tk_event** ev_out) {
  return tk_kv_send_ex(src, src_pages, dst, dst_pages, n_pages, TK_SEND_AUTO, ev_out);
}

int tk_kv_send_ex(tk_instance* src, const int32_t* src_pages, tk_instance* dst,
                  const int32_t* dst_pages, int32_t n_pages, int32_t engine, tk_event** ev_out) {
  TK_CHECK(src && dst && ev_out && (n_pages == 0 || (src_pages && dst_pages)), TK_EINVAL,
           "tk_kv_send: null argument");
  TK_CHECK(engine == TK_SEND_AUTO || engine == TK_SEND_SM || engine == TK_SEND_CE, TK_EINVAL,
           "tk_kv_send: engine must be TK_SEND_AUTO, TK_SEND_SM or TK_SEND_CE");
  TK_CHECK(src->page_bytes == dst->page_bytes, TK_EINVAL, "tk_kv_send: page geometry differs");
  for (int i = 0; i < n_pages; ++i)
    TK_CHECK(src_pages[i] >= 0 && src_pages[i] < src->kv_pages && dst_pages[i] >= 0 &&
                 dst_pages[i] < dst->kv_pages,
             TK_ECAPACITY, "tk_kv_send: page out of pool");
  TK_CUDA(cudaSetDevice(src->device));
  // order after everything already issued on the source's compute stream
  cudaEvent_t after;
  TK_CUDA(cudaEventCreateWithFlags(&after, cudaEventDisableTiming));
  TK_CUDA(cudaEventRecord(after, src->s_compute));
  TK_CUDA(cudaStreamWaitEvent(src->s_copy, after, 0));
  TK_CUDA(cudaEventDestroy(after));
  tk_event* ev;
  int rc = new_event(src, src->s_copy, &ev);
  if (rc) return rc;
  const int64_t pb = src->page_bytes;
  int peer = src->device == dst->device;
  if (!peer) TK_CUDA(cudaDeviceCanAccessPeer(&peer, src->device, dst->device));
  TK_CHECK(peer || engine != TK_SEND_SM, TK_EINVAL,
           "tk_kv_send: TK_SEND_SM needs peer access from src to dst");
  // AUTO: the page-copy kernel for a device-local handoff (co-located P and D: 2.2 vs
  // 4.2 ms for 8k tokens, the copy engines starve beside the chunk's GEMMs), the copy
  // engines across devices: the NVLink transfer then takes no SMs from the next chunk
  // (bench kv_handoff_nvlink / overlap_nvlink measure both engines).
  const bool use_sm = engine == TK_SEND_SM || (engine == TK_SEND_AUTO && src->device == dst->device);
  if (peer && use_sm) {
    // one copy kernel on the source GPU; a peer destination is written over NVLink
    int sms = 0;
    TK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, src->device));
    rc = launch_kv_copy_pages(src->pool, dst->pool, pb, src_pages, dst_pages, n_pages, sms,
                              src->s_copy);
    if (rc) return rc;
  } else {
    for (int i = 0; i < n_pages;) {
      // copy engine (requested, or no peer path): runs of consecutive pages coalesced
      int j = i + 1;
      while (j < n_pages && src_pages[j] == src_pages[j - 1] + 1 &&
             dst_pages[j] == dst_pages[j - 1] + 1)
        ++j;
      uint8_t* d = reinterpret_cast<uint8_t*>(dst->pool) + dst_pages[i] * pb;
      const uint8_t* sp = reinterpret_cast<const uint8_t*>(src->pool) + src_pages[i] * pb;
      TK_CUDA(cudaMemcpyPeerAsync(d, dst->device, sp, src->device, (j - i) * pb, src->s_copy));
      i = j;
    }
  }
  TK_CUDA(cudaEventRecord(ev->end, src->s_copy));
  *ev_out = ev;
  return TK_OK;
}

// ------------------------------------------------------------------ predictor
static int predict_impl(tk_instance* inst, const int32_t* token_ids, const int32_t* lens,
                        int32_t n, int32_t max_len, int32_t* bucket_out, float* scores_out,
                        tk_event** ev) {
  TK_CHECK(inst && ev && token_ids && lens && n > 0, TK_EINVAL, "tk_predict: null argument");
  TK_CHECK(inst->w->md.n_labels > 0, TK_EINVAL, "tk_predict: instance has no classifier head");
  const int pt = inst->geom.page_tokens;
  std::vector<tk_slice> sl(n);
  std::vector<int32_t> ids;
  std::vector<int32_t> bt;
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int len = std::min(lens[i], max_len);
    TK_CHECK(len > 0, TK_EINVAL, "tk_predict: empty prompt");
    const int np = (len + pt - 1) / pt;
    sl[i] = tk_slice{0, len, static_cast<int32_t>(bt.size()), np, 1};
    for (int p = 0; p < np; ++p) bt.push_back(static_cast<int32_t>(bt.size()));
    ids.insert(ids.end(), token_ids + off, token_ids + off + len);
    off += lens[i];
  }
  TK_CHECK(static_cast<int>(bt.size()) <= inst->kv_pages, TK_ECAPACITY,
           "tk_predict: prompts exceed the predictor's page pool");
  return prefill_impl(inst, inst->s_pred, static_cast<int32_t>(ids.size()), ids.data(), sl.data(),
                      n, bt.data(), static_cast<int32_t>(bt.size()), bucket_out, scores_out, ev,
                      true);
}

int tk_predict(tk_instance* inst, const int32_t* token_ids, const int32_t* lens, int32_t n,
               int32_t max_len, int32_t* bucket_out, tk_event** ev) {
  return predict_impl(inst, token_ids, lens, n, max_len, bucket_out, nullptr, ev);
}

int tk_predict_scores(tk_instance* inst, const int32_t* token_ids, const int32_t* lens,
                      int32_t n, int32_t max_len, int32_t* bucket_out, float* scores_out,
                      tk_event** ev) {
  TK_CHECK(scores_out, TK_EINVAL, "tk_predict_scores: null scores_out");
  return predict_impl(inst, token_ids, lens, n, max_len, bucket_out, scores_out, ev);
}

// ------------------------------------------------------------------ swap
int tk_host_alloc(int64_t bytes, void** out) {
  TK_CHECK(out && bytes > 0, TK_EINVAL, "tk_host_alloc");
  TK_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return TK_OK;
}

int tk_host_free(void* p) {
  TK_CUDA(cudaFreeHost(p));
  return TK_OK;
}

static int swap_impl(tk_instance* inst, const int32_t* pages, int32_t n, void* host, bool out,
                     tk_event** ev_out) {
  TK_CHECK(inst && ev_out && (n == 0 || (pages && host)), TK_EINVAL, "swap: null argument");
  TK_CUDA(cudaSetDevice(inst->device));
  cudaEvent_t after;
  TK_CUDA(cudaEventCreateWithFlags(&after, cudaEventDisableTiming));
  TK_CUDA(cudaEventRecord(after, inst->s_compute));
  TK_CUDA(cudaStreamWaitEvent(inst->s_copy, after, 0));
  TK_CUDA(cudaEventDestroy(after));
  tk_event* ev;
  int rc = new_event(inst, inst->s_copy, &ev);
  if (rc) return rc;
  const int64_t pb = inst->page_bytes;
  for (int i = 0; i < n; ++i) {
    TK_CHECK(pages[i] >= 0 && pages[i] < inst->kv_pages, TK_ECAPACITY, "swap: page out of pool");
    uint8_t* dev = reinterpret_cast<uint8_t*>(inst->pool) + pages[i] * pb;
    uint8_t* h = static_cast<uint8_t*>(host) + i * pb;
    if (out)
      TK_CUDA(cudaMemcpyAsync(h, dev, pb, cudaMemcpyDeviceToHost, inst->s_copy));
    else
      TK_CUDA(cudaMemcpyAsync(dev, h, pb, cudaMemcpyHostToDevice, inst->s_copy));
  }
  TK_CUDA(cudaEventRecord(ev->end, inst->s_copy));
  if (!out) {
    // later compute must see the restored pages
    cudaEvent_t fin;
    TK_CUDA(cudaEventCreateWithFlags(&fin, cudaEventDisableTiming));
    TK_CUDA(cudaEventRecord(fin, inst->s_copy));
    TK_CUDA(cudaStreamWaitEvent(inst->s_compute, fin, 0));
    TK_CUDA(cudaEventDestroy(fin));
  }
  *ev_out = ev;
  return TK_OK;
}

int tk_swap_out(tk_instance* inst, const int32_t* pages, int32_t n, void* pinned_host,
                tk_event** ev) {
  return swap_impl(inst, pages, n, pinned_host, true, ev);
}

int tk_swap_in(tk_instance* inst, const int32_t* pages, int32_t n, const void* pinned_host,
               tk_event** ev) {
  return swap_impl(inst, pages, n, const_cast<void*>(pinned_host), false, ev);
}

// ------------------------------------------------------------------ events
int tk_event_query(tk_event* ev, int64_t* elapsed_ns) {
  TK_CHECK(ev, TK_EINVAL, "tk_event_query: null event");
  if (!ev->finished) {
    cudaError_t e = cudaEventQuery(ev->end);
    if (e == cudaErrorNotReady) return 0;
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventQuery", __FILE__, __LINE__);
    int rc = finalize_event(ev);
    if (rc) return rc;
  }
  if (elapsed_ns) {
    float ms = 0.f;
    TK_CUDA(cudaEventElapsedTime(&ms, ev->start, ev->end));
    *elapsed_ns = static_cast<int64_t>(ms * 1e6);
  }
  return 1;
}

int tk_event_wait(tk_event* ev, int64_t* elapsed_ns) {
  TK_CHECK(ev, TK_EINVAL, "tk_event_wait: null event");
  int rc = finalize_event(ev);
  if (rc) return rc;
  if (elapsed_ns) {
    float ms = 0.f;
    TK_CUDA(cudaEventElapsedTime(&ms, ev->start, ev->end));
    *elapsed_ns = static_cast<int64_t>(ms * 1e6);
  }
  return TK_OK;
}

int tk_event_release(tk_event* ev) {
  if (!ev) return TK_OK;
  ev->released = true;  // host outputs are abandoned from here on
  if (ev->finished) {
    maybe_free_event(ev);
  } else if (ev->slot == nullptr) {
    // no slot to free it later: never block here, park it until it completes
    if (cudaEventQuery(ev->end) == cudaSuccess) {
      ev->finished = true;
      maybe_free_event(ev);
    } else {
      cudaGetLastError();
      std::lock_guard<std::mutex> lock(g_zombie_mu);
      g_zombies.push_back(ev);
    }
  }
  // otherwise the owning slot frees it when it is finalized on reuse
  return TK_OK;
}

int tk_instance_sync(tk_instance* inst) {
  TK_CHECK(inst, TK_EINVAL, "null instance");
  TK_CUDA(cudaSetDevice(inst->device));
  TK_CUDA(cudaStreamSynchronize(inst->s_compute));
  TK_CUDA(cudaStreamSynchronize(inst->s_copy));
  TK_CUDA(cudaStreamSynchronize(inst->s_pred));
  return TK_OK;
}

// ------------------------------------------------------------------ raw kernels
int tk_gemm_bf16(const void* A, const void* B, void* C, const void* bias, int32_t M, int32_t N,
                 int32_t K, int32_t epilogue, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  return gemm_bf16(A, B, C, bias, M, N, K, epilogue, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream));
}

int tk_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int64_t* bytes) {
  TK_CHECK(bytes, TK_EINVAL, "null");
  *bytes = gemm_workspace_bytes(M, N, K);
  return TK_OK;
}

int tk_layernorm(const float* x, const void* w, const void* b, void* y, int32_t rows,
                 int32_t cols, float eps, void* stream) {
  return launch_layernorm(x, static_cast<const __nv_bfloat16*>(w),
                          static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y),
                          rows, cols, eps, static_cast<cudaStream_t>(stream));
}

int tk_argmax(const float* logits, int32_t rows, int32_t cols, int32_t row_stride, int32_t* out,
              void* stream) {
  return launch_argmax_strided(logits, rows, cols, row_stride, out,
                               static_cast<cudaStream_t>(stream));
}

int tk_paged_decode_attention(const void* q, void* o, const void* kv_pool, int32_t layer,
                              int32_t n_layers, int32_t n_heads, int32_t head_dim,
                              int32_t page_tokens, const int32_t* block_tables, int32_t bt_stride,
                              const int32_t* ctx_lens, int32_t batch, float scale, void* workspace,
                              int64_t workspace_bytes, void* stream) {
  // ctx_lens is a device array; the split count needs the maximum on the host.
  std::vector<int32_t> h(batch);
  TK_CUDA(cudaMemcpy(h.data(), ctx_lens, batch * 4, cudaMemcpyDeviceToHost));
  int max_ctx = 0;
  for (int v : h) max_ctx = std::max(max_ctx, v);
  KvGeom g{n_layers, n_heads, head_dim, page_tokens};
  return launch_decode_attention(static_cast<const __nv_bfloat16*>(q), n_heads * head_dim,
                                 static_cast<__nv_bfloat16*>(o),
                                 static_cast<const __nv_bfloat16*>(kv_pool), g, layer,
                                 block_tables, bt_stride, ctx_lens, batch, max_ctx, scale,
                                 workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

static int chunk_attention_impl(const void* q, int32_t q_stride, void* o, const void* kv_pool,
                                int32_t layer, int32_t n_layers, int32_t n_heads,
                                int32_t head_dim, int32_t page_tokens, const tk_slice* slices,
                                int32_t n_slices, const int32_t* block_tables, int32_t n_tokens,
                                float scale, void* stream, int32_t iters, float* avg_us) {
  TK_CHECK(slices && block_tables && n_slices > 0, TK_EINVAL, "tk_chunk_attention: arguments");
  int n_bt = 0;
  for (int i = 0; i < n_slices; ++i) n_bt = std::max(n_bt, slices[i].bt_offset + slices[i].n_pages);
  const bool tc_attn = use_tc_attention(head_dim);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<void*> dev;
  auto upload = [&](const void* src, size_t bytes) -> void* {
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    dev.push_back(d);
    if (src && bytes && cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    if (!src && cudaMemset(d, 0, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    return d;
  };
  struct Freer {
    std::vector<void*>& v;
    ~Freer() { for (void* p : v) cudaFree(p); }
  } freer{dev};
  void* d_sl = upload(slices, n_slices * sizeof(tk_slice));
  void* d_bt = upload(block_tables, std::max(1, n_bt) * 4);
  void* d_part = upload(nullptr, attn_partial_bytes(n_heads, head_dim));
  TK_CHECK(d_sl && d_bt && d_part, TK_ECUDA, "tk_chunk_attention: device staging");
  FaPlan fa{};
  void *d_pairs = nullptr, *d_units = nullptr, *d_groups = nullptr, *d_off = nullptr;
  void *d_work = nullptr, *d_qb = nullptr;
  int n_qb = 0, n_work = 0;
  bool any_split = false;
  if (tc_attn) {
    const int pcap = n_slices + n_tokens / 256 + 1;
    const int ucap = pcap * n_heads + kNumSMs + 1;
    std::vector<FaPair> pairs(pcap);
    std::vector<FaUnit> units(ucap);
    std::vector<FaGroup> groups(pcap * n_heads);
    std::vector<int32_t> off(kNumSMs + 1);
    const int span = fa_span(head_dim);
    TK_CHECK(build_fa_plan(slices, n_slices, n_heads, span > 256 ? kNumSMs / 2 : kNumSMs, &fa,
                           pairs.data(), pcap, units.data(), ucap, groups.data(), pcap * n_heads,
                           off.data(), kNumSMs + 1, span) == 0,
             TK_EINVAL, "tk_chunk_attention: attention plan overflow");
    d_pairs = upload(pairs.data(), pairs.size() * sizeof(FaPair));
    d_units = upload(units.data(), units.size() * sizeof(FaUnit));
    d_groups = upload(groups.data(), groups.size() * sizeof(FaGroup));
    d_off = upload(off.data(), off.size() * 4);
    TK_CHECK(d_pairs && d_units && d_groups && d_off, TK_ECUDA, "tk_chunk_attention: staging");
  } else {
    const int qcap = n_slices + n_tokens / 128 + 1;
    std::vector<AttnQBlock> qbs(qcap);
    std::vector<AttnWork> work(qcap + kAttnMaxSplitSlots);
    n_work = build_attn_work(slices, n_slices, n_heads, qbs.data(), qcap, work.data(),
                             static_cast<int>(work.size()), &n_qb, 64);
    TK_CHECK(n_work >= 0, TK_EINVAL, "tk_chunk_attention: work list");
    for (int k = 0; k < n_qb; ++k) any_split |= qbs[k].n_splits > 1;
    d_work = upload(work.data(), std::max(1, n_work) * sizeof(AttnWork));
    d_qb = upload(qbs.data(), std::max(1, n_qb) * sizeof(AttnQBlock));
    TK_CHECK(d_work && d_qb, TK_ECUDA, "tk_chunk_attention: staging");
  }
  KvGeom g{n_layers, n_heads, head_dim, page_tokens};
  int rc = TK_OK;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (iters > 1) {
    TK_CUDA(cudaEventCreate(&ev0));
    TK_CUDA(cudaEventCreate(&ev1));
  }
  for (int it = 0; it < std::max(1, iters) && rc == TK_OK; ++it) {
  if (iters > 1 && it == 1) TK_CUDA(cudaEventRecord(ev0, s));
  if (tc_attn) {
    // the pool extent: enough pages to cover every page id referenced
    int max_page = 0;
    for (int i = 0; i < n_bt; ++i) max_page = std::max(max_page, block_tables[i]);
    rc = launch_chunk_attention_fa(
        static_cast<const __nv_bfloat16*>(q), n_tokens, q_stride, static_cast<__nv_bfloat16*>(o),
        static_cast<const __nv_bfloat16*>(kv_pool), max_page + 1, g, layer, fa,
        static_cast<FaPair*>(d_pairs), static_cast<FaUnit*>(d_units),
        static_cast<FaGroup*>(d_groups), static_cast<int32_t*>(d_off),
        static_cast<tk_slice*>(d_sl), static_cast<int32_t*>(d_bt), scale,
        static_cast<float*>(d_part), s);
  } else {
    rc = launch_chunk_attention_work(
        static_cast<const __nv_bfloat16*>(q), q_stride, static_cast<__nv_bfloat16*>(o),
        static_cast<const __nv_bfloat16*>(kv_pool), g, layer, static_cast<AttnWork*>(d_work),
        n_work, static_cast<AttnQBlock*>(d_qb), n_qb, any_split, static_cast<tk_slice*>(d_sl),
        static_cast<int32_t*>(d_bt), scale, static_cast<float*>(d_part), s);
  }
  }
  if (iters > 1 && rc == TK_OK) {
    // launches 2..iters back to back (the first one warms up)
    TK_CUDA(cudaEventRecord(ev1, s));
    TK_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    TK_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    if (avg_us) *avg_us = ms * 1e3f / static_cast<float>(iters - 1);
  }
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  TK_CUDA(cudaStreamSynchronize(s));
  return rc;
}

int tk_chunk_attention(const void* q, int32_t q_stride, void* o, const void* kv_pool,
                       int32_t layer, int32_t n_layers, int32_t n_heads, int32_t head_dim,
                       int32_t page_tokens, const tk_slice* slices, int32_t n_slices,
                       const int32_t* block_tables, int32_t n_tokens, float scale, void* stream) {
  return chunk_attention_impl(q, q_stride, o, kv_pool, layer, n_layers, n_heads, head_dim,
                              page_tokens, slices, n_slices, block_tables, n_tokens, scale, stream,
                              1, nullptr);
}

int tk_chunk_attention_timed(const void* q, int32_t q_stride, void* o, const void* kv_pool,
                             int32_t layer, int32_t n_layers, int32_t n_heads, int32_t head_dim,
                             int32_t page_tokens, const tk_slice* slices, int32_t n_slices,
                             const int32_t* block_tables, int32_t n_tokens, float scale,
                             void* stream, int32_t iters, float* avg_us) {
  TK_CHECK(iters >= 2 && avg_us, TK_EINVAL, "tk_chunk_attention_timed: iters >= 2, avg_us");
  return chunk_attention_impl(q, q_stride, o, kv_pool, layer, n_layers, n_heads, head_dim,
                              page_tokens, slices, n_slices, block_tables, n_tokens, scale, stream,
                              iters, avg_us);
}

int tk_fa_plan(const tk_slice* slices, int32_t n_slices, int32_t n_heads, int32_t max_ctas,
               int32_t* counts, int32_t* pairs, int32_t pcap, int32_t* units, int32_t ucap,
               int32_t* cta_off, int32_t ocap, int32_t span) {
  TK_CHECK(slices && counts && pairs && units && cta_off && n_slices > 0, TK_EINVAL,
           "tk_fa_plan: arguments");
  FaPlan plan{};
  std::vector<FaPair> pr(pcap);
  std::vector<FaUnit> un(ucap);
  std::vector<FaGroup> gr(std::max(1, ucap));
  TK_CHECK(span == 256 || span == 512, TK_EINVAL, "tk_fa_plan: span 256 or 512");
  TK_CHECK(build_fa_plan(slices, n_slices, n_heads, max_ctas, &plan, pr.data(), pcap, un.data(),
                         ucap, gr.data(), ucap, cta_off, ocap, span) == 0,
           TK_EINVAL, "tk_fa_plan: capacity");
  counts[0] = plan.n_pairs;
  counts[1] = plan.n_units;
  counts[2] = plan.n_ctas;
  counts[3] = plan.n_pieces;
  counts[4] = plan.n_groups;
  for (int i = 0; i < plan.n_pairs; ++i) {
    const FaPair& q = pr[i];
    const int32_t v[6] = {q.slice, q.row0, q.pos0, q.nrows0, q.nrows1, q.nblk};
    memcpy(pairs + i * 6, v, sizeof(v));
  }
  for (int i = 0; i < plan.n_units; ++i) {
    const FaUnit& u = un[i];
    const int32_t v[5] = {u.pair, u.head, u.kb0, u.kb1, u.piece};
    memcpy(units + i * 5, v, sizeof(v));
  }
  return TK_OK;
}

int tk_debug_gemm_trace(uint64_t* host, int32_t n) {
  return gemm_debug_trace(reinterpret_cast<unsigned long long*>(host), n);
}

int tk_debug_gemm_cta_trace(uint64_t* host, int32_t n) {
  return gemm_debug_cta_trace(reinterpret_cast<unsigned long long*>(host), n);
}

int tk_debug_fa_trace(uint64_t* host, int32_t n) {
  return fa_debug_trace(reinterpret_cast<unsigned long long*>(host), n);
}

int tk_event_elapsed(tk_event* a, tk_event* b, int64_t* elapsed_ns) {
  TK_CHECK(a && b && elapsed_ns, TK_EINVAL, "tk_event_elapsed: null argument");
  float ms = 0.f;
  TK_CUDA(cudaEventElapsedTime(&ms, a->start, b->end));
  *elapsed_ns = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
  return TK_OK;
}

int tk_device_memory(int32_t device, int64_t* free_bytes, int64_t* total_bytes) {
  TK_CHECK(free_bytes && total_bytes, TK_EINVAL, "tk_device_memory: null argument");
  int nd = 0;
  TK_CUDA(cudaGetDeviceCount(&nd));
  TK_CHECK(device >= 0 && device < nd, TK_EINVAL, "tk_device_memory: no such device");
  TK_CUDA(cudaSetDevice(device));
  size_t f = 0, t = 0;
  TK_CUDA(cudaMemGetInfo(&f, &t));
  *free_bytes = static_cast<int64_t>(f);
  *total_bytes = static_cast<int64_t>(t);
  return TK_OK;
}

int tk_event_anchor(int32_t device, tk_event** out) {
  TK_CHECK(out, TK_EINVAL, "tk_event_anchor: null argument");
  int nd = 0;
  TK_CUDA(cudaGetDeviceCount(&nd));
  TK_CHECK(device >= 0 && device < nd, TK_EINVAL, "tk_event_anchor: no such device");
  TK_CUDA(cudaSetDevice(device));
  std::unique_ptr<tk_event> ev(new tk_event());
  ev->device = device;
  TK_CUDA(cudaEventCreate(&ev->start));
  TK_CUDA(cudaEventCreate(&ev->end));
  // a marker on an otherwise idle stream; the caller reads its host clock
  // right after this returns (completion -> return is a few microseconds)
  cudaStream_t st;
  TK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  TK_CUDA(cudaEventRecord(ev->start, st));
  TK_CUDA(cudaEventRecord(ev->end, st));
  TK_CUDA(cudaEventSynchronize(ev->end));
  TK_CUDA(cudaStreamDestroy(st));
  ev->finished = true;
  *out = ev.release();
  return TK_OK;
}

int tk_launch_count(int64_t* n) {
  TK_CHECK(n, TK_EINVAL, "null");
  *n = g_launches.load();
  return TK_OK;
}

int tk_last_staged_bytes(tk_instance* inst, int64_t* h2d, int64_t* d2h) {
  TK_CHECK(inst && h2d && d2h, TK_EINVAL, "null");
  *h2d = inst->last_h2d;
  *d2h = inst->last_d2h;
  return TK_OK;
}

int tk_profile_enable(tk_instance* inst, int32_t on) {
  TK_CHECK(inst, TK_EINVAL, "null instance");
  inst->prof = on != 0;
  return TK_OK;
}

int tk_profile_read(tk_instance* inst, int32_t kind, int64_t* launches, double* total_ms,
                    double* flops, double* bytes) {
  TK_CHECK(inst && launches && total_ms && flops && bytes, TK_EINVAL, "null argument");
  TK_CUDA(cudaSetDevice(inst->device));
  TK_CUDA(cudaDeviceSynchronize());
  *launches = 0;
  *total_ms = *flops = *bytes = 0;
  std::vector<tk_instance::ProfRec> keep;
  for (auto& r : inst->recs) {
    if (r.kind != kind) {
      keep.push_back(r);
      continue;
    }
    float ms = 0.f;
    TK_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    *launches += 1;
    *total_ms += ms;
    *flops += r.flops;
    *bytes += r.bytes;
    inst->ev_pool.push_back(r.a);
    inst->ev_pool.push_back(r.b);
  }
  inst->recs.swap(keep);
  return TK_OK;
}

}  // extern "C"
