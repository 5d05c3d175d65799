// kernels.cu -- the non-GEMM kernels of the chunked-prefill and decode paths.
//
//   embed_*            token (+ learned position, OPT offset 2) -> fp32 residual rows
//   layernorm/rmsnorm  fp32 residual -> bf16 GEMM operand (one CTA per row)
//   kv_write           fused QKV rows -> K/V into the request's pages (+RoPE for Llama)
//   chunk_attention    K2: chunked-prefill attention, causal within each request slice
//                      over the request's paged prefix; bf16 mma.sync tiles, online
//                      softmax in fp32, cp.async double-buffered 64-token KV blocks
//   decode_attention   K3: paged decode attention, split-KV over 256-token partitions,
//                      128-bit coalesced page loads, warp-shuffle softmax, combine pass
//   argmax             greedy token per row (first maximum, like torch.argmax)
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "tk_common.cuh"
#include "tk_kernels.h"

namespace tk {

// ------------------------------------------------------------------ embeddings
__global__ void embed_opt_kernel(const int32_t* __restrict__ ids, const TokenMeta* __restrict__ meta,
                                 const __nv_bfloat16* __restrict__ tok,
                                 const __nv_bfloat16* __restrict__ pos, float* __restrict__ out,
                                 int hidden) {
  griddep_launch();
  griddep_wait();
  const int t = blockIdx.x;
  const int id = ids[t];
  const int p = meta[t].pos + 2;  // OPTLearnedPositionalEmbedding offset
  const __nv_bfloat16* te = tok + static_cast<size_t>(id) * hidden;
  const __nv_bfloat16* pe = pos + static_cast<size_t>(p) * hidden;
  float* o = out + static_cast<size_t>(t) * hidden;
  for (int c = threadIdx.x * 8; c < hidden; c += blockDim.x * 8) {
    uint4 a = *reinterpret_cast<const uint4*>(te + c);
    uint4 b = *reinterpret_cast<const uint4*>(pe + c);
    const __nv_bfloat16* av = reinterpret_cast<const __nv_bfloat16*>(&a);
    const __nv_bfloat16* bv = reinterpret_cast<const __nv_bfloat16*>(&b);
    float4 r0, r1;
    r0.x = __bfloat162float(av[0]) + __bfloat162float(bv[0]);
    r0.y = __bfloat162float(av[1]) + __bfloat162float(bv[1]);
    r0.z = __bfloat162float(av[2]) + __bfloat162float(bv[2]);
    r0.w = __bfloat162float(av[3]) + __bfloat162float(bv[3]);
    r1.x = __bfloat162float(av[4]) + __bfloat162float(bv[4]);
    r1.y = __bfloat162float(av[5]) + __bfloat162float(bv[5]);
    r1.z = __bfloat162float(av[6]) + __bfloat162float(bv[6]);
    r1.w = __bfloat162float(av[7]) + __bfloat162float(bv[7]);
    *reinterpret_cast<float4*>(o + c) = r0;
    *reinterpret_cast<float4*>(o + c + 4) = r1;
  }
}

int launch_embed_opt(const int32_t* ids, const TokenMeta* meta, int n, const __nv_bfloat16* tok_emb,
                     const __nv_bfloat16* pos_emb, float* resid, int hidden, cudaStream_t s) {
  if (n == 0) return TK_OK;
  TK_CUDA(launch_pdl(embed_opt_kernel, dim3(n), dim3(128), 0, s, ids, meta, tok_emb, pos_emb, resid,
                     hidden));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

__global__ void embed_plain_kernel(const int32_t* __restrict__ ids,
                                   const __nv_bfloat16* __restrict__ tok, float* __restrict__ out,
                                   int hidden) {
  griddep_launch();
  griddep_wait();
  const int t = blockIdx.x;
  const __nv_bfloat16* te = tok + static_cast<size_t>(ids[t]) * hidden;
  float* o = out + static_cast<size_t>(t) * hidden;
  for (int c = threadIdx.x; c < hidden; c += blockDim.x) o[c] = __bfloat162float(te[c]);
}

int launch_embed_llama(const int32_t* ids, int n, const __nv_bfloat16* tok_emb, float* resid,
                       int hidden, cudaStream_t s) {
  if (n == 0) return TK_OK;
  TK_CUDA(launch_pdl(embed_plain_kernel, dim3(n), dim3(256), 0, s, ids, tok_emb, resid, hidden));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ------------------------------------------------------------------ norms
template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float total = 0.f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) total += red[i];
  __syncthreads();
  return total;
}

constexpr int kNormThreads = 256;
constexpr int kNormMaxPer = 8;  // float4 groups per thread: cols <= 8192

__device__ __forceinline__ float4 bf16x4_to_f4(uint2 d) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// One CTA per row; thread t owns the float4 groups t, t+256, ... (PER of them,
// compile-time so the row stays in registers).  kAdd: x += delta (bf16 output
// of the preceding O-proj / FC2 GEMM, bias included) is applied first and
// written back, so the residual stream stays fp32 while those GEMMs store bf16
// instead of read-modify-writing fp32.
template <bool kRms, bool kAdd, int PER>
__global__ void __launch_bounds__(kNormThreads)
    norm_kernel(float* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                const __nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ b,
                __nv_bfloat16* __restrict__ y, int cols, float eps) {
  __shared__ float red[kNormThreads / 32];
  griddep_launch();  // the GEMM that consumes y may start prefetching its weights
  griddep_wait();    // x / delta come from the previous kernel (PDL launch)
  const size_t row = static_cast<size_t>(blockIdx.x) * cols;
  float4 v[PER];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = (threadIdx.x + k * kNormThreads) * 4;
    v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < cols) {
      v[k] = *reinterpret_cast<const float4*>(x + row + c);
      if constexpr (kAdd) {
        const float4 d = bf16x4_to_f4(*reinterpret_cast<const uint2*>(delta + row + c));
        v[k].x += d.x; v[k].y += d.y; v[k].z += d.z; v[k].w += d.w;
      }
    }
  }
  if constexpr (kAdd) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int c = (threadIdx.x + k * kNormThreads) * 4;
      if (c < cols) *reinterpret_cast<float4*>(x + row + c) = v[k];
    }
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  float mean = 0.f;
  if (!kRms) mean = block_sum<kNormThreads>(s, red) / cols;
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = (threadIdx.x + k * kNormThreads) * 4;
    if (c < cols) {
      const float a = v[k].x - mean, bb = v[k].y - mean, cc = v[k].z - mean, dd = v[k].w - mean;
      ss += (a * a + bb * bb) + (cc * cc + dd * dd);
    }
  }
  const float rstd = rsqrtf(block_sum<kNormThreads>(ss, red) / cols + eps);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = (threadIdx.x + k * kNormThreads) * 4;
    if (c >= cols) continue;
    const float4 wv = bf16x4_to_f4(*reinterpret_cast<const uint2*>(w + c));
    float4 o = make_float4((v[k].x - mean) * rstd * wv.x, (v[k].y - mean) * rstd * wv.y,
                           (v[k].z - mean) * rstd * wv.z, (v[k].w - mean) * rstd * wv.w);
    if (!kRms) {
      const float4 bv = bf16x4_to_f4(*reinterpret_cast<const uint2*>(b + c));
      o.x += bv.x; o.y += bv.y; o.z += bv.z; o.w += bv.w;
    }
    uint2 pk;
    pk.x = pack_bf16x2(o.x, o.y);
    pk.y = pack_bf16x2(o.z, o.w);
    *reinterpret_cast<uint2*>(y + row + c) = pk;
  }
}

// One WARP per row (4 rows per 128-thread CTA), for cols = 128·PER: lane l owns
// the float4 groups l, l+32, ...  Every load of the row (x, delta, then w, b) is
// issued before the first reduction, the reductions are shuffles only (no
// __syncthreads), and a 512-row chunk is a single wave of 128 CTAs -- the kernel
// is one DRAM round trip instead of the CTA-per-row kernel's load / barrier /
// barrier / store sequence.  Same arithmetic order per element as norm_kernel.
template <bool kRms, bool kAdd, int PER>
__global__ void __launch_bounds__(128)
    norm_warp_kernel(float* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                     const __nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ b,
                     __nv_bfloat16* __restrict__ y, int rows, int cols, float eps) {
  griddep_launch();
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const size_t row = static_cast<size_t>(r) * cols;
  float4 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) v[k] = *reinterpret_cast<const float4*>(x + row + (lane + 32 * k) * 4);
  if constexpr (kAdd) {
    uint2 d[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) d[k] = *reinterpret_cast<const uint2*>(delta + row + (lane + 32 * k) * 4);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const float4 f = bf16x4_to_f4(d[k]);
      v[k].x += f.x; v[k].y += f.y; v[k].z += f.z; v[k].w += f.w;
      *reinterpret_cast<float4*>(x + row + (lane + 32 * k) * 4) = v[k];
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  float mean = 0.f;
  if (!kRms) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    mean = s / cols;
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const float a = v[k].x - mean, bb = v[k].y - mean, cc = v[k].z - mean, dd = v[k].w - mean;
    ss += (a * a + bb * bb) + (cc * cc + dd * dd);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rstd = rsqrtf(ss / cols + eps);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = (lane + 32 * k) * 4;
    const float4 wv = bf16x4_to_f4(__ldg(reinterpret_cast<const uint2*>(w + c)));
    float4 o = make_float4((v[k].x - mean) * rstd * wv.x, (v[k].y - mean) * rstd * wv.y,
                           (v[k].z - mean) * rstd * wv.z, (v[k].w - mean) * rstd * wv.w);
    if (!kRms) {
      const float4 bv = bf16x4_to_f4(__ldg(reinterpret_cast<const uint2*>(b + c)));
      o.x += bv.x; o.y += bv.y; o.z += bv.z; o.w += bv.w;
    }
    uint2 pk;
    pk.x = pack_bf16x2(o.x, o.y);
    pk.y = pack_bf16x2(o.z, o.w);
    *reinterpret_cast<uint2*>(y + row + c) = pk;
  }
}

int launch_layernorm(const float* x, const __nv_bfloat16* w, const __nv_bfloat16* b,
                     __nv_bfloat16* y, int rows, int cols, float eps, cudaStream_t s) {
  return launch_add_norm(const_cast<float*>(x), nullptr, w, b, y, rows, cols, eps, false, s);
}

int launch_rmsnorm(const float* x, const __nv_bfloat16* w, __nv_bfloat16* y, int rows, int cols,
                   float eps, cudaStream_t s) {
  return launch_add_norm(const_cast<float*>(x), nullptr, w, nullptr, y, rows, cols, eps, true, s);
}

int launch_add_norm(float* x, const __nv_bfloat16* delta, const __nv_bfloat16* w,
                    const __nv_bfloat16* b, __nv_bfloat16* y, int rows, int cols, float eps,
                    bool rms, cudaStream_t s) {
  TK_CHECK(cols % 4 == 0 && cols <= kNormThreads * kNormMaxPer * 4, TK_EINVAL,
           "norm: cols must be a multiple of 4 and <= 8192");
  if (rows == 0) return TK_OK;
  const __nv_bfloat16* bb = rms ? nullptr : b;
  // The warp-per-row kernel measured slower in situ at 512 x 5120 (13.2 vs 11.6 us
  // per launch, profiles/r02_experiments.md); kept as an experiment (TK_NORM_IMPL=warp).
  static const int impl = [] {
    const char* e = getenv("TK_NORM_IMPL");
    return e && e[0] == 'w' ? 1 : 0;
  }();
  if (impl == 1 && cols % 128 == 0 && cols <= 128 * 40) {
    using WFn = void (*)(float*, const __nv_bfloat16*, const __nv_bfloat16*,
                         const __nv_bfloat16*, __nv_bfloat16*, int, int, float);
    WFn wk = nullptr;
#define TK_WNORM_CASE(P)                                                                        \
  case P:                                                                                       \
    wk = rms ? (delta ? norm_warp_kernel<true, true, P> : norm_warp_kernel<true, false, P>)     \
             : (delta ? norm_warp_kernel<false, true, P> : norm_warp_kernel<false, false, P>);  \
    break;
    switch (cols / 128) {
      TK_WNORM_CASE(6) TK_WNORM_CASE(8) TK_WNORM_CASE(16) TK_WNORM_CASE(32) TK_WNORM_CASE(40)
      TK_WNORM_CASE(2) TK_WNORM_CASE(4)
      default: break;
    }
#undef TK_WNORM_CASE
    if (wk) {
      TK_CUDA(launch_pdl(wk, dim3((rows + 3) / 4), dim3(128), 0, s, x, delta, w, bb, y, rows,
                         cols, eps));
      note_launch();
      return TK_OK;
    }
  }
  const int per = (cols + kNormThreads * 4 - 1) / (kNormThreads * 4);
  using Fn = void (*)(float*, const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                      __nv_bfloat16*, int, float);
  Fn kern = nullptr;
#define TK_NORM_CASE(P)                                                                  \
  case P:                                                                                \
    kern = rms ? (delta ? norm_kernel<true, true, P> : norm_kernel<true, false, P>)      \
               : (delta ? norm_kernel<false, true, P> : norm_kernel<false, false, P>);   \
    break;
  switch (per) {
    TK_NORM_CASE(1) TK_NORM_CASE(2) TK_NORM_CASE(3) TK_NORM_CASE(4)
    TK_NORM_CASE(5) TK_NORM_CASE(6) TK_NORM_CASE(7) TK_NORM_CASE(8)
  }
#undef TK_NORM_CASE
  static const bool norm_pdl = !getenv("TK_NORM_PDL") || atoi(getenv("TK_NORM_PDL")) != 0;
  TK_CUDA(launch_maybe_pdl(norm_pdl, kern, dim3(rows), dim3(kNormThreads), 0, s, x, delta, w, bb,
                           y, cols, eps));
  note_launch();
  return TK_OK;
}

__global__ void gather_rows_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                                   const int32_t* __restrict__ rows, int cols,
                                   float* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  const size_t r = static_cast<size_t>(rows[blockIdx.x]) * cols;
  float* dst = out + static_cast<size_t>(blockIdx.x) * cols;
  for (int c = threadIdx.x * 4; c < cols; c += blockDim.x * 4) {
    float4 q = *reinterpret_cast<const float4*>(x + r + c);
    if (delta) {
      const uint2 d = *reinterpret_cast<const uint2*>(delta + r + c);
      const float2 d01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d.x));
      const float2 d23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d.y));
      q.x += d01.x; q.y += d01.y; q.z += d23.x; q.w += d23.y;
    }
    *reinterpret_cast<float4*>(dst + c) = q;
  }
}

int launch_gather_rows_f32(const float* x, const int32_t* rows, int n, int cols, float* out,
                           cudaStream_t s, const __nv_bfloat16* delta) {
  if (n == 0) return TK_OK;
  TK_CUDA(launch_pdl(gather_rows_kernel, dim3(n), dim3(256), 0, s, x, delta, rows, cols, out));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ------------------------------------------------------------------ KV page write
// One CTA per token; threads move 16-byte chunks of K and V (and rotate Q/K
// for Llama).  qkv row layout: [q(H*D) | k(H*D) | v(H*D)].
__global__ void kv_write_kernel(__nv_bfloat16* __restrict__ qkv, const TokenMeta* __restrict__ meta,
                                __nv_bfloat16* __restrict__ pool, KvGeom g, int layer,
                                float q_scale, int rope, float rope_theta) {
  griddep_launch();
  griddep_wait();
  const int t = blockIdx.x;
  const TokenMeta m = meta[t];
  const int HD = g.n_heads * g.head_dim;
  __nv_bfloat16* row = qkv + static_cast<size_t>(t) * 3 * HD;
  if (rope) {
    // rotate_half convention: pairs (d, d + D/2) within each head.
    const int half = g.head_dim / 2;
    for (int i = threadIdx.x; i < g.n_heads * half; i += blockDim.x) {
      const int h = i / half, d = i % half;
      const float inv = powf(rope_theta, -2.f * d / g.head_dim);
      float sn, cs;
      sincosf(m.pos * inv, &sn, &cs);
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        __nv_bfloat16* base = row + part * HD + h * g.head_dim;
        const float x0 = __bfloat162float(base[d]);
        const float x1 = __bfloat162float(base[d + half]);
        base[d] = __float2bfloat16(x0 * cs - x1 * sn);
        base[d + half] = __float2bfloat16(x1 * cs + x0 * sn);
      }
    }
    __syncthreads();
  }
  if (q_scale != 1.f) {
    for (int i = threadIdx.x; i < HD; i += blockDim.x)
      row[i] = __float2bfloat16(__bfloat162float(row[i]) * q_scale);
  }
  const int chunks = HD / 8;
  for (int i = threadIdx.x; i < 2 * chunks; i += blockDim.x) {
    const int kv = i / chunks;
    const int c = i % chunks;
    const int h = (c * 8) / g.head_dim;
    const int d = (c * 8) % g.head_dim;
    const uint4 val = *reinterpret_cast<const uint4*>(row + (1 + kv) * HD + c * 8);
    *reinterpret_cast<uint4*>(pool + g.offset(m.page, layer, kv, h, m.slot) + d) = val;
  }
}

int launch_kv_write(__nv_bfloat16* qkv, const TokenMeta* meta, int n, __nv_bfloat16* pool,
                    KvGeom g, int layer, float q_scale, int rope, float rope_theta,
                    cudaStream_t s) {
  if (n == 0) return TK_OK;
  // plain launch by default (TK_KVW_PDL=1: PDL): decode step Llama-2-7B B=256 -2.1%,
  // OPT-13B B=128 -0.6%, B=32 -0.2% (profiles/r02_experiments.md)
  static const bool kvw_pdl = getenv("TK_KVW_PDL") && atoi(getenv("TK_KVW_PDL")) != 0;
  TK_CUDA(launch_maybe_pdl(kvw_pdl, kv_write_kernel, dim3(n), dim3(256), 0, s, qkv, meta, pool, g, layer, q_scale,
                     rope, rope_theta));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ------------------------------------------------------------------ chunk attention (K2)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t sz = valid ? 16u : 0u;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One CTA = 8 warps = up to 128 query rows of one slice (16 rows per warp)
// x one head x one KV split [kb0, kb1) of 64-key blocks.  The 8 warps share
// every K/V tile, so shared-memory fill per MMA is half that of 64-row CTAs.
// A q-block whose prefix is long is split over several CTAs (split-KV); each
// writes an unnormalised partial (m, l, O) that attn_combine_kernel merges.
constexpr int kAttnRows = 128;
constexpr int kAttnBlock = 64;
constexpr int kAttnThreads = 256;

template <int D>
__global__ void __launch_bounds__(kAttnThreads)
    chunk_attn_kernel(const __nv_bfloat16* __restrict__ q, int q_stride,
                      __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ pool,
                      KvGeom g, int layer, const AttnWork* __restrict__ work,
                      const AttnQBlock* __restrict__ qblocks, const tk_slice* __restrict__ slices,
                      const int32_t* __restrict__ bt, float scale_log2,
                      float* __restrict__ partial) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  constexpr int TILE = kAttnBlock * D;
  extern __shared__ __align__(128) uint8_t sm[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(sm);  // [2][64][D]
  __nv_bfloat16* sV = sK + 2 * TILE;                           // [2][64][D]

  const AttnWork w = work[blockIdx.x];
  const AttnQBlock qb = qblocks[w.qblock];
  const int head = blockIdx.y;
  const tk_slice sl = slices[qb.slice];
  const int32_t* pages = bt + sl.bt_offset;
  const int kv_end = qb.pos0 + qb.nrows;  // keys [0, kv_end) exist for this block
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int pt = g.page_tokens;

  auto load_block = [&](int j, int buf) {
    __nv_bfloat16* dk = sK + buf * TILE;
    __nv_bfloat16* dv = sV + buf * TILE;
#pragma unroll
    for (int it = 0; it < kAttnBlock * CH / kAttnThreads; ++it) {
      const int i = tid + it * kAttnThreads;
      const int r = i / CH, c = i % CH;
      const int p = j * kAttnBlock + r;
      const bool valid = p < kv_end;
      const int page = valid ? __ldg(pages + p / pt) : 0;
      const size_t off = valid ? g.offset(page, layer, 0, head, p % pt) : 0;
      const size_t offv = valid ? g.offset(page, layer, 1, head, p % pt) : 0;
      const int sw = r * D + ((c ^ (r & 7)) * 8);
      cp_async16(dk + sw, pool + off + c * 8, valid);
      cp_async16(dv + sw, pool + offv + c * 8, valid);
    }
  };

  load_block(w.kb0, 0);
  cp_async_commit();

  uint32_t qa[D / 16][4];
  const int r_lo = warp * 16 + gq, r_hi = r_lo + 8;
  {
    const __nv_bfloat16* q_lo = q + static_cast<size_t>(qb.row0 + r_lo) * q_stride + head * D;
    const __nv_bfloat16* q_hi = q + static_cast<size_t>(qb.row0 + r_hi) * q_stride + head * D;
    const bool v_lo = r_lo < qb.nrows, v_hi = r_hi < qb.nrows;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int c = ks * 16 + tq * 2;
      qa[ks][0] = v_lo ? *reinterpret_cast<const uint32_t*>(q_lo + c) : 0u;
      qa[ks][1] = v_hi ? *reinterpret_cast<const uint32_t*>(q_hi + c) : 0u;
      qa[ks][2] = v_lo ? *reinterpret_cast<const uint32_t*>(q_lo + c + 8) : 0u;
      qa[ks][3] = v_hi ? *reinterpret_cast<const uint32_t*>(q_hi + c + 8) : 0u;
    }
  }
  const int qp_lo = qb.pos0 + r_lo, qp_hi = qb.pos0 + r_hi;
  const int warp_min_q = qb.pos0 + warp * 16;
  const int warp_max_q = qb.pos0 + min(warp * 16 + 15, qb.nrows - 1);

  float acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  for (int j = w.kb0; j < w.kb1; ++j) {
    const int buf = (j - w.kb0) & 1;
    if (j + 1 < w.kb1) load_block(j + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    const int kp0 = j * kAttnBlock;
    // whole block above this warp's diagonal: nothing to do (warp-uniform)
    if (kp0 <= warp_max_q) {
      const uint32_t kbase = smem_u32(sK + buf * TILE);
      const uint32_t vbase = smem_u32(sV + buf * TILE);
      float s[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
        for (int nt = 0; nt < 8; nt += 2) {
          const int mi = lane >> 3;
          const int row = (nt + (mi >> 1)) * 8 + (lane & 7);
          const int chunk = ks * 2 + (mi & 1);
          const uint32_t addr = kbase + (row * D + ((chunk ^ (row & 7)) * 8)) * 2;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(addr, b0, b1, b2, b3);
          mma_bf16_16816(s[nt], qa[ks], b0, b1);
          mma_bf16_16816(s[nt + 1], qa[ks], b2, b3);
        }
      }
      if (kp0 + kAttnBlock - 1 > warp_min_q) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int kp = kp0 + nt * 8 + tq * 2;
          if (kp > qp_lo) s[nt][0] = -INFINITY;
          if (kp + 1 > qp_lo) s[nt][1] = -INFINITY;
          if (kp > qp_hi) s[nt][2] = -INFINITY;
          if (kp + 1 > qp_hi) s[nt][3] = -INFINITY;
        }
      }
      float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        mx_lo = fmaxf(mx_lo, fmaxf(s[nt][0], s[nt][1]) * scale_log2);
        mx_hi = fmaxf(mx_hi, fmaxf(s[nt][2], s[nt][3]) * scale_log2);
      }
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
      const float base_lo = (mx_lo == -INFINITY) ? 0.f : mx_lo;
      const float base_hi = (mx_hi == -INFINITY) ? 0.f : mx_hi;
      const float corr_lo = exp2f(m_lo - base_lo);
      const float corr_hi = exp2f(m_hi - base_hi);
      m_lo = mx_lo;
      m_hi = mx_hi;
      float sum_lo = 0.f, sum_hi = 0.f;
      uint32_t pa[4][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = exp2f(fmaf(s[nt][0], scale_log2, -base_lo));
        const float p1 = exp2f(fmaf(s[nt][1], scale_log2, -base_lo));
        const float p2 = exp2f(fmaf(s[nt][2], scale_log2, -base_hi));
        const float p3 = exp2f(fmaf(s[nt][3], scale_log2, -base_hi));
        sum_lo += p0 + p1;
        sum_hi += p2 + p3;
        const int ks = nt >> 1;
        if ((nt & 1) == 0) {
          pa[ks][0] = pack_bf16x2(p0, p1);
          pa[ks][1] = pack_bf16x2(p2, p3);
        } else {
          pa[ks][2] = pack_bf16x2(p0, p1);
          pa[ks][3] = pack_bf16x2(p2, p3);
        }
      }
      l_lo = l_lo * corr_lo + sum_lo;
      l_hi = l_hi * corr_hi + sum_hi;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        acc[i][0] *= corr_lo;
        acc[i][1] *= corr_lo;
        acc[i][2] *= corr_hi;
        acc[i][3] *= corr_hi;
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
        for (int nt = 0; nt < D / 8; nt += 2) {
          const int mi = lane >> 3;
          const int row = ks * 16 + (mi & 1) * 8 + (lane & 7);
          const int chunk = nt + (mi >> 1);
          const uint32_t addr = vbase + (row * D + ((chunk ^ (row & 7)) * 8)) * 2;
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(addr, b0, b1, b2, b3);
          mma_bf16_16816(acc[nt], pa[ks], b0, b1);
          mma_bf16_16816(acc[nt + 1], pa[ks], b2, b3);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  const int HD = g.n_heads * D;
  if (qb.n_splits == 1) {
    const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f;
    const float inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
    if (r_lo < qb.nrows) {
      __nv_bfloat16* out = o + static_cast<size_t>(qb.row0 + r_lo) * HD + head * D;
#pragma unroll
      for (int nt = 0; nt < D / 8; ++nt)
        *reinterpret_cast<uint32_t*>(out + nt * 8 + tq * 2) =
            pack_bf16x2(acc[nt][0] * inv_lo, acc[nt][1] * inv_lo);
    }
    if (r_hi < qb.nrows) {
      __nv_bfloat16* out = o + static_cast<size_t>(qb.row0 + r_hi) * HD + head * D;
#pragma unroll
      for (int nt = 0; nt < D / 8; ++nt)
        *reinterpret_cast<uint32_t*>(out + nt * 8 + tq * 2) =
            pack_bf16x2(acc[nt][2] * inv_hi, acc[nt][3] * inv_hi);
    }
  } else {
    // partial[(slot * H + head) * 128 + row][D + 4]: O unnormalised, m, l
    float* base = partial + (static_cast<size_t>(w.slot) * g.n_heads + head) * kAttnRows * (D + 4);
    float* plo = base + static_cast<size_t>(r_lo) * (D + 4);
    float* phi = base + static_cast<size_t>(r_hi) * (D + 4);
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt) {
      *reinterpret_cast<float2*>(plo + nt * 8 + tq * 2) = make_float2(acc[nt][0], acc[nt][1]);
      *reinterpret_cast<float2*>(phi + nt * 8 + tq * 2) = make_float2(acc[nt][2], acc[nt][3]);
    }
    if (tq == 0) {
      plo[D] = m_lo;
      plo[D + 1] = l_lo;
      phi[D] = m_hi;
      phi[D + 1] = l_hi;
    }
  }
}

// Merge the split partials of every multi-split q-block: grid (qblocks, heads),
// 8 warps, one query row per warp at a time, lanes across the head dim (float4)
// so every partial row is read with coalesced 16-byte accesses.
template <int D>
__global__ void __launch_bounds__(256)
    attn_combine_kernel(__nv_bfloat16* __restrict__ o, const AttnQBlock* __restrict__ qblocks,
                        int n_heads, const float* __restrict__ partial) {
  const AttnQBlock qb = qblocks[blockIdx.x];
  if (qb.n_splits <= 1) return;
  const int head = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RS = D + 4;  // partial row stride (floats)
  const size_t stride_slot = static_cast<size_t>(n_heads) * kAttnRows * RS;
  const float* base = partial + (static_cast<size_t>(qb.first_slot) * n_heads + head) * kAttnRows * RS;
  for (int row = warp; row < qb.nrows; row += 8) {
    const float* first = base + static_cast<size_t>(row) * RS;
    float M = -INFINITY;
    for (int s = 0; s < qb.n_splits; ++s) M = fmaxf(M, first[s * stride_slot + D]);
    float L = 0.f;
    float acc[D / 32];
#pragma unroll
    for (int e = 0; e < D / 32; ++e) acc[e] = 0.f;
    for (int s = 0; s < qb.n_splits; ++s) {
      const float* ps = first + s * stride_slot;
      const float m = ps[D];
      const float w = (m == -INFINITY) ? 0.f : exp2f(m - M);
      L += ps[D + 1] * w;
      if constexpr (D == 128) {
        const float4 v = *reinterpret_cast<const float4*>(ps + lane * 4);
        acc[0] += v.x * w; acc[1] += v.y * w; acc[2] += v.z * w; acc[3] += v.w * w;
      } else {
        const float2 v = *reinterpret_cast<const float2*>(ps + lane * 2);
        acc[0] += v.x * w; acc[1] += v.y * w;
      }
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    __nv_bfloat16* out = o + static_cast<size_t>(qb.row0 + row) * n_heads * D + head * D;
    if constexpr (D == 128) {
      uint2 pk;
      pk.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
      pk.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
      *reinterpret_cast<uint2*>(out + lane * 4) = pk;
    } else {
      *reinterpret_cast<uint32_t*>(out + lane * 2) = pack_bf16x2(acc[0] * inv, acc[1] * inv);
    }
  }
}

int64_t attn_partial_bytes(int n_heads, int head_dim) {
  if (use_tc_attention(head_dim)) return fa_partial_bytes();
  return static_cast<int64_t>(kAttnMaxSplitSlots) * n_heads * kAttnRows * (head_dim + 4) * 4;
}

// Host: slices -> 128-row q-blocks -> KV splits.  Splits are made only when the
// grid would otherwise be small (target ~4 CTAs per SM including heads) and
// never below kAttnMinSplitBlocks blocks of keys per split.
int build_attn_work(const tk_slice* slices, int n_slices, int n_heads, AttnQBlock* qbs,
                    int qcap, AttnWork* items, int icap, int* n_qblocks, int block_keys) {
  const int kAttnBlock = block_keys;  // keys per KV block of the consuming kernel
  int nq = 0, row = 0;
  int64_t total_blocks = 0;
  for (int i = 0; i < n_slices; ++i) {
    for (int r = 0; r < slices[i].len; r += kAttnRows) {
      if (nq >= qcap) return -1;
      AttnQBlock& q = qbs[nq++];
      q.slice = i;
      q.row0 = row + r;
      q.nrows = min(kAttnRows, slices[i].len - r);
      q.pos0 = slices[i].start + r;
      q.n_splits = 1;
      q.first_slot = -1;
      total_blocks += (q.pos0 + q.nrows + kAttnBlock - 1) / kAttnBlock;
    }
    row += slices[i].len;
  }
  const int64_t target_ctas = 4LL * kNumSMs;
  int n_items = 0, slot = 0;
  for (int k = 0; k < nq; ++k) {
    AttnQBlock& q = qbs[k];
    const int nb = (q.pos0 + q.nrows + kAttnBlock - 1) / kAttnBlock;
    int splits = 1;
    if (static_cast<int64_t>(nq) * n_heads < target_ctas) {
      const int64_t want = (target_ctas + static_cast<int64_t>(nq) * n_heads - 1) /
                           (static_cast<int64_t>(nq) * n_heads);
      splits = static_cast<int>(std::min<int64_t>(want, nb * block_keys / (64 * kAttnMinSplitBlocks)));
      splits = std::max(1, std::min(splits, 16));
      if (slot + splits > kAttnMaxSplitSlots) splits = 1;
    }
    q.n_splits = splits;
    if (splits > 1) {
      q.first_slot = slot;
    }
    for (int s = 0; s < splits; ++s) {
      if (n_items >= icap) return -1;
      AttnWork& w = items[n_items++];
      w.qblock = k;
      w.kb0 = static_cast<int>(static_cast<int64_t>(nb) * s / splits);
      w.kb1 = static_cast<int>(static_cast<int64_t>(nb) * (s + 1) / splits);
      w.slot = splits > 1 ? slot + s : -1;
    }
    if (splits > 1) slot += splits;
  }
  (void)total_blocks;
  *n_qblocks = nq;
  return n_items;
}

int launch_chunk_attention_work(const __nv_bfloat16* q, int q_stride, __nv_bfloat16* o,
                                const __nv_bfloat16* pool, KvGeom g, int layer,
                                const AttnWork* work, int n_work, const AttnQBlock* qblocks,
                                int n_qblocks, bool any_split, const tk_slice* slices_dev,
                                const int32_t* bt_dev, float scale, float* partial,
                                cudaStream_t s) {
  TK_CHECK(g.head_dim == 128 || g.head_dim == 64, TK_EUNSUPPORTED,
           "chunk attention: head_dim must be 64 or 128");
  if (n_work == 0) return TK_OK;
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(n_work, g.n_heads);
  if (g.head_dim == 128) {
    const int smem = 4 * kAttnBlock * 128 * 2;
    TK_SMEM_OPT_IN(chunk_attn_kernel<128>, smem);
    chunk_attn_kernel<128><<<grid, kAttnThreads, smem, s>>>(q, q_stride, o, pool, g, layer, work,
                                                            qblocks, slices_dev, bt_dev,
                                                            scale_log2, partial);
    TK_CUDA(cudaGetLastError());
    note_launch();
    if (any_split) return launch_attn_combine(o, qblocks, n_qblocks, g.n_heads, 128, partial, s);
  } else {
    const int smem = 4 * kAttnBlock * 64 * 2;
    chunk_attn_kernel<64><<<grid, kAttnThreads, smem, s>>>(q, q_stride, o, pool, g, layer, work,
                                                           qblocks, slices_dev, bt_dev,
                                                           scale_log2, partial);
    TK_CUDA(cudaGetLastError());
    note_launch();
    if (any_split) return launch_attn_combine(o, qblocks, n_qblocks, g.n_heads, 64, partial, s);
  }
  return TK_OK;
}

int launch_attn_combine(__nv_bfloat16* o, const AttnQBlock* qblocks, int n_qblocks, int n_heads,
                        int head_dim, float* partial, cudaStream_t s) {
  if (head_dim == 128)
    attn_combine_kernel<128><<<dim3(n_qblocks, n_heads), 256, 0, s>>>(o, qblocks, n_heads,
                                                                      partial);
  else
    attn_combine_kernel<64><<<dim3(n_qblocks, n_heads), 256, 0, s>>>(o, qblocks, n_heads, partial);
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ------------------------------------------------------------------ paged decode attention (K3)
constexpr int kDecSplitTokens = 256;

// grid (splits, heads, batch), 128 threads; each warp walks pages of the split.
// A token's D dims are spread over D/8 lanes (16-byte loads), so one warp load
// covers 32/(D/8) tokens (2 at D=128, 4 at D=64 -- the OPT-125M tiny decoder): lane l
// owns dims [(l % LPT)*8, +8) of token group l / LPT; partial (m, l, acc) of the 4
// warps are merged in smem.
template <int D>
__global__ void __launch_bounds__(128)
    decode_attn_kernel(const __nv_bfloat16* __restrict__ q, int q_stride,
                       __nv_bfloat16* __restrict__ o,
                       const __nv_bfloat16* __restrict__ pool, KvGeom g, int layer,
                       const int32_t* __restrict__ bt, int bt_stride,
                       const int32_t* __restrict__ ctx_lens, float scale_log2,
                       float* __restrict__ ws, int max_splits, int split_tokens) {
  griddep_wait();  // q / pages from the QKV GEMM + kv_write (PDL launch)
  static_assert(D == 128 || D == 64, "decode attention: head_dim 128 or 64");
  constexpr int LPT = D / 8;      // lanes per token
  constexpr int TPL = 32 / LPT;   // tokens per warp load
  constexpr int ITER = 16 / TPL;  // loads per 16-token page
  const int split = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int ctx = ctx_lens[b];
  const int n_splits = (ctx + split_tokens - 1) / split_tokens;
  if (split >= n_splits) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane / LPT, dl = (lane % LPT) * 8;  // half: token group of the lane
  const int pt = g.page_tokens;  // 16
  const int t0 = split * split_tokens;
  const int t1 = min(ctx, t0 + split_tokens);

  float qv[8];
  {
    const uint4 raw = *reinterpret_cast<const uint4*>(
        q + static_cast<size_t>(b) * q_stride + head * D + dl);
    const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int i = 0; i < 8; ++i) qv[i] = __bfloat162float(qb[i]) * scale_log2;
  }
  float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;

  const int32_t* pages = bt + static_cast<size_t>(b) * bt_stride;
  for (int base = t0 + warp * pt; base < t1; base += 4 * pt) {
    const int page = pages[base / pt];
    const __nv_bfloat16* kp = pool + g.offset(page, layer, 0, head, 0);
    const __nv_bfloat16* vp = pool + g.offset(page, layer, 1, head, 0);
    uint4 kr[ITER], vr[ITER];
#pragma unroll
    for (int i = 0; i < ITER; ++i) {
      const int tok = TPL * i + half;
      kr[i] = __ldg(reinterpret_cast<const uint4*>(kp + tok * D + dl));
      vr[i] = __ldg(reinterpret_cast<const uint4*>(vp + tok * D + dl));
    }
    float sc[ITER];
    float pmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < ITER; ++i) {
      const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(&kr[i]);
      float d = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) d += qv[e] * __bfloat162float(kb[e]);
#pragma unroll
      for (int off = LPT / 2; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
      const int tok = base + TPL * i + half;
      sc[i] = tok < t1 ? d : -INFINITY;
      pmax = fmaxf(pmax, sc[i]);
    }
#pragma unroll
    for (int off = LPT; off < 32; off <<= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, off));
    const float mn = fmaxf(m, pmax);
    const float corr = exp2f(m - mn);
    l *= corr;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= corr;
#pragma unroll
    for (int i = 0; i < ITER; ++i) {
      // slots past the context may hold stale bytes (even NaN patterns): skip them
      if (base + TPL * i + half < t1) {
        const float p = exp2f(sc[i] - mn);
        l += p;
        const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vr[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += p * __bfloat162float(vb[e]);
      }
    }
    m = mn;
  }
  // merge the token groups of the warp (same m)
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], off);
  }

  // merge 4 warps
  __shared__ float s_m[4], s_l[4];
  __shared__ float s_acc[4][D];
  if (lane == 0) {
    s_m[warp] = m;
    s_l[warp] = l;
  }
  if (half == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) s_acc[warp][dl + e] = acc[e];
  }
  __syncthreads();
  if (warp == 0) {
    float M = fmaxf(fmaxf(s_m[0], s_m[1]), fmaxf(s_m[2], s_m[3]));
    float L = 0.f;
    float w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = (s_m[i] == -INFINITY) ? 0.f : exp2f(s_m[i] - M);
      L += s_l[i] * w[i];
    }
    for (int d = lane; d < D; d += 32) {
      const float a = s_acc[0][d] * w[0] + s_acc[1][d] * w[1] + s_acc[2][d] * w[2] +
                      s_acc[3][d] * w[3];
      if (n_splits == 1) {
        o[(static_cast<size_t>(b) * g.n_heads + head) * D + d] = __float2bfloat16(a / L);
      } else {
        float* part = ws + ((static_cast<size_t>(b) * g.n_heads + head) * max_splits + split) * (D + 2);
        part[d] = a;
        if (d == 0) {
          part[D] = M;
          part[D + 1] = L;
        }
      }
    }
  }
}

template <int D>
__global__ void decode_combine_kernel(__nv_bfloat16* __restrict__ o, int n_heads,
                                      const int32_t* __restrict__ ctx_lens,
                                      const float* __restrict__ ws, int max_splits,
                                      int split_tokens) {
  griddep_launch();
  griddep_wait();
  const int head = blockIdx.x, b = blockIdx.y;
  const int n_splits = (ctx_lens[b] + split_tokens - 1) / split_tokens;
  if (n_splits <= 1) return;
  const float* parts = ws + (static_cast<size_t>(b) * n_heads + head) * max_splits * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, parts[s * (D + 2) + D]);
  float L = 0.f;
  for (int s = 0; s < n_splits; ++s)
    L += parts[s * (D + 2) + D + 1] * exp2f(parts[s * (D + 2) + D] - M);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < n_splits; ++s) a += parts[s * (D + 2) + d] * exp2f(parts[s * (D + 2) + D] - M);
    o[(static_cast<size_t>(b) * n_heads + head) * D + d] = __float2bfloat16(a / L);
  }
}

int64_t decode_attention_workspace_bytes(int batch, int n_heads, int head_dim, int max_ctx) {
  const int splits = (max_ctx + kDecSplitTokens - 1) / kDecSplitTokens;
  return static_cast<int64_t>(batch) * n_heads * splits * (head_dim + 2) * 4;
}

int launch_decode_attention(const __nv_bfloat16* q, int q_stride, __nv_bfloat16* o,
                            const __nv_bfloat16* pool,
                            KvGeom g, int layer, const int32_t* block_tables, int bt_stride,
                            const int32_t* ctx_lens, int batch, int max_ctx, float scale,
                            void* workspace, int64_t ws_bytes, cudaStream_t s) {
  TK_CHECK(g.head_dim == 128 || g.head_dim == 64, TK_EUNSUPPORTED,
           "decode attention: head_dim must be 128 or 64");
  TK_CHECK(g.page_tokens == 16, TK_EUNSUPPORTED, "decode attention: page_tokens must be 16");
  TK_CHECK(ws_bytes >= decode_attention_workspace_bytes(batch, g.n_heads, g.head_dim, max_ctx),
           TK_EINVAL, "decode attention: workspace too small");
  if (batch == 0 || max_ctx == 0) return TK_OK;
  // Partition size: 256 tokens, doubled (up to 1024) while the grid keeps at
  // least ~4 waves of CTAs -- longer partitions amortise each CTA's setup and
  // merge, and B=128 x ctx 512 needs no combine pass at all.
  int split_tokens = kDecSplitTokens;
  while (split_tokens < 4 * kDecSplitTokens &&
         static_cast<int64_t>(batch) * g.n_heads * ((max_ctx + 2 * split_tokens - 1) / (2 * split_tokens)) >=
             4 * 5 * kNumSMs)
    split_tokens *= 2;
  const int splits = (max_ctx + split_tokens - 1) / split_tokens;
  const int ws_splits = (max_ctx + kDecSplitTokens - 1) / kDecSplitTokens;  // workspace stride
  const float scale_log2 = scale * 1.4426950408889634f;
  const bool d64 = g.head_dim == 64;
  // Launched WITHOUT programmatic dependent launch (TK_DEC_ATTN_PDL=1 restores it):
  // under PDL its grid (splits x heads x batch CTAs) becomes resident while the QKV
  // GEMM and kv_write drain and waits there; a plain launch made the decode step
  // faster at every measured shape (Llama-2-7B B=256 ctx 1024: 33.5 -> 28.3 ms, OPT-13B
  // B=32 ctx 2048: 15.9 -> 14.3 ms, B=8: 6.09 -> 5.94 ms, B=128 ctx 512: equal).
  static const bool attn_pdl = getenv("TK_DEC_ATTN_PDL") && atoi(getenv("TK_DEC_ATTN_PDL")) != 0;
  TK_CUDA(launch_maybe_pdl(attn_pdl, d64 ? decode_attn_kernel<64> : decode_attn_kernel<128>,
                     dim3(splits, g.n_heads, batch), dim3(128), 0, s, q, q_stride, o, pool, g,
                     layer, block_tables, bt_stride, ctx_lens, scale_log2,
                     static_cast<float*>(workspace), ws_splits, split_tokens));
  note_launch();
  if (splits > 1) {
    static const bool comb_pdl = !getenv("TK_DCOMB_PDL") || atoi(getenv("TK_DCOMB_PDL")) != 0;
    TK_CUDA(launch_maybe_pdl(comb_pdl, d64 ? decode_combine_kernel<64> : decode_combine_kernel<128>,
                       dim3(g.n_heads, batch), dim3(128), 0, s, o, g.n_heads, ctx_lens,
                       static_cast<const float*>(workspace), ws_splits, split_tokens));
  note_launch();
  }
  return TK_OK;
}

// ------------------------------------------------------------------ argmax
__global__ void argmax_kernel(const float* __restrict__ x, int cols, int stride,
                              int32_t* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  const float* row = x + static_cast<size_t>(blockIdx.x) * stride;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = row[c];
    if (v > best || (v == best && c < idx)) {
      best = v;
      idx = c;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sb[w] = best;
    si[w] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) {
      if (sb[i] > best || (sb[i] == best && si[i] < idx)) {
        best = sb[i];
        idx = si[i];
      }
    }
    out[blockIdx.x] = idx;
  }
}

int launch_argmax_strided(const float* logits, int rows, int cols, int stride, int32_t* out,
                          cudaStream_t s) {
  if (rows == 0) return TK_OK;
  TK_CUDA(launch_pdl(argmax_kernel, dim3(rows), dim3(1024), 0, s, logits, cols, stride, out));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ------------------------------------------------------------------ init / elementwise
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void init_normal_kernel(__nv_bfloat16* w, int64_t n, uint64_t seed, float std) {
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 2; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x * 2) {
    const uint64_t r = splitmix64(seed ^ (static_cast<uint64_t>(i) * 0xD1B54A32D192ED03ull));
    const float u1 = (static_cast<float>(r >> 40) + 1.f) * (1.f / 16777216.f);
    const float u2 = static_cast<float>((r >> 16) & 0xFFFFFF) * (1.f / 16777216.f);
    const float rad = sqrtf(-2.f * logf(u1)) * std;
    float sn, cs;
    sincospif(2.f * u2, &sn, &cs);
    w[i] = __float2bfloat16(rad * cs);
    if (i + 1 < n) w[i + 1] = __float2bfloat16(rad * sn);
  }
}

int launch_init_normal(__nv_bfloat16* w, int64_t n, uint64_t seed, float std, cudaStream_t s) {
  if (n == 0) return TK_OK;
  init_normal_kernel<<<kNumSMs * 8, 256, 0, s>>>(w, n, seed, std);
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

__global__ void fill_kernel(__nv_bfloat16* w, int64_t n, float v) {
  const __nv_bfloat16 b = __float2bfloat16(v);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] = b;
}

int launch_fill(__nv_bfloat16* w, int64_t n, float value, cudaStream_t s) {
  if (n == 0) return TK_OK;
  fill_kernel<<<kNumSMs * 4, 256, 0, s>>>(w, n, value);
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

__global__ void swiglu_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out,
                              int ffn) {
  griddep_launch();
  griddep_wait();
  const int t = blockIdx.x;
  const __nv_bfloat16* row = gu + static_cast<size_t>(t) * 2 * ffn;
  for (int c = threadIdx.x; c < ffn; c += blockDim.x) {
    const float gt = __bfloat162float(row[c]);
    const float up = __bfloat162float(row[ffn + c]);
    out[static_cast<size_t>(t) * ffn + c] = __float2bfloat16(gt / (1.f + __expf(-gt)) * up);
  }
}

int launch_swiglu(const __nv_bfloat16* gate_up, __nv_bfloat16* out, int n, int ffn,
                  cudaStream_t s) {
  if (n == 0) return TK_OK;
  TK_CUDA(launch_pdl(swiglu_kernel, dim3(n), dim3(256), 0, s, gate_up, out, ffn));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

// ---------------------------------------------------------------- KV page copy
// The P->D KV handoff (pdsim/prefill.py:420-424, bytes = pdsim/costs.py:137) as one
// launch: every (page, segment) pair is a work item, CTAs stride over the items and
// move 16-byte vectors with four loads in flight per thread.  The destination may be
// a peer device's pool (NVLink stores; peer access is enabled at instance creation).
// The page list travels in the kernel parameters, so no staging copy precedes it.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(kCopyThreads)
kv_copy_pages_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                     const __grid_constant__ PageCopyList list) {
  const int64_t pv = list.page_vec;
  const int64_t seg = (pv + list.parts - 1) / list.parts;
  const int items = list.n * list.parts;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int p = it / list.parts;
    const int64_t b = (it - p * list.parts) * seg;
    const int64_t e = b + seg < pv ? b + seg : pv;
    const uint4* s = src + static_cast<int64_t>(list.src[p]) * pv;
    uint4* d = dst + static_cast<int64_t>(list.dst[p]) * pv;
    int64_t i = b + threadIdx.x;
    for (; i + 3 * kCopyThreads < e; i += 4 * kCopyThreads) {
      const uint4 v0 = ld_stream(s + i), v1 = ld_stream(s + i + kCopyThreads);
      const uint4 v2 = ld_stream(s + i + 2 * kCopyThreads), v3 = ld_stream(s + i + 3 * kCopyThreads);
      d[i] = v0;
      d[i + kCopyThreads] = v1;
      d[i + 2 * kCopyThreads] = v2;
      d[i + 3 * kCopyThreads] = v3;
    }
    for (; i < e; i += kCopyThreads) d[i] = ld_stream(s + i);
  }
}

int launch_kv_copy_pages(const void* src_pool, void* dst_pool, int64_t page_bytes,
                         const int32_t* src_pages, const int32_t* dst_pages, int n,
                         int n_sms, cudaStream_t s) {
  TK_CHECK(page_bytes % 16 == 0, TK_EINVAL, "kv copy: page bytes not a multiple of 16");
  for (int i = 0; i < n; i += kCopyMaxPages) {
    PageCopyList list;
    list.n = n - i < kCopyMaxPages ? n - i : kCopyMaxPages;
    list.page_vec = page_bytes / 16;
    // ~256 KB per work item
    const int64_t parts = (page_bytes + (256 << 10) - 1) >> 18;
    list.parts = static_cast<int>(parts < 1 ? 1 : parts);
    for (int j = 0; j < list.n; ++j) {
      list.src[j] = src_pages[i + j];
      list.dst[j] = dst_pages[i + j];
    }
    const int items = list.n * list.parts;
    const int grid = items < n_sms * kCopyCtasPerSm ? items : n_sms * kCopyCtasPerSm;
    kv_copy_pages_kernel<<<grid, kCopyThreads, 0, s>>>(
        static_cast<const uint4*>(src_pool), static_cast<uint4*>(dst_pool), list);
    TK_CUDA(cudaGetLastError());
    note_launch();
  }
  return TK_OK;
}

}  // namespace tk
