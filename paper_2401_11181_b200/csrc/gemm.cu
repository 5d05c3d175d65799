// gemm.cu -- persistent stream-K bf16 GEMM on 5th-gen tensor cores.
//
//   C[M,N] = A[M,K] . B[N,K]^T  (+bias) (relu) (+residual)
//
// A = activations (chunk tokens or decode rows), B = nn.Linear weights
// [out, in]; both K-major, so every dense GEMM of the OPT/Llama layer is the
// canonical "TN" UMMA problem.
//
// Structure (one CTA per SM, 192 threads):
//   warp 0      TMA producer: A/B tiles -> 4..6-stage 128B-swizzled smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (128xBNx16)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused bias / ReLU /
//               residual -> global; 2 TMEM accumulators so the epilogue of
//               one tile overlaps the MMAs of the next
//
// Work split: the (tile, k-block) iteration space is divided evenly over the
// persistent CTAs (stream-K).  A tile owned by one CTA is written directly;
// a tile shared by several CTAs is reduced without atomics on the data: each
// contributor takes an arrival number from a per-tile counter; every arrival
// but the last stores its fp32 partial into the slot of its contributor rank
// (k order; thread-major, 512 contiguous bytes per warp access) and raises that
// rank's ready flag with a release store; the last arrival acquires the other
// flags, sums the partials in rank order with its own TMEM accumulator at its
// rank (so the result is bit-identical whatever the arrival order), runs the
// epilogue and re-zeroes the counter and flags.  The last arrival only ever waits on CTAs
// that already hold an arrival number (i.e. are running and past their MMAs),
// so the scheme is deadlock-free at any occupancy, including when another
// instance's kernels share the GPU.  This fixes the
// wave quantisation of M=512 chunk GEMMs (e.g. 80 tiles of 128x256 at
// N=5120 on 148 SMs) and of skinny decode GEMMs alike.
//
// Weight reuse: CTAs are launched in clusters of CS = min(tiles_m, 4) along M.
// The cluster walks one weight panel in lock step; each CTA TMA-loads 1/CS of
// every weight tile and multicasts it into all CS CTAs' shared memory, and
// every CTA's MMA commit releases the stage in all CS CTAs.  Each weight byte
// is therefore fetched from L2/HBM once per GEMM (not once per m-tile), and
// each SM pulls 16 KB of A + 32/CS KB of B per k-block.  The stream-K split
// runs over the cluster-level (m-group, n-tile, k-block) space; the number of
// clusters comes from cudaOccupancyMaxActiveClusters so all are co-resident.
#include "tk_common.cuh"
#include "tk_kernels.h"

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstdlib>

namespace tk {

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // one 128-byte swizzle row of bf16
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 192;
};

struct GemmArgs {
  void* C;
  int cs;     // cluster size along M (1, 2 or 4)
  int slots;  // partial slots per tile (max contributors - 1)
  const __nv_bfloat16* bias;
  float* ws;      // [tiles][slots][BN/32][128 threads][32] fp32 partials
  int* counters;  // [tiles] arrival counters, then [tiles][slots] ready flags
  int M, N, K;
  int epi;
  int tiles_m, tiles_n, kbs;
  long long total_iters;
  int b_pol;      // weights' L2 policy: 0 evict_first (read once), 1 evict_normal, 2 evict_last
  int pf_dist;    // k-blocks of weight L2 prefetch ahead of the TMA ring (0: none)
  int entry_pf;   // L2-prefetch the first ring fill's weights at kernel entry (TK_GEMM_ENTRY_PF)
  int pf_partials;  // TK_GEMM_PFPART: L2-prefetch a final piece's partials (measured: no gain)
  int stage_epi;  // last tile's bf16 epilogue staged in shared memory (TK_GEMM_STAGE_EPI=0: off)
  int fix_depth;  // stream-K fixup: partial chunks in flight (1, or 2 = fixup_epilogue_deep)
  int wait_mode;  // TK_GEMM_WAIT: 0 all lanes poll, 1 lane 0 polls, 2 + epilogue back-off
  int exp;        // TK_GEMM_EXP (experiments): 1 no MMAs, 2 A loads only, 3 B loads only
  int trace;      // TK_GEMM_TRACE: clock64 stamps of CTA 0's pipeline (tk_debug_gemm_trace)
  QkvScatter kv;  // EPI_QKV_PAGED only
};

// Experiment hooks (pipeline stamps, load/MMA ablations, alternative waits) exist
// only in builds with TK_GEMM_EXPERIMENTS (TK_BUILD_EXPERIMENTS=1 python -m
// paper_2401_11181_b200.build): the runtime checks alone cost the production
// kernel ~12% (measured), so they are compiled out.
#ifdef TK_GEMM_EXPERIMENTS
constexpr bool kGemmExp = true;
#else
constexpr bool kGemmExp = false;
#endif

// Pipeline stamps of CTA 0 (experiments; scripts/gemm_trace.py): kind x k-block.
//   0 issuer before full-wait, 1 after it, 2 after the k-block's MMAs + commit,
//   3 producer before empty-wait, 4 after it, 5 epilogue saw the accumulator (per tile)
constexpr int kGemmTraceN = 1024;
__device__ unsigned long long g_gemm_trace[6 * kGemmTraceN];
__device__ __forceinline__ void gemm_stamp(const GemmArgs& p, int kind, long long j) {
  if constexpr (kGemmExp) {
    if (p.trace && blockIdx.x == 0 && j < kGemmTraceN) g_gemm_trace[kind * kGemmTraceN + j] = clock64();
  }
}

// Per-CTA globaltimer stamps (ns): 0 entry, 1 issuer saw the first stage, 2 last
// MMA commit issued (leaders), 3 epilogue done, 4 exit, 5 epilogue saw the last
// accumulator, 6 last fixup's partials ready.
__device__ unsigned long long g_gemm_cta[7 * 256];
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void gemm_cta_stamp(const GemmArgs& p, int kind) {
  if constexpr (kGemmExp) {
    if (p.trace && blockIdx.x < 256) g_gemm_cta[kind * 256 + blockIdx.x] = globaltimer_ns();
  }
}

int gemm_debug_cta_trace(unsigned long long* host, int n) {
  TK_CHECK(n <= 7 * 256, TK_EINVAL, "gemm cta trace: n too large");
  TK_CUDA(cudaDeviceSynchronize());
  TK_CUDA(cudaMemcpyFromSymbol(host, g_gemm_cta, n * sizeof(unsigned long long)));
  return TK_OK;
}

int gemm_debug_trace(unsigned long long* host, int n) {
  TK_CHECK(n <= 6 * kGemmTraceN, TK_EINVAL, "gemm trace: n too large");
  TK_CUDA(cudaDeviceSynchronize());
  TK_CUDA(cudaMemcpyFromSymbol(host, g_gemm_trace, n * sizeof(unsigned long long)));
  return TK_OK;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int owner_of(long long it, long long T, int G) {
  // CTA c covers [floor(c*T/G), floor((c+1)*T/G))
  return static_cast<int>(((it + 1) * G + T - 1) / T) - 1;
}

// Bias (+ ReLU) of a 32-column chunk, for the shared-memory-staged bf16 epilogue.
template <int EPI>
__device__ __forceinline__ void epilogue_math(const GemmArgs& p, int col0, float (&v)[32]) {
  if constexpr (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_RELU) {
    if (p.bias != nullptr) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (col0 + g * 8 < p.N) {
          uint4 braw = __ldg(reinterpret_cast<const uint4*>(p.bias + col0 + g * 8));
          const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&braw);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[g * 8 + j] += __bfloat162float(b[j]);
        }
      }
    }
  }
  if constexpr (EPI == EPI_BF16_BIAS_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_store(const GemmArgs& p, int row, int col0,
                                               float (&v)[32]) {
  if (row >= p.M) return;
  if constexpr (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_RELU || EPI == EPI_F32_BIAS_RESID ||
                EPI == EPI_QKV_PAGED) {
    if (p.bias != nullptr) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (col0 + g * 8 < p.N) {
          uint4 braw = __ldg(reinterpret_cast<const uint4*>(p.bias + col0 + g * 8));
          const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&braw);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[g * 8 + j] += __bfloat162float(b[j]);
        }
      }
    }
  }
  if constexpr (EPI == EPI_BF16_BIAS_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  if constexpr (EPI == EPI_QKV_PAGED) {
    const int hd = p.kv.g.n_heads * p.kv.g.head_dim;
    if (col0 >= hd) {  // K or V: 32 columns of one head -> 64 contiguous bytes of a page slot
      const TokenMeta m = p.kv.meta[row];
      const int kv = col0 >= 2 * hd ? 1 : 0;
      const int c = col0 - (1 + kv) * hd;
      __nv_bfloat16* out = p.kv.pool +
                           p.kv.g.offset(m.page, p.kv.layer, kv, c / p.kv.g.head_dim, m.slot) +
                           c % p.kv.g.head_dim;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint4 o;
        o.x = pack_bf16x2(v[g * 8 + 0], v[g * 8 + 1]);
        o.y = pack_bf16x2(v[g * 8 + 2], v[g * 8 + 3]);
        o.z = pack_bf16x2(v[g * 8 + 4], v[g * 8 + 5]);
        o.w = pack_bf16x2(v[g * 8 + 6], v[g * 8 + 7]);
        *reinterpret_cast<uint4*>(out + g * 8) = o;
      }
      return;
    }
  }
  if constexpr (EPI == EPI_F32_BIAS_RESID || EPI == EPI_F32) {
    float* out = reinterpret_cast<float*>(p.C) + static_cast<size_t>(row) * p.N + col0;
    if constexpr (EPI == EPI_F32_BIAS_RESID) {
      float4 r[8];  // loads first: no store may sit between them
#pragma unroll
      for (int g = 0; g < 8; ++g)
        if (col0 + g * 4 < p.N) r[g] = __ldcg(reinterpret_cast<const float4*>(out + g * 4));
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        v[g * 4] += r[g].x; v[g * 4 + 1] += r[g].y; v[g * 4 + 2] += r[g].z; v[g * 4 + 3] += r[g].w;
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (col0 + g * 4 < p.N)
        *reinterpret_cast<float4*>(out + g * 4) =
            make_float4(v[g * 4], v[g * 4 + 1], v[g * 4 + 2], v[g * 4 + 3]);
    }
  } else {
    __nv_bfloat16* out =
        reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<size_t>(row) * p.N + col0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (col0 + g * 8 < p.N) {
        uint4 o;
        o.x = pack_bf16x2(v[g * 8 + 0], v[g * 8 + 1]);
        o.y = pack_bf16x2(v[g * 8 + 2], v[g * 8 + 3]);
        o.z = pack_bf16x2(v[g * 8 + 4], v[g * 8 + 5]);
        o.w = pack_bf16x2(v[g * 8 + 6], v[g * 8 + 7]);
        *reinterpret_cast<uint4*>(out + g * 8) = o;
      }
    }
  }
}

// Stream-K partial tiles: [32-col chunk c][float4 group g][epilogue thread]
// float4s, so each warp-wide store/load of one (c, g) moves 512 contiguous
// bytes (the row-per-thread TMEM layout would otherwise touch 32 lines).
__device__ __forceinline__ void partial_store(float* slot, int c, int tid, const uint32_t (&r)[32]) {
  float4* dst = reinterpret_cast<float4*>(slot) + static_cast<size_t>(c) * 8 * 128 + tid;
#pragma unroll
  for (int g = 0; g < 8; ++g)
    __stcg(dst + g * 128, make_float4(__uint_as_float(r[g * 4]), __uint_as_float(r[g * 4 + 1]),
                                      __uint_as_float(r[g * 4 + 2]), __uint_as_float(r[g * 4 + 3])));
}

// Sum of the earlier contributors' partials for chunk c.
__device__ __forceinline__ void partial_load(const float* tile_ws, size_t slot_elems, int n_slots,
                                             int c, int tid, float4 (&out)[8]) {
#pragma unroll
  for (int g = 0; g < 8; ++g) out[g] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int a = 0; a < n_slots; ++a) {
    const float4* src = reinterpret_cast<const float4*>(tile_ws + a * slot_elems) +
                        static_cast<size_t>(c) * 8 * 128 + tid;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float4 t = __ldcg(src + g * 128);
      out[g].x += t.x; out[g].y += t.y; out[g].z += t.z; out[g].w += t.w;
    }
  }
}

// Split tiles with 3+ contributors: chunk c summed in contributor (k) order, the
// finishing CTA's own accumulator at its own rank, so the result does not depend on
// which contributor arrives last (with 2, a + b == b + a already makes it exact).
__device__ __forceinline__ void ranked_sum(const float* tile_ws, size_t slot_elems, int contrib,
                                           int me, int c, int tid, const uint32_t (&own)[32],
                                           float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = 0.f;
  for (int a = 0; a < contrib; ++a) {
    if (a == me) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(own[j]);
    } else {
      const float4* src = reinterpret_cast<const float4*>(tile_ws + a * slot_elems) +
                          static_cast<size_t>(c) * 8 * 128 + tid;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 t = __ldcg(src + g * 128);
        v[g * 4] += t.x; v[g * 4 + 1] += t.y; v[g * 4 + 2] += t.z; v[g * 4 + 3] += t.w;
      }
    }
  }
}

// Last arriver of a split tile: TMEM accumulator + partials -> epilogue, the
// partial loads of chunk c+1 in flight while chunk c is finished.
template <int EPI, int NCHUNK>
__device__ __forceinline__ void fixup_epilogue(const GemmArgs& p, uint32_t t_row, int row,
                                               int col_base, const float* tile_ws,
                                               size_t slot_elems, int n_slots, int tid) {
  float4 cur[8];
  partial_load(tile_ws, slot_elems, n_slots, 0, tid, cur);
#pragma unroll 1
  for (int c = 0; c < NCHUNK; ++c) {
    float4 nxt[8];
    if (c + 1 < NCHUNK) partial_load(tile_ws, slot_elems, n_slots, c + 1, tid, nxt);
    uint32_t r[32];
    tmem_ld_32x32b_x32(t_row + c * 32, r);
    tmem_wait_ld();
    float v[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      v[g * 4] = __uint_as_float(r[g * 4]) + cur[g].x;
      v[g * 4 + 1] = __uint_as_float(r[g * 4 + 1]) + cur[g].y;
      v[g * 4 + 2] = __uint_as_float(r[g * 4 + 2]) + cur[g].z;
      v[g * 4 + 3] = __uint_as_float(r[g * 4 + 3]) + cur[g].w;
    }
    epilogue_store<EPI>(p, row, col_base + c * 32, v);
    if (c + 1 < NCHUNK) {
#pragma unroll
      for (int g = 0; g < 8; ++g) cur[g] = nxt[g];
    }
  }
}

// Same, with the partial loads of chunks c+1 and c+2 in flight while chunk c is
// finished (the fixup at the end of a stream-K range is load-latency bound).
template <int EPI, int NCHUNK>
__device__ __forceinline__ void fixup_epilogue_deep(const GemmArgs& p, uint32_t t_row, int row,
                                                    int col_base, const float* tile_ws,
                                                    size_t slot_elems, int n_slots, int tid) {
  float4 buf[3][8];
  partial_load(tile_ws, slot_elems, n_slots, 0, tid, buf[0]);
  if (NCHUNK > 1) partial_load(tile_ws, slot_elems, n_slots, 1, tid, buf[1]);
#pragma unroll
  for (int c = 0; c < NCHUNK; ++c) {
    if (c + 2 < NCHUNK) partial_load(tile_ws, slot_elems, n_slots, c + 2, tid, buf[(c + 2) % 3]);
    uint32_t r[32];
    tmem_ld_32x32b_x32(t_row + c * 32, r);
    tmem_wait_ld();
    float v[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float4 q = buf[c % 3][g];
      v[g * 4] = __uint_as_float(r[g * 4]) + q.x;
      v[g * 4 + 1] = __uint_as_float(r[g * 4 + 1]) + q.y;
      v[g * 4 + 2] = __uint_as_float(r[g * 4 + 2]) + q.z;
      v[g * 4 + 3] = __uint_as_float(r[g * 4 + 3]) + q.w;
    }
    epilogue_store<EPI>(p, row, col_base + c * 32, v);
  }
}

template <int BN, int EPI, int CS>
__global__ void __launch_bounds__(GemmCfg<BN>::THREADS, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const GemmArgs p) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);  // released by the MMA commit of every CTA of the cluster
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  if constexpr (CS > 1) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // cluster-level stream-K partition over (m-group, n-tile, k-block)
  const int rank = CS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int cluster = blockIdx.x / CS;
  const int G = gridDim.x / CS;
  const int groups_m = p.tiles_m / CS;
  const long long T = p.total_iters;
  const long long it_begin = static_cast<long long>(cluster) * T / G;
  const long long it_end = static_cast<long long>(cluster + 1) * T / G;
  const int kbs = p.kbs;
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CS) - 1);
  constexpr int B_SLICE_ROWS = BN / CS;
  constexpr int B_SLICE_BYTES = B_SLICE_ROWS * Cfg::BK * 2;

  // programmatic dependent launch: everything but the producer's first weight
  // tiles waits for the previous kernel on the stream
  griddep_launch();
  if (warp != 0) griddep_wait();
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_a = l2_policy_evict_last();   // activations: reused by every n-tile
      const uint64_t pol_b = l2_policy_evict_first();  // weights: streamed once per GEMM
      auto load_a = [&](int ctile, int kb, int stage) {
        const int m_idx = (ctile % groups_m) * CS + rank;
        tma_load_2d(sa + stage * Cfg::A_BYTES, &tmap_a, &full[stage], kb * Cfg::BK,
                    m_idx * Cfg::BM, pol_a);
      };
      auto load_b = [&](int ctile, int kb, int stage) {
        const int n_idx = ctile / groups_m;
        if constexpr (CS == 1) {
          tma_load_2d(sb + stage * Cfg::B_BYTES, &tmap_b, &full[stage], kb * Cfg::BK, n_idx * BN,
                      pol_b);
        } else {
          tma_load_2d_mc(sb + stage * Cfg::B_BYTES + rank * B_SLICE_BYTES, &tmap_b, &full[stage],
                         kb * Cfg::BK, n_idx * BN + rank * B_SLICE_ROWS, kMask, pol_b);
        }
      };
      // Weight tiles of the first stages do not depend on the previous kernel:
      // issue them before the programmatic-launch dependency wait.
      const int pre = static_cast<int>(it_end - it_begin < Cfg::STAGES ? it_end - it_begin : Cfg::STAGES);
      const int tile0 = static_cast<int>(it_begin / kbs), kb0 = static_cast<int>(it_begin % kbs);
      int ctile = tile0, kb = kb0;
      for (int st = 0; st < pre; ++st) {
        mbar_expect_tx(&full[st], Cfg::STAGE_BYTES);
        load_b(ctile, kb, st);
        if (++kb == kbs) { kb = 0; ++ctile; }
      }
      griddep_wait();
      ctile = tile0;
      kb = kb0;
      for (int st = 0; st < pre; ++st) {
        load_a(ctile, kb, st);
        if (++kb == kbs) { kb = 0; ++ctile; }
      }
      int stage = pre % Cfg::STAGES;
      uint32_t phase = pre == Cfg::STAGES ? 1u : 0u;
      for (long long i = it_begin + pre; i < it_end; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
        load_a(ctile, kb, stage);
        load_b(ctile, kb, stage);
        if (++kb == kbs) { kb = 0; ++ctile; }
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else {
      griddep_wait();
    }
  } else if (warp == 1) {
    {
      // ------------------------------------------------ MMA issuer (converged
      // warp, one elected lane issues: operands stay in uniform registers)
      constexpr uint32_t idesc = umma_idesc_bf16(Cfg::BM, BN);
      const uint32_t sa_base = smem_u32(sa), sb_base = smem_u32(sb);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (long long i = it_begin; i < it_end;) {
        const int ctile = static_cast<int>(i / kbs);
        const long long seg_end = min(it_end, static_cast<long long>(ctile + 1) * kbs);
        const int nkb = static_cast<int>(seg_end - i);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int k = 0; k < nkb; ++k) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = umma_desc_sw128(sa_base + stage * Cfg::A_BYTES);
          const uint64_t b_desc = umma_desc_sw128(sb_base + stage * Cfg::B_BYTES);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < Cfg::BK / 16; ++kk)
              umma_bf16(d_tmem, a_desc + 2 * kk, b_desc + 2 * kk, idesc, (k > 0 || kk > 0) ? 1u : 0u);
            if constexpr (CS == 1) umma_commit(&empty[stage]);
            else umma_commit_mc(&empty[stage], kMask);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(&tfull[acc]);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        i = seg_end;
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = static_cast<int>(quarter * 32 + lane);
    const bool leader = (warp == 2 && lane == 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (long long i = it_begin; i < it_end;) {
      const int ctile = static_cast<int>(i / kbs);
      const long long tile_first = static_cast<long long>(ctile) * kbs;
      const long long seg_end = min(it_end, tile_first + kbs);
      const int m_idx = (ctile % groups_m) * CS + rank;
      const int n_idx = ctile / groups_m;
      const int tile = n_idx * p.tiles_m + m_idx;
      const int row = m_idx * Cfg::BM + row_in_tile;
      const int col_base = n_idx * BN;
      const int contrib = owner_of(tile_first + kbs - 1, T, G) - owner_of(tile_first, T, G) + 1;

      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((quarter * 32) << 16) + acc * BN;

      if (contrib == 1) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + c * 32, r);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          epilogue_store<EPI>(p, row, col_base + c * 32, v);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        // Stream-K fixup without atomics: arrival order decides who finalises.
        // Earlier arrivals store their partial tile (coalesced, thread-major)
        // into their own slot and raise a flag; the last arrival waits for the
        // flags, adds the partials to its TMEM accumulator and runs the epilogue.
        int* counter = p.counters + tile;
        int* flags = p.counters + p.tiles_m * p.tiles_n + static_cast<size_t>(tile) * p.slots;
        if (leader) *last_flag = atomicAdd(counter, 1);
        named_bar_sync(1, 128);
        const int arrival = *last_flag;
        const size_t slot_elems = static_cast<size_t>(BN / 32) * 128 * 32;
        float* tile_ws = p.ws + static_cast<size_t>(tile) * p.slots * slot_elems;
        const int tid_e = static_cast<int>(threadIdx.x) - 64;  // 0..127, epilogue thread index
        // slots are indexed by contributor rank (k order), not arrival
        const int me = cluster - owner_of(tile_first, T, G);
        if (arrival < contrib - 1) {
          float* mine = tile_ws + static_cast<size_t>(me) * slot_elems;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_row + c * 32, r);
            tmem_wait_ld();
            partial_store(mine, c, tid_e, r);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          __threadfence();
          named_bar_sync(1, 128);
          if (leader) st_release(flags + me, 1);
        } else {
          if (leader) {
            for (int a = 0; a < contrib; ++a)
              while (a != me && ld_acquire(flags + a) == 0) {
              }
          }
          named_bar_sync(1, 128);
          __threadfence();
          if (contrib == 2) {
            fixup_epilogue<EPI, BN / 32>(p, t_row, row, col_base,
                                         tile_ws + static_cast<size_t>(1 - me) * slot_elems,
                                         slot_elems, 1, tid_e);
          } else {
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(t_row + c * 32, r);
              tmem_wait_ld();
              float v[32];
              ranked_sum(tile_ws, slot_elems, contrib, me, c, tid_e, r, v);
              epilogue_store<EPI>(p, row, col_base + c * 32, v);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          named_bar_sync(1, 128);
          if (leader) {
            for (int a = 0; a < contrib; ++a) flags[a] = 0;
            *counter = 0;
          }
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      i = seg_end;
    }
  }

  tc_fence_before();
  // no CTA may leave while a peer can still multicast into it / arrive on it
  if constexpr (CS > 1) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}


// ============================================================================
// Skinny GEMM for decode-sized M (<= 128 rows): swap A/B so the weight tile is
// the 128-row UMMA operand and the batch is the UMMA N (NB = 16..128).
//   D^T[n, m] = W[n, :] . X[m, :]      (TMEM: 128 lanes = output features,
//                                        NB columns = batch rows)
// The kernel is weight-streaming (HBM) bound: 8..12 TMA stages of 16 KB weight
// tiles per SM keep ~150 KB in flight per SM; stream-K over (n-tile, k-block)
// keeps every SM streaming; partial tiles are only 128 x NB fp32.
template <int NB>
struct SkinnyCfg {
  static constexpr int BM = 128;  // weight rows per tile
  static constexpr int BK = 64;
  static constexpr int W_BYTES = BM * BK * 2;
  static constexpr int X_BYTES = NB * BK * 2;
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 12 ? 12 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * NB < 32) ? 32 : 2 * NB;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 1024;
  static constexpr int THREADS = 192;
};

template <int NB, int EPI>
__device__ __forceinline__ void skinny_store(const GemmArgs& p, int n, int m0, const float* v,
                                             int count) {
  // v[j] = D[n, m0 + j]: output feature n of batch row m0 + j
  if (n >= p.N) return;
  float b = 0.f;
  if constexpr (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_RELU || EPI == EPI_F32_BIAS_RESID ||
                EPI == EPI_QKV_PAGED) {
    if (p.bias != nullptr) b = __bfloat162float(p.bias[n]);
  }
  const int rows = min(count, p.M - m0);
  if constexpr (EPI == EPI_QKV_PAGED) {
    // decode QKV: K and V features go straight into the batch rows' KV page slots
    // (the lanes of a warp hold consecutive features: 64 contiguous bytes per row),
    // Q features to C -- no separate kv_write pass
    const int hd = p.kv.g.n_heads * p.kv.g.head_dim;
    if (n >= hd) {
      const int kv = n >= 2 * hd ? 1 : 0;
      const int c = n - (1 + kv) * hd;
      const int head = c / p.kv.g.head_dim, d = c % p.kv.g.head_dim;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j >= rows) break;
        const TokenMeta m = p.kv.meta[m0 + j];
        p.kv.pool[p.kv.g.offset(m.page, p.kv.layer, kv, head, m.slot) + d] =
            __float2bfloat16(v[j] + b);
      }
      return;
    }
  }
  if constexpr (EPI == EPI_F32_BIAS_RESID) {
    // all residual loads first (independent), then the stores
    float* c = reinterpret_cast<float*>(p.C) + static_cast<size_t>(m0) * p.N + n;
    float r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < rows) r[j] = __ldcg(c + static_cast<size_t>(j) * p.N);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < rows) c[static_cast<size_t>(j) * p.N] = r[j] + v[j] + b;
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= rows) break;
      float x = v[j] + b;
      if constexpr (EPI == EPI_BF16_BIAS_RELU) x = fmaxf(x, 0.f);
      const size_t off = static_cast<size_t>(m0 + j) * p.N + n;
      if constexpr (EPI == EPI_F32) reinterpret_cast<float*>(p.C)[off] = x;
      else reinterpret_cast<__nv_bfloat16*>(p.C)[off] = __float2bfloat16(x);
    }
  }
}

template <int NB, int EPI>
__global__ void __launch_bounds__(SkinnyCfg<NB>::THREADS, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmap_w,
                       const __grid_constant__ CUtensorMap tmap_x, const GemmArgs p) {
  using Cfg = SkinnyCfg<NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sw = smem;
  uint8_t* sx = smem + Cfg::STAGES * Cfg::W_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.total_iters;
  const int G = gridDim.x;
  const long long it_begin = static_cast<long long>(blockIdx.x) * T / G;
  const long long it_end = static_cast<long long>(blockIdx.x + 1) * T / G;
  const int kbs = p.kbs;

  // programmatic dependent launch: everything but the producer's first weight
  // tiles waits for the previous kernel on the stream
  griddep_launch();
  if (warp != 0) griddep_wait();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();
      const uint64_t pol_x = l2_policy_evict_last();
      auto load_w = [&](int tile, int kb, int stage) {
        tma_load_2d(sw + stage * Cfg::W_BYTES, &tmap_w, &full[stage], kb * Cfg::BK,
                    tile * Cfg::BM, pol_w);
      };
      auto load_x = [&](int tile, int kb, int stage) {
        (void)tile;
        tma_load_2d(sx + stage * Cfg::X_BYTES, &tmap_x, &full[stage], kb * Cfg::BK, 0, pol_x);
      };
      // the weight stream starts before the dependency wait (decode: the
      // previous kernel's tail overlaps this kernel's first weight tiles)
      const int pre = static_cast<int>(it_end - it_begin < Cfg::STAGES ? it_end - it_begin : Cfg::STAGES);
      const int tile0 = static_cast<int>(it_begin / kbs), kb0 = static_cast<int>(it_begin % kbs);
      int tile = tile0, kb = kb0;
      for (int st = 0; st < pre; ++st) {
        mbar_expect_tx(&full[st], Cfg::STAGE_BYTES);
        load_w(tile, kb, st);
        if (++kb == kbs) { kb = 0; ++tile; }
      }
      griddep_wait();
      tile = tile0;
      kb = kb0;
      for (int st = 0; st < pre; ++st) {
        load_x(tile, kb, st);
        if (++kb == kbs) { kb = 0; ++tile; }
      }
      int stage = pre % Cfg::STAGES;
      uint32_t phase = pre == Cfg::STAGES ? 1u : 0u;
      for (long long i = it_begin + pre; i < it_end; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
        load_w(tile, kb, stage);
        load_x(tile, kb, stage);
        if (++kb == kbs) { kb = 0; ++tile; }
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else {
      griddep_wait();
    }
  } else if (warp == 1) {
    {  // converged warp, one elected lane issues
      constexpr uint32_t idesc = umma_idesc_bf16(Cfg::BM, NB);
      const uint32_t sw_base = smem_u32(sw), sx_base = smem_u32(sx);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (long long i = it_begin; i < it_end;) {
        const int tile = static_cast<int>(i / kbs);
        const long long seg_end = min(it_end, static_cast<long long>(tile + 1) * kbs);
        const int nkb = static_cast<int>(seg_end - i);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * NB;
        for (int k = 0; k < nkb; ++k) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t w_desc = umma_desc_sw128(sw_base + stage * Cfg::W_BYTES);
          const uint64_t x_desc = umma_desc_sw128(sx_base + stage * Cfg::X_BYTES);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < Cfg::BK / 16; ++kk)
              umma_bf16(d_tmem, w_desc + 2 * kk, x_desc + 2 * kk, idesc, (k > 0 || kk > 0) ? 1u : 0u);
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(&tfull[acc]);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        i = seg_end;
      }
    }
  } else {
    const uint32_t quarter = warp & 3;
    const int feat_in_tile = static_cast<int>(quarter * 32 + lane);
    const bool leader = (warp == 2 && lane == 0);
    const int tid_e = static_cast<int>(threadIdx.x) - 64;
    constexpr int CH = NB >= 32 ? 32 : NB;  // columns per TMEM load
    int acc = 0;
    uint32_t acc_phase = 0;
    for (long long i = it_begin; i < it_end;) {
      const int tile = static_cast<int>(i / kbs);
      const long long tile_first = static_cast<long long>(tile) * kbs;
      const long long seg_end = min(it_end, tile_first + kbs);
      const int n = tile * Cfg::BM + feat_in_tile;
      const int contrib = owner_of(tile_first + kbs - 1, T, G) - owner_of(tile_first, T, G) + 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((quarter * 32) << 16) + acc * NB;
      if (contrib == 1) {
#pragma unroll 1
        for (int c = 0; c < NB / CH; ++c) {
          uint32_t r[32];
          if constexpr (CH == 32) tmem_ld_32x32b_x32(t_row + c * CH, *reinterpret_cast<uint32_t(*)[32]>(r));
          else tmem_ld_32x32b_x16(t_row + c * CH, r);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int j = 0; j < CH; ++j) v[j] = __uint_as_float(r[j]);
          skinny_store<NB, EPI>(p, n, c * CH, v, CH);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        int* counter = p.counters + tile;
        int* flags = p.counters + p.tiles_n + static_cast<size_t>(tile) * p.slots;
        if (leader) *last_flag = atomicAdd(counter, 1);
        named_bar_sync(1, 128);
        const int arrival = *last_flag;
        const size_t slot_elems = static_cast<size_t>(NB) * 128;
        float* tile_ws = p.ws + static_cast<size_t>(tile) * p.slots * slot_elems;
        // slots indexed by contributor rank (k order): the finishing CTA sums in that
        // order with its own accumulator at its rank -- arrival order cannot change
        // the rounding
        const int me = static_cast<int>(blockIdx.x) - owner_of(tile_first, T, G);
        if (arrival < contrib - 1) {
          float* mine = tile_ws + static_cast<size_t>(me) * slot_elems;
#pragma unroll 1
          for (int c = 0; c < NB / CH; ++c) {
            uint32_t r[32];
            if constexpr (CH == 32) tmem_ld_32x32b_x32(t_row + c * CH, *reinterpret_cast<uint32_t(*)[32]>(r));
            else tmem_ld_32x32b_x16(t_row + c * CH, r);
            tmem_wait_ld();
            float4* dst = reinterpret_cast<float4*>(mine + (static_cast<size_t>(c) * 128 + tid_e) * CH);
#pragma unroll
            for (int g = 0; g < CH / 4; ++g)
              __stcg(dst + g, make_float4(__uint_as_float(r[g * 4]), __uint_as_float(r[g * 4 + 1]),
                                          __uint_as_float(r[g * 4 + 2]), __uint_as_float(r[g * 4 + 3])));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          __threadfence();
          named_bar_sync(1, 128);
          if (leader) st_release(flags + me, 1);
        } else {
          if (leader) {
            for (int a = 0; a < contrib; ++a)
              while (a != me && ld_acquire(flags + a) == 0) {
              }
          }
          named_bar_sync(1, 128);
          __threadfence();
#pragma unroll 1
          for (int c = 0; c < NB / CH; ++c) {
            uint32_t r[32];
            if constexpr (CH == 32) tmem_ld_32x32b_x32(t_row + c * CH, *reinterpret_cast<uint32_t(*)[32]>(r));
            else tmem_ld_32x32b_x16(t_row + c * CH, r);
            tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < CH; ++j) v[j] = 0.f;
            for (int a = 0; a < contrib; ++a) {
              if (a == me) {
#pragma unroll
                for (int j = 0; j < CH; ++j) v[j] += __uint_as_float(r[j]);
                continue;
              }
              const float4* src = reinterpret_cast<const float4*>(
                  tile_ws + static_cast<size_t>(a) * slot_elems + (static_cast<size_t>(c) * 128 + tid_e) * CH);
#pragma unroll
              for (int g = 0; g < CH / 4; ++g) {
                const float4 t = __ldcg(src + g);
                v[g * 4] += t.x; v[g * 4 + 1] += t.y; v[g * 4 + 2] += t.z; v[g * 4 + 3] += t.w;
              }
            }
            skinny_store<NB, EPI>(p, n, c * CH, v, CH);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          named_bar_sync(1, 128);
          if (leader) {
            for (int a = 0; a < contrib; ++a) flags[a] = 0;
            *counter = 0;
          }
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      i = seg_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}


// ============================================================================
// CTA-pair GEMM (tcgen05.mma.cta_group::2): a pair of CTAs on one TPC computes
// a 256 x 256 tile; each CTA holds 128 rows of A and 128 rows (half) of the
// B tile, the leader (even) CTA issues UMMA M=256 N=256 that reads both CTAs'
// shared memory and accumulates into both CTAs' TMEM (128 lanes x 256 cols
// each).  Per SM and k-block this moves 32 KB into shared memory for the
// same MMA work the 1-CTA kernel needs 48 KB for, which removes its
// shared-memory-bandwidth ceiling.  With CS = 4 two pairs (two 256-row
// m-groups) form a cluster and every B half is loaded as two 64-row slices
// multicast to the CTAs of both pairs that hold that half, so weights are
// still fetched once per GEMM.
//
// BN (tile width) is 256 (stream-K), or 160 for a one-wave data-parallel
// schedule: O-proj at M=512 as 32 clusters of 512x160 (no split tile); 256-
// wide tiles would leave SMs idle or need a split-K exchange per tile.
// KS = 64-wide k-blocks per ring stage (one barrier round trip per KS blocks).
template <int BN, int KS = 1>
struct PairCfg {
  static constexpr int A_BYTES = 128 * 64 * 2 * KS;
  static constexpr int BH_BYTES = (BN / 2) * 64 * 2 * KS;
  static constexpr int STAGE_BYTES = A_BYTES + BH_BYTES;
  static constexpr int STAGES = (232448 - 2048) / STAGE_BYTES > 8 ? 8 : (232448 - 2048) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256 + 1024;
};

template <int EPI, int CS, int BN, int KS>
__global__ void __launch_bounds__(192, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b, const GemmArgs p) {
  constexpr int BM = 128, BK = 64;
  // BN % 32 != 0 (144): data-parallel one-tile-per-CTA schedules with a staged bf16
  // epilogue only (the host guarantees it); the last 32-column chunk is half used
  // CS = 2: one pair; CS = 4: two pairs along M (all 512 rows) sharing every B half;
  // CS = 8: 2 x 2 pairs -- two along M share B halves, two along N share A tiles, so
  // every A and B byte of the cluster's 512 x 2BN block is fetched from L2 once.
  constexpr int NMP = CS == 8 ? 2 : CS / 2;  // pairs along M (share each B half)
  constexpr int NNP = CS == 8 ? 2 : 1;       // pairs along N (share each A tile)
  constexpr int MT = 2 * NMP;                // 128-row m-tiles per cluster
  static_assert(BN % 16 == 0 && BN <= 256 && (BN / 2 / NMP) % 8 == 0, "pair tile width");
  constexpr int NCH = (BN + 31) / 32;
  constexpr int STAGES = PairCfg<BN, KS>::STAGES;
  constexpr int A_BOX = BM * BK * 2;          // own 128 rows of one 64-wide k-block
  constexpr int BH_BOX = (BN / 2) * BK * 2;   // own half of the B tile, one k-block
  constexpr int A_BYTES = KS * A_BOX;         // per stage (KS k-blocks)
  constexpr int BH_BYTES = KS * BH_BOX;
  constexpr int STAGE_BYTES = A_BYTES + BH_BYTES;
  constexpr int PAIR_STAGE_BYTES = 2 * STAGE_BYTES;
  constexpr int NPAIRS = CS / 2;
  constexpr int SLICE_ROWS = (BN / 2) / NMP;        // B-half rows each CTA loads
  constexpr int SLICE_BYTES = SLICE_ROWS * BK * 2;  // per k-block box
  constexpr int A_SLICE_ROWS = BM / NNP;            // A rows each CTA loads
  constexpr int A_SLICE_BYTES = A_SLICE_ROWS * BK * 2;
  constexpr int TMEM_COLS = 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  uint64_t* fix_bar = reinterpret_cast<uint64_t*>(last_flag + 1);  // final fixup's bulk load

  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) gemm_cta_stamp(p, 0);
  const int rank = static_cast<int>(cluster_ctarank());
  const int pair = rank >> 1;
  const int half = rank & 1;
  const bool leader = half == 0;
  const int mp = pair % NMP, np = pair / NMP;  // position of the pair in the cluster
  const int m_local = mp * 2 + half;           // this CTA's 128-row m-tile in the cluster
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if (p.entry_pf) {
      // The first ring fill's weight tiles come from DRAM: start pulling them into L2
      // now, while the barriers, TMEM and the cluster are being set up.
      const int cl = blockIdx.x / CS, g = gridDim.x / CS, gm = p.tiles_m / MT;
      const long long b0 = static_cast<long long>(cl) * p.total_iters / g;
      const long long b1 = static_cast<long long>(cl + 1) * p.total_iters / g;
      int ct = static_cast<int>(b0 / p.kbs), kq = static_cast<int>(b0 % p.kbs);
      for (long long i = b0; i < b1 && i < b0 + STAGES; ++i) {
        const int row = (ct / gm) * NNP * BN + np * BN + half * (BN / 2) + mp * SLICE_ROWS;
#pragma unroll
        for (int s = 0; s < KS; ++s) tma_prefetch_2d(&tmap_b, (kq * KS + s) * BK, row);
        if (++kq == p.kbs) { kq = 0; ++ct; }
      }
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);        // leader: its expect_tx arrive (+ all TMA bytes of the pair)
      mbar_init(&empty[s], NPAIRS);  // one MMA-commit arrive per pair reading this stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // leader: 4 epilogue warps x 2 CTAs
    }
    mbar_init(fix_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int cluster = blockIdx.x / CS;
  const int G = gridDim.x / CS;
  const int groups_m = p.tiles_m / MT;  // cluster m-groups of MT 128-row m-tiles
  const long long T = p.total_iters;
  const long long it_begin = static_cast<long long>(cluster) * T / G;
  const long long it_end = static_cast<long long>(cluster + 1) * T / G;
  const int kbs = p.kbs;
  const uint16_t all_mask = static_cast<uint16_t>((1u << CS) - 1);
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pair));
  // CTAs holding this CTA's B half (same n-pair and half, every m-pair), and its A
  // tile (same m-pair and half, every n-pair)
  uint16_t half_mask = 0, a_mask = 0;
#pragma unroll
  for (int q = 0; q < NMP; ++q) half_mask |= static_cast<uint16_t>(1u << ((np * NMP + q) * 2 + half));
#pragma unroll
  for (int q = 0; q < NNP; ++q) a_mask |= static_cast<uint16_t>(1u << ((q * NMP + mp) * 2 + half));

  // programmatic dependent launch: everything but the producer's first weight
  // tiles waits for the previous kernel on the stream
  griddep_launch();
  if (warp != 0) griddep_wait();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = l2_policy_evict_last();
      const uint64_t pol_b = p.b_pol == 0   ? l2_policy_evict_first()
                             : p.b_pol == 1 ? l2_policy_evict_normal()
                                            : l2_policy_evict_last();
      const int xbytes = !kGemmExp ? PAIR_STAGE_BYTES
                         : p.exp == 2 ? 2 * A_BYTES
                         : p.exp == 3 ? PAIR_STAGE_BYTES - 2 * A_BYTES
                                      : PAIR_STAGE_BYTES;
      // tile coordinates: A row of this CTA's 128-row m-tile, B row of its slice
      auto a_row_of = [&](int ctile) {
        return ((ctile % groups_m) * MT + m_local) * BM + np * A_SLICE_ROWS;
      };
      auto b_row_of = [&](int ctile) {
        return (ctile / groups_m) * NNP * BN + np * BN + half * (BN / 2) + mp * SLICE_ROWS;
      };
      auto load_a_at = [&](int arow, int kb, int stage) {
        if (kGemmExp && p.exp == 3) return;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          if constexpr (NNP == 1)
            tma_load_2d_pair(sa + stage * A_BYTES + s * A_BOX, &tmap_a, &full[stage],
                             (kb * KS + s) * BK, arow, pol_a);
          else
            tma_load_2d_pair_mc(sa + stage * A_BYTES + s * A_BOX + np * A_SLICE_BYTES, &tmap_a,
                                &full[stage], (kb * KS + s) * BK, arow, a_mask, pol_a);
        }
      };
      auto load_b_at = [&](int brow, int kb, int stage) {
        if (kGemmExp && p.exp == 2) return;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          uint8_t* bdst = sb + stage * BH_BYTES + s * BH_BOX + mp * SLICE_BYTES;
          if constexpr (NMP == 1)
            tma_load_2d_pair(bdst, &tmap_b, &full[stage], (kb * KS + s) * BK, brow, pol_b);
          else
            tma_load_2d_pair_mc(bdst, &tmap_b, &full[stage], (kb * KS + s) * BK, brow, half_mask,
                                pol_b);
        }
      };
      auto load_a = [&](int ctile, int kb, int stage) { load_a_at(a_row_of(ctile), kb, stage); };
      auto load_b = [&](int ctile, int kb, int stage) { load_b_at(b_row_of(ctile), kb, stage); };
      // optional L2 prefetch of this CTA's weight slice ahead of the ring (TK_GEMM_PF;
      // measured slower, off by default)
      const int pf_dist = p.pf_dist;
      int pf_tile = 0, pf_kb = 0;
      long long pf_i = it_begin;
      auto prefetch_b_upto = [&](long long upto) {
        for (; pf_i < upto && pf_i < it_end; ++pf_i) {
          const int n_idx = pf_tile / groups_m;
          tma_prefetch_2d(&tmap_b, pf_kb * KS * BK, n_idx * NNP * BN + np * BN + half * (BN / 2) + mp * SLICE_ROWS);
          if (++pf_kb == kbs) { pf_kb = 0; ++pf_tile; }
        }
      };
      // weight tiles first (independent of the previous kernel), then wait for it
      const int pre = static_cast<int>(it_end - it_begin < STAGES ? it_end - it_begin : STAGES);
      const int tile0 = static_cast<int>(it_begin / kbs), kb0 = static_cast<int>(it_begin % kbs);
      int ctile = tile0, kb = kb0;
      for (int st = 0; st < pre; ++st) {
        if (leader) mbar_expect_tx(&full[st], xbytes);
        load_b(ctile, kb, st);
        if (++kb == kbs) { kb = 0; ++ctile; }
      }
      pf_tile = ctile;
      pf_kb = kb;
      pf_i = it_begin + pre;
      if (kGemmExp && pf_dist > 0) prefetch_b_upto(it_begin + pre + pf_dist);
      griddep_wait();
      ctile = tile0;
      kb = kb0;
      for (int st = 0; st < pre; ++st) {
        load_a(ctile, kb, st);
        if (++kb == kbs) { kb = 0; ++ctile; }
      }
      int stage = pre % STAGES;
      uint32_t phase = pre == STAGES ? 1u : 0u;
      // steady state: the weight (B) slice first -- it comes from DRAM, A from L2
      int arow = a_row_of(ctile), brow = b_row_of(ctile);
      for (long long i = it_begin + pre; i < it_end; ++i) {
        if (kGemmExp && pf_dist > 0) prefetch_b_upto(i + pf_dist + 1);
        gemm_stamp(p, 3, i - it_begin);
        mbar_wait(&empty[stage], phase ^ 1);
        gemm_stamp(p, 4, i - it_begin);
        if (leader) mbar_expect_tx(&full[stage], xbytes);
        load_b_at(brow, kb, stage);
        load_a_at(arow, kb, stage);
        if (++kb == kbs) {
          kb = 0;
          ++ctile;
          arow = a_row_of(ctile);
          brow = b_row_of(ctile);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else {
      griddep_wait();
    }
  } else if (warp == 1) {
    // The leader's whole warp runs the issue loop (converged: descriptors and
    // counters stay in uniform registers); one elected lane issues tcgen05 ops.
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN);
      // Descriptors are built once; a stage's are the base plus a constant step
      // (16-byte units of the start-address field, which cannot carry out of it:
      // shared memory is < 256 KB), so the per-stage issue is a few uniform adds
      // and the MMAs -- the issuing warp must stay ahead of the tensor pipe
      // (72 cycles per 144-wide MMA).
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sa));
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sb));
      constexpr uint32_t A_STEP = A_BYTES >> 4, B_STEP = BH_BYTES >> 4;
      const uint32_t empty0 = smem_u32(empty);
      uint32_t a_off = 0, b_off = 0, bar_off = 0;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (long long i = it_begin; i < it_end;) {
        const int ctile = static_cast<int>(i / kbs);
        const long long seg_end = min(it_end, static_cast<long long>(ctile + 1) * kbs);
        const int nkb = static_cast<int>(seg_end - i);
        if (kGemmExp && p.wait_mode) mbar_wait_lane0(&tempty[acc], acc_phase ^ 1); else mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int k = 0; k < nkb; ++k) {
          if (lane == 0) gemm_stamp(p, 0, i - it_begin + k);
          if (kGemmExp && p.wait_mode) mbar_wait_lane0(&full[stage], phase); else mbar_wait(&full[stage], phase);
          if (lane == 0) {
            gemm_stamp(p, 1, i - it_begin + k);
            if (i - it_begin + k == 0) gemm_cta_stamp(p, 1);
          }
          tc_fence_after();
          if (elect_one_sync()) {
            if (!kGemmExp || p.exp != 1) {
              const uint64_t a_desc = a_desc0 + a_off, b_desc = b_desc0 + b_off;
              umma_bf16_pair(d_tmem, a_desc, b_desc, idesc, k > 0 ? 1u : 0u);
#pragma unroll
              for (int q = 1; q < KS * (BK / 16); ++q) {
                // +32 B per K step = +2 descriptor units; KS boxes per stage
                const uint32_t s = q / (BK / 16), kk = q % (BK / 16);
                umma_bf16_pair(d_tmem, a_desc + s * (A_BOX >> 4) + 2 * kk,
                               b_desc + s * (BH_BOX >> 4) + 2 * kk, idesc, 1u);
              }
            }
            umma_commit_pair_mc_addr(empty0 + bar_off, all_mask);
            gemm_stamp(p, 2, i - it_begin + k);
          }
          __syncwarp();
          a_off += A_STEP;
          b_off += B_STEP;
          bar_off += 8;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
            a_off = b_off = bar_off = 0;
          }
        }
        if (elect_one_sync()) umma_commit_pair_mc(&tfull[acc], pair_mask);
        __syncwarp();
        if (lane == 0 && seg_end == it_end) gemm_cta_stamp(p, 2);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        i = seg_end;
      }
    }
  } else {
    const uint32_t quarter = warp & 3;
    const int row_in_tile = static_cast<int>(quarter * 32 + lane);
    const bool ep_leader = (warp == 2 && lane == 0);
    const int tid_e = static_cast<int>(threadIdx.x) - 64;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (long long i = it_begin; i < it_end;) {
      const int ctile = static_cast<int>(i / kbs);
      const long long tile_first = static_cast<long long>(ctile) * kbs;
      const long long seg_end = min(it_end, tile_first + kbs);
      const int m_idx = (ctile % groups_m) * MT + m_local;
      const int n_idx = (ctile / groups_m) * NNP + np;
      const int tile = n_idx * p.tiles_m + m_idx;
      const int row = m_idx * BM + row_in_tile;
      const int col_base = n_idx * BN;
      const int contrib = owner_of(tile_first + kbs - 1, T, G) - owner_of(tile_first, T, G) + 1;
      if constexpr (EPI == EPI_F32_BIAS_RESID) {
        // pull this row's residual segment into L2 while the MMAs run: the
        // epilogue's read-modify-write then waits on L2, not HBM
        if (row < p.M) {
          const float* seg = reinterpret_cast<const float*>(p.C) + static_cast<size_t>(row) * p.N + col_base;
#pragma unroll
          for (int c = 0; c < BN; c += 32)
            if (col_base + c < p.N) prefetch_l2(seg + c);
        }
      }
      if (kGemmExp && p.pf_partials && contrib > 1 && seg_end == it_end && i > tile_first) {
        // the final piece of a split tile: its other contributors' partials were
        // stored early (they own the tile's head) and may have left L2 under the
        // weight stream; pull them back while this piece's MMAs run
        const size_t slot_elems = static_cast<size_t>(BN / 32) * 128 * 32;
        const float* ws0 = p.ws + static_cast<size_t>(tile) * p.slots * slot_elems;
        for (int a = 0; a < contrib - 1; ++a)
          for (size_t e = static_cast<size_t>(tid_e) * 32; e < slot_elems; e += 128 * 32)
            prefetch_l2(ws0 + a * slot_elems + e);
      }
      if (kGemmExp && p.wait_mode == 2) mbar_wait_sleep(&tfull[acc], acc_phase);
      else if (kGemmExp && p.wait_mode) mbar_wait_lane0(&tfull[acc], acc_phase);
      else mbar_wait(&tfull[acc], acc_phase);
      if (ep_leader) {
        gemm_stamp(p, 5, (i - it_begin) / kbs);
        if (seg_end == it_end) gemm_cta_stamp(p, 5);
      }
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((quarter * 32) << 16) + acc * 256;
      auto release_tmem = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[acc]);
      };
      // The CTA's last tile (the shared-memory ring is idle once its MMAs are done):
      // stage the bf16 tile in shared memory and write whole rows (512 B per warp
      // instruction) instead of 16 B per thread across 32 rows.
      constexpr bool kStageable = EPI == EPI_BF16 || EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_RELU;
      constexpr int ROWB = BN * 2 + 16;
      auto stage_and_store = [&](auto&& chunk_values) {
        uint8_t* stg = smem;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          float v[32];
          chunk_values(c, v);
          epilogue_math<EPI>(p, col_base + c * 32, v);
          uint4* dst = reinterpret_cast<uint4*>(stg + row_in_tile * ROWB + c * 64);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (c * 32 + g * 8 < BN) dst[g] = make_uint4(pack_bf16x2(v[g * 8 + 0], v[g * 8 + 1]), pack_bf16x2(v[g * 8 + 2], v[g * 8 + 3]),
                                pack_bf16x2(v[g * 8 + 4], v[g * 8 + 5]), pack_bf16x2(v[g * 8 + 6], v[g * 8 + 7]));
        }
        release_tmem();
        named_bar_sync(1, 128);
        __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C);
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
          const int rr = static_cast<int>(quarter) * 32 + r;
          const int grow = m_idx * BM + rr;
          const int col = col_base + static_cast<int>(lane) * 8;
          if (grow < p.M && static_cast<int>(lane) < BN / 8 && col < p.N)
            *reinterpret_cast<uint4*>(C + static_cast<size_t>(grow) * p.N + col) =
                *reinterpret_cast<const uint4*>(stg + rr * ROWB + lane * 16);
        }
      };
      const bool staged = kStageable && p.stage_epi && seg_end == it_end;
      if constexpr (BN % 32 != 0) {
        if (!staged || contrib != 1) __trap();  // host picks such tiles only when staged
      }
      if (contrib == 1 && staged) {
        stage_and_store([&](int c, float (&v)[32]) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        });
      } else if (contrib == 1) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_row + c * 32, r);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          epilogue_store<EPI>(p, row, col_base + c * 32, v);
        }
        release_tmem();
      } else {
        int* counter = p.counters + tile;
        int* flags = p.counters + p.tiles_m * p.tiles_n + static_cast<size_t>(tile) * p.slots;
        if (ep_leader) *last_flag = atomicAdd(counter, 1);
        named_bar_sync(1, 128);
        const int arrival = *last_flag;
        const size_t slot_elems = static_cast<size_t>(BN / 32) * 128 * 32;
        float* tile_ws = p.ws + static_cast<size_t>(tile) * p.slots * slot_elems;
        // slots are indexed by contributor rank (k order), not arrival: the finishing
        // CTA's sum does not depend on which contributor arrives last
        const int me = cluster - owner_of(tile_first, T, G);
        if (arrival < contrib - 1) {
          float* mine = tile_ws + static_cast<size_t>(me) * slot_elems;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_row + c * 32, r);
            tmem_wait_ld();
            partial_store(mine, c, tid_e, r);
          }
          release_tmem();
          __threadfence();
          named_bar_sync(1, 128);
          if (ep_leader) st_release(flags + me, 1);
        } else {
          if (ep_leader) {
            for (int a = 0; a < contrib; ++a)
              while (a != me && ld_acquire(flags + a) == 0) {
              }
            if (seg_end == it_end) gemm_cta_stamp(p, 6);
          }
          named_bar_sync(1, 128);
          __threadfence();
          if (contrib == 2) {
            // one other partial: own + other is exact in either order
            const float* ows = tile_ws + static_cast<size_t>(1 - me) * slot_elems;
            // Final fixup of the CTA: one bulk copy brings the partial into the idle
            // ring behind the staging tile (one round trip instead of one per 32-column
            // chunk, which left ~7 us on the critical path).
            constexpr int kStageArea = (128 * ROWB + 1023) & ~1023;
            const bool bulk = staged && kStageArea + static_cast<int>(slot_elems) * 4 <=
                                            STAGES * STAGE_BYTES;
            if (bulk) {
              float* pbuf = reinterpret_cast<float*>(smem + kStageArea);
              if (ep_leader) {
                fence_proxy_async_global();
                const uint32_t slot_bytes = static_cast<uint32_t>(slot_elems) * 4;
                mbar_expect_tx(fix_bar, slot_bytes);
                for (uint32_t off = 0; off < slot_bytes; off += 32768)
                  bulk_g2s(reinterpret_cast<uint8_t*>(pbuf) + off,
                           reinterpret_cast<const uint8_t*>(ows) + off,
                           slot_bytes - off < 32768 ? slot_bytes - off : 32768, fix_bar);
              }
              mbar_wait(fix_bar, 0);
              const float4* p4 = reinterpret_cast<const float4*>(pbuf);
              stage_and_store([&](int c, float (&v)[32]) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(t_row + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                  const float4 q = p4[(c * 8 + g) * 128 + tid_e];
                  v[g * 4] = __uint_as_float(r[g * 4]) + q.x;
                  v[g * 4 + 1] = __uint_as_float(r[g * 4 + 1]) + q.y;
                  v[g * 4 + 2] = __uint_as_float(r[g * 4 + 2]) + q.z;
                  v[g * 4 + 3] = __uint_as_float(r[g * 4 + 3]) + q.w;
                }
              });
            } else if (staged) {
              stage_and_store([&](int c, float (&v)[32]) {
                float4 q[8];
                partial_load(ows, slot_elems, 1, c, tid_e, q);
                uint32_t r[32];
                tmem_ld_32x32b_x32(t_row + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                  v[g * 4] = __uint_as_float(r[g * 4]) + q[g].x;
                  v[g * 4 + 1] = __uint_as_float(r[g * 4 + 1]) + q[g].y;
                  v[g * 4 + 2] = __uint_as_float(r[g * 4 + 2]) + q[g].z;
                  v[g * 4 + 3] = __uint_as_float(r[g * 4 + 3]) + q[g].w;
                }
              });
            } else {
              if (kGemmExp && p.fix_depth >= 2)
                fixup_epilogue_deep<EPI, BN / 32>(p, t_row, row, col_base, ows, slot_elems, 1,
                                                  tid_e);
              else
                fixup_epilogue<EPI, BN / 32>(p, t_row, row, col_base, ows, slot_elems, 1, tid_e);
              release_tmem();
            }
          } else if (staged) {
            stage_and_store([&](int c, float (&v)[32]) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(t_row + c * 32, r);
              tmem_wait_ld();
              ranked_sum(tile_ws, slot_elems, contrib, me, c, tid_e, r, v);
            });
          } else {
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(t_row + c * 32, r);
              tmem_wait_ld();
              float v[32];
              ranked_sum(tile_ws, slot_elems, contrib, me, c, tid_e, r, v);
              epilogue_store<EPI>(p, row, col_base + c * 32, v);
            }
            release_tmem();
          }
          named_bar_sync(1, 128);
          if (ep_leader) {
            for (int a = 0; a < contrib; ++a) flags[a] = 0;
            *counter = 0;
          }
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      i = seg_end;
    }
    if (ep_leader) gemm_cta_stamp(p, 3);
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem_base);
  if (threadIdx.x == 0) gemm_cta_stamp(p, 4);
}



// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// rows x cols bf16 row-major (cols = K contiguous), box = box_rows x 64, SW128.
// Experiment switches, read once (getenv scans the environment: too slow per launch).
struct GemmEnv {
  bool no_skinny, no_pair, no_narrow;
  int fbn = 0, fcs = 0, fdp = -1;  // TK_GEMM_CFG="BN,CS,DP"
  int bpol = -1;                    // TK_GEMM_BPOL: weights' L2 policy (experiments)
  bool trace = false;               // TK_GEMM_TRACE: pipeline stamps (experiments)
  int pf = -1;                      // TK_GEMM_PF: weight prefetch distance (k-blocks)
  int exp = 0;                      // TK_GEMM_EXP: pipeline experiments (wrong results)
  int wait_mode = -1;               // TK_GEMM_WAIT
  int fix_depth = -1;               // TK_GEMM_FIXDEPTH
  int stage_epi = -1;               // TK_GEMM_STAGE_EPI
  int ks = -1;                      // TK_GEMM_KS: k-blocks per ring stage of 160-wide tiles
  int entry_pf = -1;                // TK_GEMM_ENTRY_PF
  int skinny_ctas = 0;              // TK_GEMM_SKINNY_CTAS: CTA cap of the decode GEMMs
  bool no144 = false;               // TK_NO_144: keep 160-wide 4-CTA clusters
  bool cs8 = false;                 // TK_GEMM_CS8=1: 8-CTA (2 x 2 pair) clusters, experiments
  int pf_partials = -1;             // TK_GEMM_PFPART
  GemmEnv() {
    no_skinny = getenv("TK_NO_SKINNY") != nullptr;
    no_pair = getenv("TK_NO_PAIR") != nullptr;
    no_narrow = getenv("TK_NO_NARROW") != nullptr;
    if (const char* f = getenv("TK_GEMM_CFG")) sscanf(f, "%d,%d,%d", &fbn, &fcs, &fdp);
    if (const char* f = getenv("TK_GEMM_BPOL")) bpol = atoi(f);
    trace = getenv("TK_GEMM_TRACE") != nullptr;
    if (const char* f = getenv("TK_GEMM_PF")) pf = atoi(f);
    if (const char* f = getenv("TK_GEMM_EXP")) exp = atoi(f);
    if (const char* f = getenv("TK_GEMM_WAIT")) wait_mode = atoi(f);
    if (const char* f = getenv("TK_GEMM_FIXDEPTH")) fix_depth = atoi(f);
    if (const char* f = getenv("TK_GEMM_STAGE_EPI")) stage_epi = atoi(f);
    if (const char* f = getenv("TK_GEMM_KS")) ks = atoi(f);
    if (const char* f = getenv("TK_GEMM_ENTRY_PF")) entry_pf = atoi(f);
    if (const char* f = getenv("TK_GEMM_SKINNY_CTAS")) skinny_ctas = atoi(f);
    no144 = getenv("TK_NO_144") != nullptr;
    if (const char* f = getenv("TK_GEMM_CS8")) cs8 = atoi(f) != 0;
    if (const char* f = getenv("TK_GEMM_PFPART")) pf_partials = atoi(f);
    if (const char* c = getenv("TK_GEMM_MAX_CTAS")) max_ctas = atoi(c);
  }
  int max_ctas = 0;  // TK_GEMM_MAX_CTAS: cap the CTAs (skips the split-minimising pick)
};
static const GemmEnv& genv() {
  static const GemmEnv e;
  return e;
}

// Tensor maps are encoded once per (base, rows, cols, box): weights and the
// runtime's activation buffers have fixed addresses, so decode steps (hundreds
// of GEMMs each) reuse them instead of calling cuTensorMapEncodeTiled per launch.
struct TmapKey {
  const void* base;
  uint64_t rows, cols;
  uint32_t box;
  bool operator==(const TmapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && box == o.box;
  }
};
struct TmapHash {
  size_t operator()(const TmapKey& k) const {
    return std::hash<const void*>()(k.base) ^ (k.rows * 0x9E3779B97F4A7C15ull) ^ (k.cols << 20) ^ k.box;
  }
};

static int encode_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_rows);

int make_tmap_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows) {
  static std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  const TmapKey key{base, rows, cols, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return TK_OK;
  }
  const int rc = encode_kmajor(map, base, rows, cols, box_rows);
  if (rc) return rc;
  if (cache.size() > 16384) cache.clear();  // freed buffers' addresses may be reused: bounded
  cache.emplace(key, *map);
  return TK_OK;
}

static int encode_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  TK_CHECK(fn != nullptr, TK_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TK_CHECK(r == CUDA_SUCCESS, TK_ECUDA,
           "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return TK_OK;
}

// KV pool viewed as 4 KB blocks of (page, layer, head, K|V): {64 d,
// page_tokens slots, 2 d-halves, blocks}; one box = one block, landing in
// shared memory as [half][slot][128 B] with the 128-byte swizzle (the UMMA
// MN-major layout of V for one page).
int make_tmap_kv_pages(CUtensorMap* map, const void* pool, uint64_t blocks, uint32_t page_tokens) {
  EncodeTiledFn fn = encode_fn();
  TK_CHECK(fn != nullptr, TK_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const uint64_t row = 128 * 2;  // bytes per slot (head_dim 128)
  cuuint64_t dims[4] = {64, page_tokens, 2, blocks};
  cuuint64_t strides[3] = {row, 128, page_tokens * row};
  cuuint32_t box[4] = {64, page_tokens, 2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pool), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TK_CHECK(r == CUDA_SUCCESS, TK_ECUDA,
           "cuTensorMapEncodeTiled (kv pages) failed (" + std::to_string(static_cast<int>(r)) + ")");
  return TK_OK;
}

static int pick_bn(int N) { return N >= 1024 ? 256 : 128; }

// Co-resident clusters of size cs for the BN variant (queried once per variant).
static int max_clusters_for(int bn, int cs);

// Counter/flag region at the head of every GEMM workspace.  It is shared by all
// GEMM shapes that use the workspace and is zero between launches (the last
// contributor of each tile resets what it used), so it must never overlap the
// partial slots of any shape: it has a fixed size.
constexpr int64_t kCounterBytes = 1 << 20;

constexpr int kSkinnyMaxM = 128;

static int skinny_nb(int M) { return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128; }

struct GemmPlan {
  bool counters_fit;
  bool pair;    // cta_group::2 path (tiles_m even)
  bool skinny;  // swap-AB weight-streaming path (M <= 128)
  int nb;       // skinny: UMMA N (batch rows, padded)
  int bn, cs, tiles_m, tiles_n, kbs, clusters, slots;
  int ks;  // pair kernel: 64-wide k-blocks per ring stage (kbs counts stages)
  long long total_iters;
  int64_t ws_bytes;
};

static int max_skinny_ctas(int nb);
static int max_pair_clusters(int cs);

// Stream-K range boundaries that fall inside a tile cost a partial-tile
// exchange.  Among cluster counts in [0.85*max, max] take the one with the
// fewest split tiles (ties: more clusters), e.g. QKV at M=512 has 60 cluster
// tiles -> 30 clusters own exactly two tiles each and nothing is split.
static int pick_clusters(long long total_iters, int kbs, int max_clusters) {
  int best = max_clusters, best_splits = 1 << 30;
  for (int g = max_clusters; g >= std::max(1, (max_clusters * 85) / 100); --g) {
    int splits = 0;
    for (int c = 1; c < g; ++c)
      if ((static_cast<long long>(c) * total_iters / g) % kbs != 0) ++splits;
    if (splits < best_splits) {
      best_splits = splits;
      best = g;
    }
  }
  return best;
}

static GemmPlan plan_skinny(int M, int N, int K, int max_ctas) {
  GemmPlan pl{};
  pl.skinny = true;
  pl.nb = skinny_nb(M);
  pl.bn = 128;
  pl.cs = 1;
  pl.tiles_m = 1;
  pl.tiles_n = (N + 127) / 128;
  pl.kbs = K / 64;
  pl.total_iters = static_cast<long long>(pl.tiles_n) * pl.kbs;
  // 120 of the 148 SMs (measured best for decode chains at M=8..128: 4-11% faster
  // than all SMs): the next GEMM's CTAs start on the free SMs and stream their first
  // weight tiles (PDL) while this one drains.  TK_GEMM_SKINNY_CTAS overrides.
  int ctas = std::min(max_skinny_ctas(pl.nb), genv().skinny_ctas > 0 ? genv().skinny_ctas : 120);
  // TK_GEMM_SKINNY_MAP="N,K,G;...": per-shape CTA counts (experiments)
  if (const char* m = getenv("TK_GEMM_SKINNY_MAP")) {
    int n_, k_, g_, used = 0;
    while (sscanf(m, "%d,%d,%d%n", &n_, &k_, &g_, &used) == 3) {
      if (n_ == N && k_ == K) ctas = std::min(max_skinny_ctas(pl.nb), g_);
      m += used;
      if (*m != ';') break;
      ++m;
    }
  }
  if (max_ctas > 0) ctas = std::min(ctas, max_ctas);
  ctas = static_cast<int>(std::min<long long>(ctas, std::max<long long>(1, pl.total_iters / 4)));
  pl.clusters = ctas;
  int most = 1;
  for (long long t = 0; t < pl.tiles_n; ++t) {
    const int c = owner_of((t + 1) * pl.kbs - 1, pl.total_iters, ctas) -
                  owner_of(t * pl.kbs, pl.total_iters, ctas) + 1;
    most = std::max(most, c);
  }
  pl.slots = most;  // rank-indexed partial slots (the finishing rank leaves its own unused)
  pl.ws_bytes = kCounterBytes + static_cast<int64_t>(pl.tiles_n) * pl.slots * 128LL * pl.nb * 4;
  pl.counters_fit = static_cast<int64_t>(pl.tiles_n) * (1 + pl.slots) * 4 <= kCounterBytes;
  return pl;
}

static GemmPlan plan_gemm(int M, int N, int K, int max_ctas) {
  if (M <= kSkinnyMaxM && !genv().no_skinny) return plan_skinny(M, N, K, max_ctas);
  GemmPlan pl{};
  pl.bn = pick_bn(N);
  pl.tiles_m = (M + 127) / 128;
  pl.pair = pl.bn == 256 && pl.tiles_m % 2 == 0 && !genv().no_pair;
  pl.cs = pl.tiles_m % 4 == 0 ? 4 : (pl.tiles_m % 2 == 0 ? 2 : 1);
  if (pl.pair && pl.cs == 1) pl.cs = 2;
  pl.kbs = K / 64;
  int clusters = pl.pair ? max_pair_clusters(pl.cs) : max_clusters_for(pl.bn, pl.cs);
  if (max_ctas > 0) clusters = std::min(clusters, std::max(1, max_ctas / pl.cs));
  bool data_parallel = false;
  if (pl.pair) {
    // Tile shape.  Default: 256-wide tiles, stream-K over the clusters (every
    // split tile costs a partial exchange).  When 160-wide tiles cover the
    // GEMM in one wave of clusters and K is short (nothing to amortise the
    // exchange over), a data-parallel schedule with one tile per cluster wins:
    // O-proj at M=512 38 -> 46 us (measured); for long K (FC2) or several
    // waves (QKV, FC1) the narrow tiles lose to their extra L2 traffic for A.
    // TK_GEMM_CFG="BN,CS,DP" forces a schedule (experiments)
    const int fbn = genv().fbn, fcs = genv().fcs, fdp = genv().fdp;
    if (fdp >= 0 && (fbn == 256 || fbn == 160) && (fcs == 2 || (fcs == 4 && pl.tiles_m % 4 == 0))) {
      pl.bn = fbn;
      pl.cs = fcs;
      clusters = max_pair_clusters(fcs);
      if (max_ctas > 0) clusters = std::min(clusters, std::max(1, max_ctas / fcs));
      if (fdp) {
        const long long T = static_cast<long long>(pl.tiles_m / fcs) * ((N + fbn - 1) / fbn);
        long long g = std::min<long long>(T, clusters);
        while (T % g) --g;
        clusters = static_cast<int>(g);
        data_parallel = true;
      }
    } else if (K <= 8192 && !genv().no_narrow) {
      const int groups_m = pl.tiles_m / pl.cs;
      const int tn = (N + 159) / 160;
      if (tn * groups_m <= clusters && 4 * tn * groups_m >= 3 * clusters) {
        pl.bn = 160;
        clusters = tn * groups_m;  // one tile per cluster
        data_parallel = true;
      }
    }
  }
  pl.tiles_n = (N + pl.bn - 1) / pl.bn;
  // 8-CTA clusters (2 x 2 pairs: A shared along N as well as B along M) for the
  // 256-wide stream-K schedule: a third less L2->SM traffic per FLOP, but only 12
  // such clusters (96 SMs) are co-resident on a B200, so it is off by default
  // (TK_GEMM_CS8=1; profiles/r02_experiments.md)
  if (pl.pair && pl.bn == 256 && pl.cs == 4 && !data_parallel && pl.tiles_n % 2 == 0 &&
      genv().cs8 && genv().fcs == 0) {
    const int c8 = max_pair_clusters(8);
    if (c8 >= 8) {
      pl.cs = 8;
      clusters = max_ctas > 0 ? std::min(c8, std::max(1, max_ctas / 8)) : c8;
    }
  }
  pl.ks = 1;
  // 160-wide tiles: two k-blocks per ring stage (O-proj at M=512: 34.8 -> 32.8 us,
  // the per-launch fill cost halves); TK_GEMM_KS=1 restores one
  if (pl.pair && pl.kbs % 2 == 0 &&
      ((pl.bn == 160 && genv().ks != 1) || (pl.bn == 256 && genv().ks == 4))) {
    pl.ks = 2;
    pl.kbs /= 2;
  }
  // cluster tiles: (tiles_m / MT) m-groups x (tiles_n / NNP) n-groups
  pl.total_iters = pl.cs == 8
                       ? static_cast<long long>(pl.tiles_m / 4) * (pl.tiles_n / 2) * pl.kbs
                       : static_cast<long long>(pl.tiles_m / pl.cs) * pl.tiles_n * pl.kbs;
  clusters = static_cast<int>(std::min<long long>(clusters, std::max<long long>(1, pl.total_iters / 4)));
  // Long K (FC2: 320 k-blocks per tile) amortises a split tile's exchange: use
  // every cluster; short K prefers the count with the fewest split tiles.
  if (max_ctas <= 0 && !data_parallel && pl.kbs < 256)
    clusters = pick_clusters(pl.total_iters, pl.kbs, clusters);
  pl.clusters = clusters;
  // most CTAs (clusters) sharing one tile, over all cluster tiles
  const long long ctiles = pl.total_iters / pl.kbs;
  int most = 1;
  for (long long t = 0; t < ctiles; ++t) {
    const int c = owner_of((t + 1) * pl.kbs - 1, pl.total_iters, clusters) -
                  owner_of(t * pl.kbs, pl.total_iters, clusters) + 1;
    most = std::max(most, c);
  }
  pl.slots = most;  // rank-indexed partial slots (the finishing rank leaves its own unused)
  const int64_t tiles = static_cast<int64_t>(pl.tiles_m) * pl.tiles_n;
  // [kCounterBytes: per-tile counters + ready flags, always left zeroed][partial slots]
  pl.ws_bytes = kCounterBytes + tiles * pl.slots * 128LL * pl.bn * 4;
  pl.counters_fit = tiles * (1 + pl.slots) * 4 <= kCounterBytes;
  return pl;
}

int64_t gemm_workspace_bytes(int M, int N, int K) {
  return plan_gemm(M, N, K, genv().max_ctas).ws_bytes;
}

// Programmatic dependent launch (TK_NO_PDL=1 disables): the GEMM may start
// while the previous kernel on the stream drains; its producer prefetches
// weight tiles and then waits (griddepcontrol.wait) before touching activations.
static int set_pdl(cudaLaunchAttribute* attr, int n) {
  if (!pdl_enabled()) return n;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  return n + 1;
}

template <int NB, int EPI>
static int launch_skinny(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a,
                         int ctas, cudaStream_t stream) {
  using Cfg = SkinnyCfg<NB>;
  auto kern = gemm_skinny_kernel<NB, EPI>;
  TK_SMEM_OPT_IN(kern, Cfg::SMEM_BYTES);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  cfg.numAttrs = set_pdl(attr, 0);
  cfg.attrs = attr;
  TK_CUDA(cudaLaunchKernelEx(&cfg, kern, tw, tx, a));
  TK_CUDA(cudaGetLastError());
  note_launch();
  return TK_OK;
}

template <int NB>
static int skinny_epi(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a, int ctas,
                      cudaStream_t s) {
  switch (a.epi) {
    case EPI_BF16: return launch_skinny<NB, EPI_BF16>(tw, tx, a, ctas, s);
    case EPI_BF16_BIAS: return launch_skinny<NB, EPI_BF16_BIAS>(tw, tx, a, ctas, s);
    case EPI_BF16_BIAS_RELU: return launch_skinny<NB, EPI_BF16_BIAS_RELU>(tw, tx, a, ctas, s);
    case EPI_F32_BIAS_RESID: return launch_skinny<NB, EPI_F32_BIAS_RESID>(tw, tx, a, ctas, s);
    case EPI_F32: return launch_skinny<NB, EPI_F32>(tw, tx, a, ctas, s);
    case EPI_QKV_PAGED: return launch_skinny<NB, EPI_QKV_PAGED>(tw, tx, a, ctas, s);
  }
  set_error("unknown gemm epilogue");
  return TK_EINVAL;
}

template <int EPI, int CS, int BN, int KS>
static int launch_pair_ks(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                          int clusters, cudaStream_t stream) {
  auto kern = gemm_pair_kernel<EPI, CS, BN, KS>;
  TK_SMEM_OPT_IN(kern, PairCfg<BN, KS>::SMEM);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CS);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = PairCfg<BN, KS>::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = set_pdl(attr, 1);
  TK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
  note_launch();
  return TK_OK;
}

// a.kbs counts stages of KS k-blocks
template <int EPI, int CS, int BN>
static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                       int clusters, cudaStream_t stream, int ks) {
  if (ks == 2) return launch_pair_ks<EPI, CS, BN, 2>(ta, tb, a, clusters, stream);
  return launch_pair_ks<EPI, CS, BN, 1>(ta, tb, a, clusters, stream);
}

template <int CS, int BN>
static int pair_epi(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, int clusters,
                    cudaStream_t s, int ks = 1) {
  switch (a.epi) {
    case EPI_BF16: return launch_pair<EPI_BF16, CS, BN>(ta, tb, a, clusters, s, ks);
    case EPI_BF16_BIAS: return launch_pair<EPI_BF16_BIAS, CS, BN>(ta, tb, a, clusters, s, ks);
    case EPI_BF16_BIAS_RELU: return launch_pair<EPI_BF16_BIAS_RELU, CS, BN>(ta, tb, a, clusters, s, ks);
    case EPI_F32_BIAS_RESID: return launch_pair<EPI_F32_BIAS_RESID, CS, BN>(ta, tb, a, clusters, s, ks);
    case EPI_F32: return launch_pair<EPI_F32, CS, BN>(ta, tb, a, clusters, s, ks);
    case EPI_QKV_PAGED: return launch_pair<EPI_QKV_PAGED, CS, BN>(ta, tb, a, clusters, s, ks);
  }
  set_error("unknown gemm epilogue");
  return TK_EINVAL;
}

template <int CS>
static int query_pair_clusters() {
  auto kern = gemm_pair_kernel<EPI_BF16, CS, 256, 1>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<256>::SMEM) !=
      cudaSuccess) {
    cudaGetLastError();
    return kNumSMs / CS;
  }
  cudaLaunchConfig_t q{};
  q.gridDim = dim3(kNumSMs / CS * CS);
  q.blockDim = dim3(192);
  q.dynamicSmemBytes = PairCfg<256>::SMEM;
  cudaLaunchAttribute qa[1];
  qa[0].id = cudaLaunchAttributeClusterDimension;
  qa[0].val.clusterDim.x = CS;
  qa[0].val.clusterDim.y = 1;
  qa[0].val.clusterDim.z = 1;
  q.attrs = qa;
  q.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return kNumSMs / CS;
  }
  return n;
}

static int max_pair_clusters(int cs) {
  static int c2 = 0, c4 = 0, c8 = 0;
  if (cs == 8) {
    if (!c8) c8 = query_pair_clusters<8>();
    return c8;
  }
  if (cs == 4) {
    if (!c4) c4 = query_pair_clusters<4>();
    return c4;
  }
  if (!c2) c2 = query_pair_clusters<2>();
  return c2;
}

static int max_skinny_ctas(int nb) {
  (void)nb;
  return kNumSMs;  // one CTA per SM (>100 KB of smem each)
}

template <int BN, int EPI, int CS>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                       int clusters, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tn_kernel<BN, EPI, CS>;
  TK_SMEM_OPT_IN(kern, Cfg::SMEM_BYTES);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CS);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = set_pdl(attr, 1);
  TK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
  note_launch();
  return TK_OK;
}

template <int BN, int CS>
static int query_clusters() {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tn_kernel<BN, EPI_BF16, CS>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) !=
      cudaSuccess)
    return kNumSMs / CS;
  if (CS == 1) return kNumSMs;
  cudaLaunchConfig_t q{};
  q.gridDim = dim3(kNumSMs / CS * CS);
  q.blockDim = dim3(Cfg::THREADS);
  q.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cudaLaunchAttribute qa[1];
  qa[0].id = cudaLaunchAttributeClusterDimension;
  qa[0].val.clusterDim.x = CS;
  qa[0].val.clusterDim.y = 1;
  qa[0].val.clusterDim.z = 1;
  q.attrs = qa;
  q.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return kNumSMs / CS;
  }
  return n;
}

static int max_clusters_for(int bn, int cs) {
  static int cache[2][3] = {{0, 0, 0}, {0, 0, 0}};
  const int bi = bn == 256 ? 1 : 0;
  const int ci = cs == 4 ? 2 : (cs == 2 ? 1 : 0);
  int& v = cache[bi][ci];
  if (v == 0) {
    if (bn == 256) v = cs == 4 ? query_clusters<256, 4>() : cs == 2 ? query_clusters<256, 2>() : query_clusters<256, 1>();
    else v = cs == 4 ? query_clusters<128, 4>() : cs == 2 ? query_clusters<128, 2>() : query_clusters<128, 1>();
  }
  return v;
}

template <int BN, int CS>
static int dispatch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                        int clusters, cudaStream_t s) {
  switch (a.epi) {
    case EPI_BF16: return launch_gemm<BN, EPI_BF16, CS>(ta, tb, a, clusters, s);
    case EPI_BF16_BIAS: return launch_gemm<BN, EPI_BF16_BIAS, CS>(ta, tb, a, clusters, s);
    case EPI_BF16_BIAS_RELU: return launch_gemm<BN, EPI_BF16_BIAS_RELU, CS>(ta, tb, a, clusters, s);
    case EPI_F32_BIAS_RESID: return launch_gemm<BN, EPI_F32_BIAS_RESID, CS>(ta, tb, a, clusters, s);
    case EPI_F32: return launch_gemm<BN, EPI_F32, CS>(ta, tb, a, clusters, s);
    case EPI_QKV_PAGED: return launch_gemm<BN, EPI_QKV_PAGED, CS>(ta, tb, a, clusters, s);
  }
  set_error("unknown gemm epilogue");
  return TK_EINVAL;
}

template <int BN>
static int dispatch_cs(const void* B, int N, int K, const CUtensorMap& ta, GemmArgs& a,
                       int clusters, cudaStream_t s) {
  CUtensorMap tb;
  int rc = make_tmap_kmajor(&tb, B, N, K, BN / a.cs);
  if (rc) return rc;
  switch (a.cs) {
    case 4: return dispatch_epi<BN, 4>(ta, tb, a, clusters, s);
    case 2: return dispatch_epi<BN, 2>(ta, tb, a, clusters, s);
    default: return dispatch_epi<BN, 1>(ta, tb, a, clusters, s);
  }
}

bool gemm_is_skinny(int M) { return M <= kSkinnyMaxM && !genv().no_skinny; }

int gemm_bf16(const void* A, const void* B, void* C, const void* bias, int M, int N, int K,
              int epi, void* workspace, int64_t ws_bytes, cudaStream_t stream, int max_ctas,
              const QkvScatter* scatter) {
  TK_CHECK(epi != EPI_QKV_PAGED || (scatter && N % 32 == 0 &&
                                    N == 3 * scatter->g.n_heads * scatter->g.head_dim &&
                                    scatter->g.head_dim % 32 == 0),
           TK_EINVAL, "gemm: EPI_QKV_PAGED needs a scatter target, M above the skinny range");
  TK_CHECK(M > 0 && N > 0 && K > 0, TK_EINVAL, "gemm: empty problem");
  TK_CHECK(K % 64 == 0, TK_EINVAL, "gemm: K must be a multiple of 64");
  TK_CHECK(N % 8 == 0, TK_EINVAL, "gemm: N must be a multiple of 8");
  if (max_ctas <= 0 && genv().max_ctas > 0) max_ctas = genv().max_ctas;  // experiments only
  // plans depend only on the shape (and the experiment switches): cache them
  static std::unordered_map<uint64_t, GemmPlan> plans;
  static std::mutex plans_mu;
  std::unique_lock<std::mutex> plans_lock(plans_mu);
  const uint64_t pkey = (static_cast<uint64_t>(M) << 44) ^ (static_cast<uint64_t>(N) << 22) ^
                        static_cast<uint64_t>(K) ^ (static_cast<uint64_t>(max_ctas) << 58);
  auto pit = plans.find(pkey);
  if (pit == plans.end()) pit = plans.emplace(pkey, plan_gemm(M, N, K, max_ctas)).first;
  const GemmPlan pl = pit->second;
  plans_lock.unlock();
  static const bool debug = getenv("TK_GEMM_DEBUG") != nullptr;
  if (debug)
    fprintf(stderr, "gemm M=%d N=%d K=%d: %s bn=%d cs=%d clusters=%d slots=%d\n", M, N, K,
            pl.skinny ? "skinny" : pl.pair ? "pair" : "tn", pl.bn, pl.cs, pl.clusters, pl.slots);
  TK_CHECK(ws_bytes >= pl.ws_bytes, TK_EINVAL, "gemm: workspace too small");
  TK_CHECK(pl.counters_fit, TK_EINVAL, "gemm: too many tiles for the counter region");
  GemmPlan pl144 = pl;
  if (pl.pair && pl.tiles_m % 2 == 0 &&
      (epi == EPI_BF16 || epi == EPI_BF16_BIAS || epi == EPI_BF16_BIAS_RELU) &&
      genv().stage_epi != 0 && !genv().no144 && max_ctas <= 0 &&
      (genv().fbn == 0 || genv().fbn == 160)) {
    // One wave of 144-wide tiles on 2-CTA clusters, one tile per pair (cuBLAS's
    // structure for these shapes): up to 74 pairs = 148 SMs, where 4-CTA clusters
    // reach 132 and a stream-K schedule pays split-tile fixups.  O-proj and FC2 at
    // M=512: 72 pairs.  O-proj -4.4% in situ, FC2 88.5 -> 84.4 us isolated.
    const int tn = (N + 143) / 144, groups = pl.tiles_m / 2;
    const int cmax = max_pair_clusters(2);
    if (tn * groups <= cmax && 10 * tn * groups >= 9 * cmax) {
      const int kb64 = K / 64;
      pl144.ks = (kb64 % 2 == 0 && genv().ks != 1) ? 2 : 1;
      pl144.kbs = kb64 / pl144.ks;
      pl144.bn = 144;
      pl144.cs = 2;
      pl144.tiles_n = tn;
      pl144.clusters = tn * groups;
      pl144.total_iters = static_cast<long long>(groups) * tn * pl144.kbs;
    }
  }
  if (pl.skinny) {
    CUtensorMap tw, tx;
    int rc = make_tmap_kmajor(&tw, B, N, K, 128);
    if (rc) return rc;
    rc = make_tmap_kmajor(&tx, A, M, K, pl.nb);
    if (rc) return rc;
    GemmArgs a{};
    a.kv = scatter ? *scatter : QkvScatter{};
    a.C = C;
    a.bias = static_cast<const __nv_bfloat16*>(bias);
    a.M = M;
    a.N = N;
    a.K = K;
    a.epi = epi;
    a.tiles_m = 1;
    a.tiles_n = pl.tiles_n;
    a.kbs = pl.kbs;
    a.cs = 1;
    a.slots = pl.slots;
    a.total_iters = pl.total_iters;
    a.counters = static_cast<int*>(workspace);
    a.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + kCounterBytes);
    switch (pl.nb) {
      case 16: return skinny_epi<16>(tw, tx, a, pl.clusters, stream);
      case 32: return skinny_epi<32>(tw, tx, a, pl.clusters, stream);
      case 64: return skinny_epi<64>(tw, tx, a, pl.clusters, stream);
      default: return skinny_epi<128>(tw, tx, a, pl.clusters, stream);
    }
  }
  CUtensorMap ta;
  int rc = make_tmap_kmajor(&ta, A, M, K, 128);
  if (rc) return rc;
  GemmArgs a;
  a.C = C;
  a.bias = static_cast<const __nv_bfloat16*>(bias);
  a.M = M;
  a.N = N;
  a.K = K;
  a.epi = epi;
  a.tiles_m = pl.tiles_m;
  a.tiles_n = pl.tiles_n;
  a.kbs = pl.kbs;
  a.cs = pl.cs;
  // weights: evict first (measured best for every schedule, also 2-CTA clusters whose
  // two m-groups both read each weight tile; TK_GEMM_BPOL overrides)
  a.b_pol = genv().bpol >= 0 ? genv().bpol : 0;
  a.trace = genv().trace ? 1 : 0;
  a.pf_dist = genv().pf >= 0 ? genv().pf : 0;
  a.exp = genv().exp;
  a.wait_mode = genv().wait_mode >= 0 ? genv().wait_mode : 0;
  a.fix_depth = genv().fix_depth >= 0 ? genv().fix_depth : 1;
  a.stage_epi = genv().stage_epi >= 0 ? genv().stage_epi : 1;
  a.entry_pf = genv().entry_pf >= 0 ? genv().entry_pf : 0;  // measured: slightly slower
  a.pf_partials = genv().pf_partials >= 0 ? genv().pf_partials : 0;
  a.slots = pl.slots;
  a.total_iters = pl.total_iters;
  a.counters = static_cast<int*>(workspace);
  a.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + kCounterBytes);
  a.kv = scatter ? *scatter : QkvScatter{};
  if (pl.pair) {
    // each CTA loads 64-row (CS=4) or 128-row (CS=2) slices of its B half
    CUtensorMap tb;
    if (pl144.bn == 144) {
      a.tiles_n = pl144.tiles_n;
      a.cs = 2;
      a.kbs = pl144.kbs;
      a.total_iters = pl144.total_iters;
      rc = make_tmap_kmajor(&tb, B, N, K, 72);
      if (rc) return rc;
      return pair_epi<2, 144>(ta, tb, a, pl144.clusters, stream, pl144.ks);
    }
    rc = make_tmap_kmajor(&tb, B, N, K, pl.bn / 2 / (pl.cs == 8 ? 2 : pl.cs / 2));
    if (rc) return rc;
    if (pl.cs == 8) {
      // each CTA loads half of its A tile (64 rows) and multicasts it to its N-neighbour
      rc = make_tmap_kmajor(&ta, A, M, K, 64);
      if (rc) return rc;
      return pair_epi<8, 256>(ta, tb, a, pl.clusters, stream, pl.ks);
    }
    if (pl.bn == 160) {
      if (pl.cs == 4) return pair_epi<4, 160>(ta, tb, a, pl.clusters, stream, pl.ks);
      return pair_epi<2, 160>(ta, tb, a, pl.clusters, stream, pl.ks);
    }
    if (pl.cs == 4) return pair_epi<4, 256>(ta, tb, a, pl.clusters, stream, pl.ks);
    return pair_epi<2, 256>(ta, tb, a, pl.clusters, stream, pl.ks);
  }
  if (pl.bn == 256) return dispatch_cs<256>(B, N, K, ta, a, pl.clusters, stream);
  return dispatch_cs<128>(B, N, K, ta, a, pl.clusters, stream);
}

}  // namespace tk
