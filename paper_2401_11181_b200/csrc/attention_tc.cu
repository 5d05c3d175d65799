// attention_tc.cu -- chunked-prefill attention (K2) on 5th-gen tensor cores.
//
// One CTA = one head x one <=128-row query block x one KV split (128-key
// blocks).  Per block:  S = Q K^T  (UMMA 128x128x128 -> TMEM),  softmax by
// warps 0-3 with one query row per thread straight out of TMEM (no shuffles),
// P (bf16) written to shared memory in the UMMA K-major SW128 layout,
// O += P V  (UMMA, V as an MN-major operand -> TMEM).  K and V tiles are
// TMA-loaded from the page-major KV pool by 16 lanes of the producer warp in
// parallel (2 KB [16 keys][64 d] boxes into [d-half][64 keys][128 B] tiles),
// 64-key blocks in a 4-stage ring so three blocks are in flight ahead of the
// tensor core; V is consumed as an MN-major operand.
//
// Warp roles (192 threads): 0-3 softmax / O correction / output, 4 TMA
// producer, 5 TMEM allocator + single-thread UMMA issuer.  The issuer runs
// S_{j+1} as soon as the softmax warps have pulled S_j into registers, so the
// tensor core overlaps the exponentials.  O is rescaled in TMEM only when a
// row maximum grows by more than 2^8 (exp2 domain; decided per warp, since
// TMEM loads/stores are warp-collective); the final normalisation uses the
// same stale maximum, so results are exact up to fp32 rounding.
#include "tk_common.cuh"
#include "tk_kernels.h"

#include <cstdlib>

namespace tk {

namespace {
constexpr int kRows = 128;
constexpr int kKeys = 64;                  // keys per KV block
constexpr int kD = 128;
constexpr int kStages = 4;                 // K/V blocks in flight
constexpr int kPBuf = 2;                   // P double buffer: softmax j+1 overlaps PV j
constexpr int kQTile = kRows * kD * 2;     // 32 KB: Q as two SW128 atom columns [128][64]
constexpr int kQHalf = kQTile / 2;
constexpr int kKvHalf = kKeys * 64 * 2;    // 8 KB: one d-half of a K or V block
constexpr int kKTile = 2 * kKvHalf;        // 16 KB: [half][64 keys][128 B]
constexpr int kStageBytes = 2 * kKTile;    // K then V
constexpr int kPTile = kRows * kKeys * 2;  // 16 KB: P [128][64] bf16 (one atom column)
constexpr int kSmem = kQTile + kStages * kStageBytes + kPBuf * kPTile + 256;
constexpr float kRescaleThreshold = 8.f;  // log2 units
}  // namespace

// 2^x on the FMA/ALU pipes (no MUFU): x = n + f with |f| <= 1/2 by the
// magic-constant rounding trick, 2^f by a degree-5 polynomial, 2^n added to
// the exponent field with an integer add.  -inf maps to 2^-126 ~ 0.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.f);
  // round-to-nearest split via the 1.5 * 2^23 magic constant: x = n + f, |f| <= 1/2
  const float y = x + 12582912.f;
  const float n = y - 12582912.f;
  const float f = x - n;
  float q = 1.3333558e-3f;  // 2^f, degree-5 Taylor in f*ln2 (rel. err < 3e-6 on [-1/2,1/2])
  q = fmaf(q, f, 9.6181291e-3f);
  q = fmaf(q, f, 5.5504109e-2f);
  q = fmaf(q, f, 2.4022651e-1f);
  q = fmaf(q, f, 6.9314718e-1f);
  q = fmaf(q, f, 1.0f);
  return __int_as_float(__float_as_int(q) + ((__float_as_int(y) - 0x4B400000) << 23));
}

struct TcAttnParams {
  const AttnWork* work;
  const AttnQBlock* qblocks;
  const tk_slice* slices;
  const int32_t* bt;
  __nv_bfloat16* o;
  float* partial;
  int n_layers, n_heads, layer, page_tokens;
  float scale_log2;
};

__global__ void __launch_bounds__(192, 1)
    chunk_attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_q,
                         const __grid_constant__ CUtensorMap tmap_k, const TcAttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];  // SW128 atoms need 1 KB alignment
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kQTile;                           // [stage]{K [half][64][128 B], V same}
  uint8_t* sP = sKV + kStages * kStageBytes;              // [kPBuf][128][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPBuf * kPTile);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;               // [kStages]
  uint64_t* kv_empty = kv_full + kStages;     // [kStages]
  uint64_t* s_full = kv_empty + kStages;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;       // [kPBuf] per P buffer
  uint64_t* o_done = p_full + kPBuf;   // [kPBuf]: PV_j retired (j % kPBuf)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + kPBuf);

  const uint32_t warp = warp_id(), lane = lane_id();
  const AttnWork w = p.work[blockIdx.x];
  const AttnQBlock qb = p.qblocks[w.qblock];
  const int head = blockIdx.y;
  const tk_slice sl = p.slices[qb.slice];
  const int32_t* pages = p.bt + sl.bt_offset;
  const int kv_end = qb.pos0 + qb.nrows;
  const int nblk = w.kb1 - w.kb0;

  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    for (int b = 0; b < kPBuf; ++b) {
      mbar_init(&p_full[b], 4);
      mbar_init(&o_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S at col 0, O at col 128

  if (warp == 4) {
    // ------------------------------------------------------------ producer warp
    // lane 0 owns the barriers; lanes 0-15 each issue one 2 KB box per block:
    // lanes 0-7 K (page i, d-half h), lanes 8-15 V, into [half][64 keys][128 B].
    const uint64_t pol = l2_policy_evict_first();
    if (lane == 0) {
      mbar_expect_tx(q_full, kQTile);
      for (int h = 0; h < 2; ++h)
        tma_load_2d(sQ + h * kQHalf, &tmap_q, q_full, head * kD + h * 64, qb.row0, pol);
    }
    const int pt = p.page_tokens;
    for (int j = 0; j < nblk; ++j) {
      const int st = j % kStages;
      if (lane == 0) {
        mbar_wait(&kv_empty[st], ((j / kStages) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], kStageBytes);
      }
      __syncwarp();
      if (lane < 16) {
        const int kv = lane >> 3, i = (lane >> 1) & 3, h = lane & 1;
        const int pi = (w.kb0 + j) * kKeys / pt + i;
        const int page = pi < sl.n_pages ? pages[pi] : pages[0];  // beyond: masked
        const int blk = ((page * p.n_layers + p.layer) * p.n_heads + head) * 2 + kv;
        tma_load_2d(sKV + st * kStageBytes + kv * kKTile + h * kKvHalf + i * pt * 128, &tmap_k,
                    &kv_full[st], h * 64, blk * pt, pol);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ------------------------------------------------------------ UMMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(kRows, kKeys);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(kRows, kD) | (1u << 16);  // B MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int st = j % kStages;
        mbar_wait(&kv_full[st], (j / kStages) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sKV + st * kStageBytes);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          umma_bf16(tmem, umma_desc_sw128(q_addr + (kk >> 2) * kQHalf + (kk & 3) * 32),
                    umma_desc_sw128(k_addr + (kk >> 2) * kKvHalf + (kk & 3) * 32), idesc_s,
                    kk > 0 ? 1u : 0u);
        umma_commit(s_full);
      };
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) {
          mbar_wait(s_free, j & 1);  // S_j is in the softmax warps' registers
          issue_s(j + 1);
        }
        const int pb = j % kPBuf;
        mbar_wait(&p_full[pb], (j / kPBuf) & 1);
        tc_fence_after();
        const int st = j % kStages;
        const uint32_t v_addr = smem_u32(sKV + st * kStageBytes + kKTile);
        const uint32_t p_addr = smem_u32(sP + pb * kPTile);
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk)  // V: MN-major, d-halves 8 KB apart
          umma_bf16(tmem + kKeys, umma_desc_sw128(p_addr + kk * 32),
                    umma_desc_sw128_mn(v_addr + kk * 2048, kKvHalf, 1024), idesc_pv,
                    (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&o_done[pb]);
        umma_commit(&kv_empty[st]);
      }
    }
  } else {
    // -------------------------------------------------------------- softmax warps
    const int r = static_cast<int>(warp * 32 + lane);
    const int qp = qb.pos0 + r;
    const uint32_t t_lane = tmem + ((warp * 32) << 16);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      float s[kKeys];
#pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(t_lane + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(u[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      const int k0 = (w.kb0 + j) * kKeys;
      const int lim = min(qp, kv_end - 1);  // last key this row may see
      // Blocks entirely below every row's diagonal need no mask (warp-uniform).
      const bool full = __all_sync(0xffffffffu, k0 + kKeys - 1 <= lim);
      // 8 independent max chains (a single 64-long FMNMX chain is pure latency)
      float mxv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) mxv[q] = -INFINITY;
      if (full) {
#pragma unroll
        for (int c = 0; c < kKeys; ++c) mxv[c & 7] = fmaxf(mxv[c & 7], s[c]);
      } else {
#pragma unroll
        for (int c = 0; c < kKeys; ++c) {
          s[c] = (k0 + c <= lim) ? s[c] : -INFINITY;
          mxv[c & 7] = fmaxf(mxv[c & 7], s[c]);
        }
      }
      const float raw_mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                                 fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
      const float mx = raw_mx * p.scale_log2;  // scale > 0: max commutes
      float corr = 1.f;
      bool rescale = false;
      if (mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx != -INFINITY)) {
        corr = (m_used == -INFINITY) ? 0.f : exp2f(m_used - mx);
        m_used = mx;
        rescale = true;
      }
      l *= corr;
      const float base = (m_used == -INFINITY) ? 0.f : m_used;
      // P_j's buffer was last read by PV_{j-kPBuf}
      if (j >= kPBuf) {
        mbar_wait(&o_done[j % kPBuf], ((j / kPBuf) & 1) ^ 1);
        tc_fence_after();
      }
      uint8_t* prow = sP + (j % kPBuf) * kPTile + r * 128;
      float lsum[8];  // 8 independent accumulation chains
#pragma unroll
      for (int q = 0; q < 8; ++q) lsum[q] = 0.f;
#pragma unroll
      for (int c = 0; c < kKeys / 8; ++c) {
        float e[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float x = fmaf(s[c * 8 + t], p.scale_log2, -base);
          // 1 in 4 exponentials on the FMA pipe, the rest on MUFU (balanced issue)
          e[t] = ((c & 3) == 3) ? exp2_poly(x) : exp2f(x);
          lsum[t] += e[t];
        }
        uint4 pk;
        pk.x = pack_bf16x2(e[0], e[1]);
        pk.y = pack_bf16x2(e[2], e[3]);
        pk.z = pack_bf16x2(e[4], e[5]);
        pk.w = pack_bf16x2(e[6], e[7]);
        *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) = pk;
      }
      l += ((lsum[0] + lsum[1]) + (lsum[2] + lsum[3])) + ((lsum[4] + lsum[5]) + (lsum[6] + lsum[7]));
      // tcgen05.ld/st are warp-collective: rescale if any row of the warp needs it
      // (rows that do not need it multiply by corr == 1)
      if (__any_sync(0xffffffffu, rescale && j > 0)) {
        // O must hold PV_{j-1} before it is rescaled
        mbar_wait(&o_done[(j - 1) % kPBuf], ((j - 1) / kPBuf) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(t_lane + kKeys + c * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * corr);
          tmem_st_32x32b_x32(t_lane + kKeys + c * 32, u);
        }
        tmem_wait_st();
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j % kPBuf]);
    }
    // final O row
    mbar_wait(&o_done[(nblk - 1) % kPBuf], ((nblk - 1) / kPBuf) & 1);
    tc_fence_after();
    const int HD = p.n_heads * kD;
    if (qb.n_splits == 1) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* out = p.o + static_cast<size_t>(qb.row0 + r) * HD + head * kD;
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(t_lane + kKeys + c * 32, u);
        tmem_wait_ld();
        if (r < qb.nrows) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 pk;
            pk.x = pack_bf16x2(__uint_as_float(u[g * 8 + 0]) * inv, __uint_as_float(u[g * 8 + 1]) * inv);
            pk.y = pack_bf16x2(__uint_as_float(u[g * 8 + 2]) * inv, __uint_as_float(u[g * 8 + 3]) * inv);
            pk.z = pack_bf16x2(__uint_as_float(u[g * 8 + 4]) * inv, __uint_as_float(u[g * 8 + 5]) * inv);
            pk.w = pack_bf16x2(__uint_as_float(u[g * 8 + 6]) * inv, __uint_as_float(u[g * 8 + 7]) * inv);
            *reinterpret_cast<uint4*>(out + c * 32 + g * 8) = pk;
          }
        }
      }
    } else {
      float* dst = p.partial +
                   ((static_cast<size_t>(w.slot) * p.n_heads + head) * kRows + r) * (kD + 4);  // 16-byte aligned rows
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t u[32];
        tmem_ld_32x32b_x32(t_lane + kKeys + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<float4*>(dst + c * 32 + g * 4) =
              make_float4(__uint_as_float(u[g * 4]), __uint_as_float(u[g * 4 + 1]),
                          __uint_as_float(u[g * 4 + 2]), __uint_as_float(u[g * 4 + 3]));
      }
      dst[kD] = m_used;
      dst[kD + 1] = l;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc<256>(tmem);
}

int make_tmap_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows);
int make_tmap_kv_pages(CUtensorMap* map, const void* pool, uint64_t blocks, uint32_t page_tokens);

// Q rows live in the fused qkv buffer: a [rows, row_elems] map, 128 x 64 boxes.
static int make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t row_elems,
                          uint32_t box_rows) {
  return make_tmap_kmajor(map, base, rows, row_elems, box_rows);
}

int launch_chunk_attention_tc(const __nv_bfloat16* qkv, int q_rows, int q_stride,
                              __nv_bfloat16* o, const __nv_bfloat16* pool, int pool_pages,
                              KvGeom g, int layer, const AttnWork* work, int n_work,
                              const AttnQBlock* qblocks, int n_qblocks, bool any_split,
                              const tk_slice* slices_dev, const int32_t* bt_dev, float scale,
                              float* partial, cudaStream_t s) {
  TK_CHECK(g.head_dim == kD, TK_EUNSUPPORTED, "tcgen05 attention: head_dim 128");
  TK_CHECK(g.page_tokens == 16, TK_EUNSUPPORTED, "tcgen05 attention: 16-token pages");
  if (n_work == 0) return TK_OK;
  CUtensorMap tq, tk;
  int rc = make_tmap_rows(&tq, qkv, q_rows, q_stride, kRows);
  if (rc) return rc;
  const uint64_t blocks = static_cast<uint64_t>(pool_pages) * g.n_layers * g.n_heads * 2;
  rc = make_tmap_rows(&tk, pool, blocks * g.page_tokens, kD, g.page_tokens);
  if (rc) return rc;
  static bool cfg = false;
  if (!cfg) {
    TK_CUDA(cudaFuncSetAttribute(chunk_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmem));
    cfg = true;
  }
  TcAttnParams prm;
  prm.work = work;
  prm.qblocks = qblocks;
  prm.slices = slices_dev;
  prm.bt = bt_dev;
  prm.o = o;
  prm.partial = partial;
  prm.n_layers = g.n_layers;
  prm.n_heads = g.n_heads;
  prm.layer = layer;
  prm.page_tokens = g.page_tokens;
  prm.scale_log2 = scale * 1.4426950408889634f;
  chunk_attn_tc_kernel<<<dim3(n_work, g.n_heads), 192, kSmem, s>>>(tq, tk, prm);
  TK_CUDA(cudaGetLastError());
  note_launch();
  if (any_split) {
    rc = launch_attn_combine(o, qblocks, n_qblocks, g.n_heads, g.head_dim, partial, s);
    if (rc) return rc;
  }
  return TK_OK;
}

}  // namespace tk
