// attention_tc.cu -- chunked-prefill attention (K2) on 5th-gen tensor cores.
//
// One CTA = one head x one <=128-row query block x one KV split (128-key
// blocks).  Per block:  S = Q K^T  (UMMA 128x128x128 -> TMEM),  softmax by
// warps 0-3 with one query row per thread straight out of TMEM (no shuffles),
// P (bf16) written to shared memory in the UMMA K-major SW128 layout,
// O += P V  (UMMA, V as an MN-major operand -> TMEM).  K and V tiles are
// TMA-loaded page by page from the page-major KV pool (16-token pages are
// 2 KB-aligned [16][64] boxes per head-dim half), double buffered.
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

namespace tk {

namespace {
constexpr int kRows = 128;
constexpr int kKeys = 128;
constexpr int kD = 128;
constexpr int kTile = kRows * kD * 2;     // 32 KB: two SW128 atom columns of [128][64]
constexpr int kHalf = kTile / 2;          // 16 KB: one atom column
constexpr int kSmem = kTile * 6 + 1024 + 256;  // Q, K[2], V[2], P + barriers + align
constexpr float kRescaleThreshold = 8.f;  // log2 units
}  // namespace

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
                         const __grid_constant__ CUtensorMap tmap_kv, const TcAttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTile;          // [2]
  uint8_t* sV = smem + 3 * kTile;      // [2]
  uint8_t* sP = smem + 5 * kTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTile);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* s_free = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* o_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

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
    tma_prefetch_desc(&tmap_kv);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S at col 0, O at col 128

  if (warp == 4) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      const uint64_t pol = l2_policy_evict_first();
      mbar_expect_tx(q_full, kTile);
      for (int h = 0; h < 2; ++h)
        tma_load_2d(sQ + h * kHalf, &tmap_q, q_full, head * kD + h * 64, qb.row0, pol);
      const int pt = p.page_tokens;
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * kTile);
        const int first_page = (w.kb0 + j) * kKeys / pt;
        for (int i = 0; i < kKeys / pt; ++i) {
          const int pi = first_page + i;
          const int page = pi < sl.n_pages ? pages[pi] : pages[0];  // beyond: masked
          const int row_k = (((page * p.n_layers + p.layer) * 2 + 0) * p.n_heads + head) * pt;
          const int row_v = row_k + p.n_heads * pt;
          for (int h = 0; h < 2; ++h) {
            tma_load_2d(sK + st * kTile + h * kHalf + i * pt * 128, &tmap_kv, &kv_full[st],
                        h * 64, row_k, pol);
            tma_load_2d(sV + st * kTile + h * kHalf + i * pt * 128, &tmap_kv, &kv_full[st],
                        h * 64, row_v, pol);
          }
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ------------------------------------------------------------ UMMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(kRows, kKeys);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(kRows, kD) | (1u << 16);  // B MN-major
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * kTile);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
          umma_bf16(tmem, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_s,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
      };
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) {
          mbar_wait(s_free, j & 1);  // S_j is in the softmax warps' registers
          issue_s(j + 1);
        }
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const int st = j & 1;
        const uint32_t v_addr = smem_u32(sV + st * kTile);
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk) {
          const uint32_t a_off = (kk >> 2) * kHalf + (kk & 3) * 32;  // P: K = keys
          umma_bf16(tmem + kKeys, umma_desc_sw128(p_addr + a_off),
                    umma_desc_sw128_mn(v_addr + kk * 2048, kHalf, 1024), idesc_pv,
                    (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_done);
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
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kKeys; ++c) {
        const float v = (k0 + c <= lim) ? s[c] * p.scale_log2 : -INFINITY;
        s[c] = v;
        mx = fmaxf(mx, v);
      }
      float corr = 1.f;
      bool rescale = false;
      if (mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx != -INFINITY)) {
        corr = (m_used == -INFINITY) ? 0.f : exp2f(m_used - mx);
        m_used = mx;
        rescale = true;
      }
      l *= corr;
      const float base = (m_used == -INFINITY) ? 0.f : m_used;
      // P_{j-1} is still being read by PV_{j-1} and O is being written: wait
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
      }
      uint8_t* prow = sP + r * 128;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float e[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            e[t] = exp2f(s[a * 64 + c * 8 + t] - base);
            l += e[t];
          }
          uint4 pk;
          pk.x = pack_bf16x2(e[0], e[1]);
          pk.y = pack_bf16x2(e[2], e[3]);
          pk.z = pack_bf16x2(e[4], e[5]);
          pk.w = pack_bf16x2(e[6], e[7]);
          *reinterpret_cast<uint4*>(prow + a * kHalf + ((c ^ (r & 7)) << 4)) = pk;
        }
      }
      // tcgen05.ld/st are warp-collective: rescale if any row of the warp needs it
      // (rows that do not need it multiply by corr == 1)
      if (__any_sync(0xffffffffu, rescale && j > 0)) {
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
      if (lane == 0) mbar_arrive(p_full);
    }
    // final O row
    mbar_wait(o_done, (nblk - 1) & 1);
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
  TK_CHECK(kKeys % g.page_tokens == 0, TK_EUNSUPPORTED, "tcgen05 attention: page size");
  if (n_work == 0) return TK_OK;
  CUtensorMap tq, tkv;
  int rc = make_tmap_rows(&tq, qkv, q_rows, q_stride, kRows);
  if (rc) return rc;
  const uint64_t pool_rows =
      static_cast<uint64_t>(pool_pages) * g.n_layers * 2 * g.n_heads * g.page_tokens;
  rc = make_tmap_rows(&tkv, pool, pool_rows, kD, g.page_tokens);
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
  chunk_attn_tc_kernel<<<dim3(n_work, g.n_heads), 192, kSmem, s>>>(tq, tkv, prm);
  TK_CUDA(cudaGetLastError());
  note_launch();
  if (any_split) {
    rc = launch_attn_combine(o, qblocks, n_qblocks, g.n_heads, g.head_dim, partial, s);
    if (rc) return rc;
  }
  return TK_OK;
}

}  // namespace tk
