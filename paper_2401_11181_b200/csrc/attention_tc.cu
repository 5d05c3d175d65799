// attention_tc.cu -- chunked-prefill attention (K2) on 5th-gen tensor cores.
//
// Replaces the stand-in pdsim/costs.py:142-152 (chunk_cost) for the attention
// part of one chunk: every query row of a slice attends causally over its
// request's paged KV prefix (pdsim/prefill.py:140-165 defines the slices).
//
// Work unit = one head x one *pair* of 128-row query tiles of the same slice
// (rows r..r+255) x a range of 128-key blocks.  Both tiles share every K/V
// block that is staged in shared memory, which halves the L2->SM traffic per
// FLOP compared to one tile per CTA (at 128 rows per K/V tile the kernel is
// L2-bandwidth-bound long before the tensor core is busy).
//
// Persistent CTAs, one per SM (320 threads):
//   warps 0-3  softmax for tile 0, one query row per thread
//   warps 4-7  softmax for tile 1
//   warp  8    TMA producer: Q tiles, then K_j / V_j (2 KB [16 keys][64 d]
//              boxes, one per page and d-half) into a 4-entry 32 KB ring
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 columns): S_t at 128 t, O_t at 256 + 128 t.  S_t = Q_t K_j^T
// (UMMA 128x128x128); the softmax warps read S_t, write P_t (bf16, packed two
// per column) back over S_t with tcgen05.st, and O_t += P_t V_j reads P_t
// straight from TMEM (A operand in tensor memory), so P never touches shared
// memory.  The issue order S_0(j+1) after PV_0(j), then PV_1(j), S_1(j+1)
// ping-pongs the two tiles: while warps 0-3 exponentiate S_0, the tensor core
// runs tile 1's MMAs and vice versa.  tcgen05.mma ops of one thread execute
// in order, which makes "S_t(j+1) overwrites P_t(j)" safe after PV_t(j).
//
// Softmax: 128 scores per row per block, 3-input max (FMNMX3), packed fp32x2
// FMA/add (FFMA2/FADD2), 3/4 of the exponentials on MUFU.EX2 and 1/4 by a
// polynomial on the FMA pipe (MUFU throughput would otherwise equal the
// tensor time).  O is rescaled lazily, only when a row maximum grows by more
// than 2^8 (exp2 domain); the final normalisation uses the same stale maximum,
// so results are exact up to fp32 rounding.
//
// Load balance: the (head, pair, key block) space is split stream-K style
// into equal contiguous ranges, one per CTA; a (head, pair) cut by a range
// boundary is computed as pieces whose unnormalised partials (O, m, l) are
// merged by fa_combine_kernel.
#include "tk_common.cuh"
#include "tk_kernels.h"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace tk {

namespace {
constexpr int kRows = 128;                 // query rows per tile
constexpr int kKeys = 128;                 // keys per KV block
constexpr int kD = 128;
constexpr int kRing = 4;                   // K/V ring entries (K_j and V_j alternate)
constexpr int kQTile = kRows * kD * 2;     // 32 KB: Q as two SW128 atom columns [128][64]
constexpr int kQHalf = kQTile / 2;
constexpr int kKvHalf = kKeys * 128;       // 16 KB: one d-half of a K or V block
constexpr int kEntry = 2 * kKvHalf;        // 32 KB
constexpr int kBarBytes = 256;
constexpr int kSmem = 2 * kQTile + kRing * kEntry + kBarBytes + 1024;
constexpr int kThreads = 320;
constexpr float kRescaleThreshold = 8.f;  // log2 units
// partial row (bytes): unnormalised O[128] as bf16 (relative precision is what bf16
// keeps, magnitude-independent), then m, l as fp32; 16-byte aligned rows
constexpr int kPartRowBytes = kD * 2 + 16;
constexpr int kMinBlocksPerCta = 2;
}  // namespace

int64_t fa_partial_bytes() {
  return static_cast<int64_t>(kFaMaxPieces) * 2 * kRows * kPartRowBytes;
}

// ------------------------------------------------------------ fp32x2 helpers
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a pair on the FMA pipe: x = n + f (|f| <= 1/2, magic-constant
// rounding), 2^f by a degree-5 polynomial (rel. err < 3e-6), 2^n added to the
// exponent field.  x is clamped at -127 so masked (-inf) scores give ~0.
template <int DEG = 5>
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& e0, float& e1) {
  x0 = fmaxf(x0, -127.f);
  x1 = fmaxf(x1, -127.f);
  const uint64_t magic = f2(12582912.f, 12582912.f);
  const uint64_t nmagic = f2(-12582912.f, -12582912.f);
  const uint64_t x = f2(x0, x1);
  const uint64_t y = f2_add(x, magic);
  const uint64_t n = f2_add(y, nmagic);
  float n0, n1;
  f2_split(n, n0, n1);
  const uint64_t f = f2_add(x, f2(-n0, -n1));
  uint64_t q;
  if constexpr (DEG >= 5) {
    q = f2(1.3333558e-3f, 1.3333558e-3f);
    q = f2_fma(q, f, f2(9.6181291e-3f, 9.6181291e-3f));
    q = f2_fma(q, f, f2(5.5504109e-2f, 5.5504109e-2f));
    q = f2_fma(q, f, f2(2.4022651e-1f, 2.4022651e-1f));
    q = f2_fma(q, f, f2(6.9314718e-1f, 6.9314718e-1f));
    q = f2_fma(q, f, f2(1.0f, 1.0f));
  } else {
    // degree 3 on |f| <= 1/2: rel. err < 1e-4, well below bf16 P rounding (3.9e-3)
    q = f2(5.5855685e-2f, 5.5855685e-2f);
    q = f2_fma(q, f, f2(2.4017581e-1f, 2.4017581e-1f));
    q = f2_fma(q, f, f2(6.9304585e-1f, 6.9304585e-1f));
    q = f2_fma(q, f, f2(1.0000041f, 1.0000041f));
  }
  float q0, q1, y0, y1;
  f2_split(q, q0, q1);
  f2_split(y, y0, y1);
  e0 = __int_as_float(__float_as_int(q0) + ((__float_as_int(y0) - 0x4B400000) << 23));
  e1 = __int_as_float(__float_as_int(q1) + ((__float_as_int(y1) - 0x4B400000) << 23));
}

// Timing trace of CTA 0 (TK_FA_VARIANT=7 only): clock64 stamps per pipeline
// event and block, read back by tk_debug_fa_trace (scripts/attn_trace.py).
__device__ unsigned long long g_fa_trace[10 * 2 * 512];
__device__ __forceinline__ void fa_stamp(int kind, int t, int j) {
  if (blockIdx.x == 0 && j < 512) g_fa_trace[(kind * 2 + t) * 512 + j] = clock64();
}

struct FaParams {
  const FaPair* pairs;
  const FaUnit* units;
  const int32_t* cta_off;
  const tk_slice* slices;
  const int32_t* bt;
  __nv_bfloat16* o;
  float* partial;
  int n_layers, n_heads, layer;
  float scale_log2;
};

struct UnitView {
  FaPair pr;
  int head, kb0, nblk, piece;
  int n[2];        // key blocks of this unit each tile computes (tile 0 may stop early)
  int kv_end[2];   // keys [0, kv_end) exist for the tile's last row
};

__device__ __forceinline__ UnitView unit_view(const FaParams& p, int u) {
  const FaUnit un = p.units[u];
  UnitView v;
  v.pr = p.pairs[un.pair];
  v.head = un.head;
  v.kb0 = un.kb0;
  v.nblk = un.kb1 - un.kb0;
  v.piece = un.piece;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int nrows = t ? v.pr.nrows1 : v.pr.nrows0;
    v.kv_end[t] = v.pr.pos0 + t * kRows + nrows;
    const int nb = nrows > 0 ? (v.kv_end[t] + kKeys - 1) / kKeys : 0;
    v.n[t] = max(0, min(nb - v.kb0, v.nblk));
  }
  return v;
}

// D = head_dim: 128 (OPT-13B, Llama-2-7B) or 64 (the OPT-125M-class length
// predictor and tiny decoder): a 64-wide head is one SW128 atom column of Q/K/V,
// so its S MMA is K=64 (4 UMMAs) and O_t uses 64 TMEM columns; the K/V ring
// keeps the same 128 KB as 8 entries of 16 KB.
template <int D, int POLY, bool LD_BATCH, int EXP = 0, int DEG = 5>
__global__ void __launch_bounds__(kThreads, 1)
    chunk_attn_fa_kernel(const __grid_constant__ CUtensorMap tmap_q,
                         const __grid_constant__ CUtensorMap tmap_kv, const FaParams p) {
  static_assert(D == 128 || D == 64, "tcgen05 attention: head_dim 128 or 64");
  constexpr int kD = D;                          // (shadow the 128-wide defaults)
  constexpr int kHalves = D / 64;                // 64-wide SW128 atom columns
  constexpr int kQTile = kRows * D * 2;
  constexpr int kQHalf = kRows * 128;            // stride between Q atom columns
  constexpr int kEntry = kHalves * kKvHalf;
  constexpr int kRing = (4 * 2 * kKvHalf) / kEntry;
  constexpr int kPartRowBytes = D * 2 + 16;
  griddep_launch();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                       // [tile][2 d-halves][128 rows][128 B]
  uint8_t* sKV = smem + 2 * kQTile;         // [kRing][2 d-halves][128 keys][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kRing * kEntry);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;             // [kRing]
  uint64_t* kv_empty = kv_full + kRing;     // [kRing]
  uint64_t* s_full = kv_empty + kRing;      // [2] S_t in TMEM
  uint64_t* p_full = s_full + 2;            // [2] P_t in TMEM (4 warps)
  uint64_t* o_full = p_full + 2;            // [2] last PV_t of the unit retired
  uint64_t* o_free = o_full + 2;            // [2] O_t read out (4 warps)
  uint64_t* p_half = o_free + 2;            // [2] first 64 keys of P_t in TMEM (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_half + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_kv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
      mbar_init(&p_half[t], 4);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_free[t], 4);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // Q rows and K/V pages come from the QKV GEMM (PDL launch)
  const uint32_t tmem = *tmem_slot;
  const int u_begin = p.cta_off[blockIdx.x], u_end = p.cta_off[blockIdx.x + 1];

  if (warp == 8) {
    // ------------------------------------------------------------ producer warp
    // lane 0 owns the barriers; lanes 0-15 each issue one 2 KB box per K or V
    // block: page i = lane/2 of the block's 8 pages, d-half h = lane%2.
    const uint64_t pol_q = l2_policy_evict_first();
    const uint64_t pol_kv = l2_policy_evict_last();  // re-read by the other pairs of the head
    int ent = 0, uc = 0;
    for (int u = u_begin; u < u_end; ++u, ++uc) {
      const UnitView v = unit_view(p, u);
      const tk_slice sl = p.slices[v.pr.slice];
      const int32_t* pages = p.bt + sl.bt_offset;
      if (lane == 0) {
        mbar_wait(q_empty, (uc & 1) ^ 1);
        const bool two = v.pr.nrows1 > 0;
        mbar_expect_tx(q_full, two ? 2 * kQTile : kQTile);
        for (int t = 0; t < (two ? 2 : 1); ++t)
          for (int h = 0; h < kHalves; ++h)
            tma_load_2d(sQ + t * kQTile + h * kQHalf, &tmap_q, q_full, v.head * kD + h * 64,
                        v.pr.row0 + t * kRows, pol_q);
      }
      // lanes 0 .. 8*kHalves-1: page i of the block's 8, d-half h
      const int i = (lane / kHalves) & 7, h = lane % kHalves;
      constexpr int kLoadLanes = 8 * kHalves;
      auto page_of = [&](int kb) {
        const int pi = kb * (kKeys / 16) + i;
        return pi < sl.n_pages ? __ldg(pages + pi) : __ldg(pages);  // beyond: masked keys
      };
      int pg_next = lane < kLoadLanes ? page_of(v.kb0) : 0;
      for (int j = 0; j < v.nblk; ++j) {
        const int pg = pg_next;
        if (lane < kLoadLanes && j + 1 < v.nblk) pg_next = page_of(EXP == 2 ? v.kb0 : v.kb0 + j + 1);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ent) {
          const int st = ent % kRing;
          if (lane == 0) {
            mbar_wait(&kv_empty[st], ((ent / kRing) & 1) ^ 1);
            mbar_expect_tx(&kv_full[st], kEntry);
            if constexpr (EXP >= 3) fa_stamp(5 + kv, 0, ent / 2);
          }
          __syncwarp();
          if (lane < kLoadLanes) {
            const int blk = ((pg * p.n_layers + p.layer) * p.n_heads + v.head) * 2 + kv;
            tma_load_2d(sKV + st * kEntry + h * kKvHalf + i * 16 * 128, &tmap_kv, &kv_full[st],
                        h * 64, blk * 16, pol_kv);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ UMMA issuer
    // The whole warp runs the loop (converged, so descriptors and counters are
    // warp-uniform and feed tcgen05.mma from uniform registers directly); one
    // elected lane issues every tcgen05 operation.
    constexpr uint32_t idesc_s = umma_idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_pv = umma_idesc_bf16(kRows, kD) | (1u << 16);  // B MN-major
    const uint64_t q_desc[2] = {umma_desc_sw128(smem_u32(sQ)), umma_desc_sw128(smem_u32(sQ + kQTile))};
    const uint32_t kv_base = smem_u32(sKV);
    int ent = 0, uc = 0;
    uint32_t pc[2] = {0, 0}, oc[2] = {0, 0};
    for (int u = u_begin; u < u_end; ++u, ++uc) {
      const UnitView v0 = unit_view(p, u);
      const int nblk = __shfl_sync(0xffffffffu, v0.nblk, 0);
      const int nt[2] = {__shfl_sync(0xffffffffu, v0.n[0], 0), __shfl_sync(0xffffffffu, v0.n[1], 0)};
      mbar_wait(q_full, uc & 1);
      tc_fence_after();
      auto entry_addr = [&](int e) {
        const int st = e % kRing;
        mbar_wait(&kv_full[st], (e / kRing) & 1);
        tc_fence_after();
        return kv_base + st * kEntry;
      };
      auto issue_s = [&](int t, uint32_t k_addr) {
        if (elect_one_sync()) {
          if constexpr (D == 128)
            umma_bf16_k128<kQHalf / 16, kKvHalf / 16>(tmem + t * 128, q_desc[t],
                                                       umma_desc_sw128(k_addr), idesc_s, 0u);
          else
            umma_bf16_k64(tmem + t * 128, q_desc[t], umma_desc_sw128(k_addr), idesc_s, 0u);
          umma_commit(&s_full[t]);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one_sync()) umma_commit(bar);
        __syncwarp();
      };
      // block 0: S_0(0), S_1(0)
      {
        const uint32_t k_addr = entry_addr(ent);
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (nt[t] > 0) issue_s(t, k_addr);
        commit(&kv_empty[ent % kRing]);
        if (nblk == 1) commit(q_empty);
      }
      for (int j = 0; j < nblk; ++j) {
        const int ek = ent + 2 * j, ev = ek + 1, ek_next = ek + 2;
        uint32_t v_addr = 0, k_next = 0;
        bool have_v = false, have_k = false;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j >= nt[t]) continue;
          // PV_t(j) in two halves: keys 0-63 as soon as the softmax warps
          // have stored that half of P_t, keys 64-127 after the rest
          mbar_wait(&p_half[t], pc[t] & 1);
          tc_fence_after();
          if constexpr (EXP >= 3) {
            if (lane == 0) fa_stamp(2, t, ent / 2 + j);
          }
          if (j == 0) {
            mbar_wait(&o_free[t], (oc[t] & 1) ^ 1);
            ++oc[t];
            tc_fence_after();
          }
          if (!have_v) {
            v_addr = entry_addr(ev);
            have_v = true;
          }
          // V: MN-major, d-halves 16 KB apart, 16 keys (2 KB) per K step
          const uint64_t v_desc = umma_desc_sw128_mn(v_addr, kKvHalf, 1024);
          if (elect_one_sync())
            umma_bf16_ts_k64(tmem + 256 + t * 128, tmem + t * 128, v_desc, idesc_pv,
                             j > 0 ? 1u : 0u);
          __syncwarp();
          mbar_wait(&p_full[t], pc[t] & 1);
          ++pc[t];
          tc_fence_after();
          if (elect_one_sync())
            umma_bf16_ts_k64(tmem + 256 + t * 128, tmem + t * 128 + 32, v_desc + 512, idesc_pv,
                             1u);
          __syncwarp();
          if constexpr (EXP >= 3) {
            if (lane == 0) fa_stamp(3, t, ent / 2 + j);
          }
          if (j == nt[t] - 1) commit(&o_full[t]);
          if (j + 1 < nt[t]) {
            if (!have_k) {
              k_next = entry_addr(ek_next);
              have_k = true;
            }
            issue_s(t, k_next);
            if constexpr (EXP >= 3) {
              if (lane == 0) fa_stamp(4, t, ent / 2 + j);
            }
          }
        }
        commit(&kv_empty[ev % kRing]);
        if (j + 1 < nblk) commit(&kv_empty[ek_next % kRing]);
        if (j + 2 == nblk) commit(q_empty);  // the unit's last S has been issued
      }
      ent += 2 * nblk;
    }
  } else {
    // -------------------------------------------------------------- softmax warps
    const int t = static_cast<int>(warp >> 2);
    const int r = static_cast<int>((warp & 3) * 32 + lane);
    const uint32_t t_lane = tmem + (((warp & 3) * 32) << 16);
    const uint32_t t_s = t_lane + t * 128;
    const uint32_t t_o = t_lane + 256 + t * 128;
    const int HD = p.n_heads * kD;
    const float sc = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    int blk_cnt = 0;  // key blocks of earlier units (trace index)
    for (int u = u_begin; u < u_end; blk_cnt += unit_view(p, u).nblk, ++u) {
      const UnitView v = unit_view(p, u);
      const int nrows = t ? v.pr.nrows1 : v.pr.nrows0;
      const int n_t = t ? v.n[1] : v.n[0];
      const int kv_end_t = t ? v.kv_end[1] : v.kv_end[0];
      if (n_t == 0) {
        if (v.piece >= 0 && nrows > 0) {  // nothing visible in this piece: empty partial
          uint8_t* dst = reinterpret_cast<uint8_t*>(p.partial) +
                         ((static_cast<size_t>(v.piece) * 2 + t) * kRows + r) * kPartRowBytes;
          for (int c = 0; c < kD * 2; c += 16)
            *reinterpret_cast<uint4*>(dst + c) = make_uint4(0u, 0u, 0u, 0u);
          reinterpret_cast<float*>(dst + kD * 2)[0] = -INFINITY;
          reinterpret_cast<float*>(dst + kD * 2)[1] = 0.f;
        }
        continue;
      }
      const int qp = v.pr.pos0 + t * kRows + r;
      const int lim = min(qp, kv_end_t - 1);  // last key this row may see
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_t; ++j) {
        mbar_wait(&s_full[t], s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        if constexpr (EXP >= 3) {
          if ((warp & 3) == 0 && lane == 0) fa_stamp(0, t, blk_cnt + j);
        }
        if constexpr (EXP == 1 || EXP == 4) {  // timing experiment: no softmax work at all
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&p_half[t]);
            mbar_arrive(&p_full[t]);
          }
          continue;
        }
        float s[kKeys];
        if constexpr (LD_BATCH) {
          uint32_t w[kKeys];
#pragma unroll
          for (int c = 0; c < kKeys / 32; ++c)
            tmem_ld_32x32b_x32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(w + c * 32));
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < kKeys; ++e) s[e] = __uint_as_float(w[e]);
        } else {
#pragma unroll
          for (int c = 0; c < kKeys / 32; ++c) {
            uint32_t w[32];
            tmem_ld_32x32b_x32(t_s + c * 32, w);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(w[e]);
          }
        }
        const int k0 = (v.kb0 + j) * kKeys;
        // blocks entirely below every row's diagonal need no mask (warp-uniform)
        if (!__all_sync(0xffffffffu, k0 + kKeys - 1 <= lim)) {
#pragma unroll
          for (int c = 0; c < kKeys; ++c) s[c] = (k0 + c <= lim) ? s[c] : -INFINITY;
        }
        float mx4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mx4[q] = fmax3(s[2 * q], s[2 * q + 1], -INFINITY);
#pragma unroll
        for (int c = 8; c < kKeys; c += 8) {
#pragma unroll
          for (int q = 0; q < 4; ++q) mx4[q] = fmax3(mx4[q], s[c + 2 * q], s[c + 2 * q + 1]);
        }
        const float raw_mx = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]);
        const float mx = raw_mx * sc;  // scale > 0: max commutes
        float corr = 1.f;
        bool rescale = false;
        if (mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx != -INFINITY)) {
          corr = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
          m_used = mx;
          rescale = true;
        }
        l *= corr;
        // tcgen05.ld/st are warp-collective: rescale if any row of the warp needs it.
        // S_t(j) retired => PV_t(j-1) retired (in-order), so O_t is final here.
        if (__any_sync(0xffffffffu, rescale && j > 0)) {
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t w[32];
            tmem_ld_32x32b_x32(t_o + c * 32, w);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(__uint_as_float(w[e]) * corr);
            tmem_st_32x32b_x32(t_o + c * 32, w);
          }
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const uint64_t sc2 = f2(sc, sc), nb2 = f2(-base, -base);
        uint64_t sum2[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int k = c * 32 + 2 * i;
            float x0, x1, e0, e1;
            f2_split(f2_fma(f2(s[k], s[k + 1]), sc2, nb2), x0, x1);
            if (POLY > 0 && (i % (POLY > 0 ? POLY : 1)) == POLY - 1) {
              exp2_poly2<DEG>(x0, x1, e0, e1);
            } else {
              e0 = ex2(x0);
              e1 = ex2(x1);
            }
            sum2[i & 1] = f2_add(sum2[i & 1], f2(e0, e1));
            pk[i] = pack_bf16x2(e0, e1);
          }
          tmem_st_32x32b_x16(t_s + c * 16, pk);
          if (c == 1) {  // keys 0-63 of P_t are in TMEM: the first PV half may start
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_half[t]);
          }
        }
        float a0, a1, b0, b1;
        f2_split(sum2[0], a0, a1);
        f2_split(sum2[1], b0, b1);
        l += (a0 + a1) + (b0 + b1);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if constexpr (EXP >= 3) {
          if ((warp & 3) == 0 && lane == 0) fa_stamp(1, t, blk_cnt + j);
        }
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // ---- epilogue: O_t -> bf16 rows (or an unnormalised partial)
      mbar_wait(&o_full[t], o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      if (v.piece < 0) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        __nv_bfloat16* out =
            p.o + static_cast<size_t>(v.pr.row0 + t * kRows + r) * HD + v.head * kD;
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_o + c * 32, w);
          tmem_wait_ld();
          if (r < nrows) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              uint4 pk;
              pk.x = pack_bf16x2(__uint_as_float(w[g * 8 + 0]) * inv, __uint_as_float(w[g * 8 + 1]) * inv);
              pk.y = pack_bf16x2(__uint_as_float(w[g * 8 + 2]) * inv, __uint_as_float(w[g * 8 + 3]) * inv);
              pk.z = pack_bf16x2(__uint_as_float(w[g * 8 + 4]) * inv, __uint_as_float(w[g * 8 + 5]) * inv);
              pk.w = pack_bf16x2(__uint_as_float(w[g * 8 + 6]) * inv, __uint_as_float(w[g * 8 + 7]) * inv);
              *reinterpret_cast<uint4*>(out + c * 32 + g * 8) = pk;
            }
          }
        }
      } else {
        uint8_t* dst = reinterpret_cast<uint8_t*>(p.partial) +
                       ((static_cast<size_t>(v.piece) * 2 + t) * kRows + r) * kPartRowBytes;
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_o + c * 32, w);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 pk;
            pk.x = pack_bf16x2(__uint_as_float(w[g * 8 + 0]), __uint_as_float(w[g * 8 + 1]));
            pk.y = pack_bf16x2(__uint_as_float(w[g * 8 + 2]), __uint_as_float(w[g * 8 + 3]));
            pk.z = pack_bf16x2(__uint_as_float(w[g * 8 + 4]), __uint_as_float(w[g * 8 + 5]));
            pk.w = pack_bf16x2(__uint_as_float(w[g * 8 + 6]), __uint_as_float(w[g * 8 + 7]));
            *reinterpret_cast<uint4*>(dst + c * 64 + g * 16) = pk;
          }
        }
        reinterpret_cast<float*>(dst + kD * 2)[0] = m_used;
        reinterpret_cast<float*>(dst + kD * 2)[1] = l;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------ CTA-pair kernel
// cta_group::2 form (head_dim 128).  A cluster of two CTAs computes one unit
// (head, 512-row quad of a slice, key range) as two 256-row super-tiles t = 0, 1;
// CTA c owns rows 256 t + 128 c .. + 127 of super-tile t (its two Q tiles, its
// S_t / O_t in its own TMEM), keys 64 c .. 64 c + 63 of every K block and d-half
// c of every V block.  The even CTA issues S_t = Q_t K^T and O_t += P_t V as
// M=256 pair MMAs (each CTA's TMEM receives its 128 rows x all 128 columns; P
// is read from both CTAs' TMEM).  Per SM and 128-key block the shared-memory
// traffic falls from 256 KB (S operands 128 KB, V 64 KB, K/V fills 64 KB) to
// 160 KB (96 + 32 + 32): the single-CTA kernel's S MMA reads both operands at
// the 128 B/clk shared-memory port limit (profiles/r01_attn_pipeline.md).
// Softmax, lazy rescale and the epilogue are those of chunk_attn_fa_kernel;
// the P / O-free handshakes arrive on the even CTA's barriers (8 warps).
namespace {
constexpr int kPairKvEntry = kKvHalf;                // 16 KB per CTA: K keys-half or V d-half
constexpr int kPairRing = 8;
constexpr int kPairSmem = 2 * kQTile + kPairRing * kPairKvEntry + kBarBytes + 1024;
constexpr int kQuadRows = 4 * kRows;
}  // namespace

struct QuadView {
  FaPair pr;
  int head, kb0, nblk, piece;
  int n[2];        // key blocks super-tile t computes
  int kv_end[2];   // keys [0, kv_end) exist for super-tile t's last row
};

__device__ __forceinline__ QuadView quad_view(const FaParams& p, int u) {
  const FaUnit un = p.units[u];
  QuadView v;
  v.pr = p.pairs[un.pair];
  v.head = un.head;
  v.kb0 = un.kb0;
  v.nblk = un.kb1 - un.kb0;
  v.piece = un.piece;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int rows = max(0, min(2 * kRows, v.pr.nrows0 - t * 2 * kRows));
    v.kv_end[t] = v.pr.pos0 + t * 2 * kRows + rows;
    const int nb = rows > 0 ? (v.kv_end[t] + kKeys - 1) / kKeys : 0;
    v.n[t] = max(0, min(nb - v.kb0, v.nblk));
  }
  return v;
}

template <int POLY = 4, int DEG = 3>  // 1 of POLY exponential pairs on the FMA pipe
__global__ void __launch_bounds__(kThreads, 1)
    chunk_attn_fa_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                              const __grid_constant__ CUtensorMap tmap_kv, const FaParams p) {
  griddep_launch();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                       // [super-tile][2 d-halves][128 rows][128 B]
  uint8_t* sKV = smem + 2 * kQTile;         // [kPairRing][16 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kPairRing * kPairKvEntry);
  uint64_t* q_full = bars;                  // even CTA: both CTAs' Q bytes
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;             // [kPairRing] even CTA: both CTAs' bytes
  uint64_t* kv_empty = kv_full + kPairRing; // [kPairRing]
  uint64_t* s_full = kv_empty + kPairRing;  // [2]
  uint64_t* p_full = s_full + 2;            // [2] even CTA: 4 warps x 2 CTAs
  uint64_t* o_full = p_full + 2;            // [2]
  uint64_t* o_free = o_full + 2;            // [2] even CTA: 4 warps x 2 CTAs
  uint64_t* p_half = o_free + 2;            // [2] even CTA: 4 warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_half + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int c = static_cast<int>(cluster_ctarank());
  const bool leader = c == 0;
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_kv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kPairRing; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 8);
      mbar_init(&p_half[t], 8);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_free[t], 8);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  griddep_wait();  // Q rows and K/V pages come from the QKV GEMM (PDL launch)
  const uint32_t tmem = *tmem_slot;
  const int cl = static_cast<int>(blockIdx.x >> 1);
  const int u_begin = p.cta_off[cl], u_end = p.cta_off[cl + 1];

  if (warp == 8) {
    // ------------------------------------------------------------ producer warp
    // Both CTAs load their own operands; the TMA completes on the even CTA's
    // full barriers, whose expected bytes the even CTA's lane 0 posts.
    const uint64_t pol_q = l2_policy_evict_first();
    const uint64_t pol_kv = l2_policy_evict_last();
    int ent = 0, uc = 0;
    for (int u = u_begin; u < u_end; ++u, ++uc) {
      const QuadView v = quad_view(p, u);
      const tk_slice sl = p.slices[v.pr.slice];
      const int32_t* pages = p.bt + sl.bt_offset;
      if (lane == 0) {
        mbar_wait(q_empty, (uc & 1) ^ 1);
        const int ntile = v.n[1] > 0 || v.pr.nrows0 > 2 * kRows ? 2 : 1;
        if (leader) mbar_expect_tx(q_full, 2 * ntile * kQTile);
        for (int t = 0; t < ntile; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_2d_pair(sQ + t * kQTile + h * kQHalf, &tmap_q, q_full, v.head * kD + h * 64,
                             v.pr.row0 + t * 2 * kRows + c * kRows, pol_q);
      }
      // lanes 0-7: K box (page 4c + lane/2 of the block, d-half lane%2); V box (page
      // lane, d-half c)
      auto page_of = [&](int pi) {
        return pi < sl.n_pages ? __ldg(pages + pi) : __ldg(pages);  // beyond: masked keys
      };
      const int ki = lane >> 1, kh = lane & 1;
      int kpg_next = 0, vpg_next = 0;
      if (lane < 8) {
        kpg_next = page_of(v.kb0 * 8 + 4 * c + ki);
        vpg_next = page_of(v.kb0 * 8 + static_cast<int>(lane));
      }
      for (int j = 0; j < v.nblk; ++j) {
        const int kpg = kpg_next, vpg = vpg_next;
        if (lane < 8 && j + 1 < v.nblk) {
          kpg_next = page_of((v.kb0 + j + 1) * 8 + 4 * c + ki);
          vpg_next = page_of((v.kb0 + j + 1) * 8 + static_cast<int>(lane));
        }
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++ent) {
          const int st = ent % kPairRing;
          if (lane == 0) {
            mbar_wait(&kv_empty[st], ((ent / kPairRing) & 1) ^ 1);
            if (leader) mbar_expect_tx(&kv_full[st], 2 * kPairKvEntry);
          }
          __syncwarp();
          if (lane < 8) {
            const int pg = kv ? vpg : kpg;
            const int blk = ((pg * p.n_layers + p.layer) * p.n_heads + v.head) * 2 + kv;
            uint8_t* dst = kv ? sKV + st * kPairKvEntry + lane * 16 * 128
                              : sKV + st * kPairKvEntry + kh * (kPairKvEntry / 2) + ki * 16 * 128;
            tma_load_2d_pair(dst, &tmap_kv, &kv_full[st], (kv ? c : kh) * 64, blk * 16, pol_kv);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ UMMA issuer
    if (leader) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(2 * kRows, kKeys);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(2 * kRows, kD) | (1u << 16);  // B MN-major
      const uint64_t q_desc[2] = {umma_desc_sw128(smem_u32(sQ)), umma_desc_sw128(smem_u32(sQ + kQTile))};
      const uint32_t kv_base = smem_u32(sKV);
      constexpr uint16_t kBoth = 3;
      int ent = 0, uc = 0;
      uint32_t pc[2] = {0, 0}, oc[2] = {0, 0};
      for (int u = u_begin; u < u_end; ++u, ++uc) {
        const QuadView v0 = quad_view(p, u);
        const int nblk = __shfl_sync(0xffffffffu, v0.nblk, 0);
        const int nt[2] = {__shfl_sync(0xffffffffu, v0.n[0], 0), __shfl_sync(0xffffffffu, v0.n[1], 0)};
        mbar_wait(q_full, uc & 1);
        tc_fence_after();
        auto entry_addr = [&](int e) {
          const int st = e % kPairRing;
          mbar_wait(&kv_full[st], (e / kPairRing) & 1);
          tc_fence_after();
          return kv_base + st * kPairKvEntry;
        };
        auto issue_s = [&](int t, uint32_t k_addr) {
          if (elect_one_sync()) {
            umma_bf16_pair_k128<kQHalf / 16, (kPairKvEntry / 2) / 16>(
                tmem + t * 128, q_desc[t], umma_desc_sw128(k_addr), idesc_s, 0u);
            umma_commit_pair_mc(&s_full[t], kBoth);
          }
          __syncwarp();
        };
        auto commit = [&](uint64_t* bar) {
          if (elect_one_sync()) umma_commit_pair_mc(bar, kBoth);
          __syncwarp();
        };
        {
          const uint32_t k_addr = entry_addr(ent);
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (nt[t] > 0) issue_s(t, k_addr);
          commit(&kv_empty[ent % kPairRing]);
          if (nblk == 1) commit(q_empty);
        }
        for (int j = 0; j < nblk; ++j) {
          const int ek = ent + 2 * j, ev = ek + 1, ek_next = ek + 2;
          uint32_t v_addr = 0, k_next = 0;
          bool have_v = false, have_k = false;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (j >= nt[t]) continue;
            mbar_wait(&p_half[t], pc[t] & 1);
            tc_fence_after();
            if (j == 0) {
              mbar_wait(&o_free[t], (oc[t] & 1) ^ 1);
              ++oc[t];
              tc_fence_after();
            }
            if (!have_v) {
              v_addr = entry_addr(ev);
              have_v = true;
            }
            // V: MN-major, this CTA's d-half (one 128-byte atom column), 16 keys per K step
            const uint64_t v_desc = umma_desc_sw128_mn(v_addr, kKvHalf, 1024);
            if (elect_one_sync())
              umma_bf16_pair_ts_k64(tmem + 256 + t * 128, tmem + t * 128, v_desc, idesc_pv,
                                    j > 0 ? 1u : 0u);
            __syncwarp();
            mbar_wait(&p_full[t], pc[t] & 1);
            ++pc[t];
            tc_fence_after();
            if (elect_one_sync())
              umma_bf16_pair_ts_k64(tmem + 256 + t * 128, tmem + t * 128 + 32, v_desc + 512,
                                    idesc_pv, 1u);
            __syncwarp();
            if (j == nt[t] - 1) commit(&o_full[t]);
            if (j + 1 < nt[t]) {
              if (!have_k) {
                k_next = entry_addr(ek_next);
                have_k = true;
              }
              issue_s(t, k_next);
            }
          }
          commit(&kv_empty[ev % kPairRing]);
          if (j + 1 < nblk) commit(&kv_empty[ek_next % kPairRing]);
          if (j + 2 == nblk) commit(q_empty);
        }
        ent += 2 * nblk;
      }
    }
  } else {
    // -------------------------------------------------------------- softmax warps
    const int t = static_cast<int>(warp >> 2);
    const int r = static_cast<int>((warp & 3) * 32 + lane);
    const uint32_t t_lane = tmem + (((warp & 3) * 32) << 16);
    const uint32_t t_s = t_lane + t * 128;
    const uint32_t t_o = t_lane + 256 + t * 128;
    const int HD = p.n_heads * kD;
    const float sc = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    for (int u = u_begin; u < u_end; ++u) {
      const QuadView v = quad_view(p, u);
      const int sub = 2 * t + c;  // this CTA's 128-row sub-tile of the quad
      const int nrows = max(0, min(kRows, v.pr.nrows0 - sub * kRows));
      const int n_t = v.n[t];
      if (n_t == 0) {
        if (v.piece >= 0 && nrows > 0) {  // nothing visible in this piece: empty partial
          uint8_t* dst = reinterpret_cast<uint8_t*>(p.partial) +
                         ((static_cast<size_t>(v.piece) * 4 + sub) * kRows + r) * kPartRowBytes;
          for (int e = 0; e < kD * 2; e += 16)
            *reinterpret_cast<uint4*>(dst + e) = make_uint4(0u, 0u, 0u, 0u);
          reinterpret_cast<float*>(dst + kD * 2)[0] = -INFINITY;
          reinterpret_cast<float*>(dst + kD * 2)[1] = 0.f;
        }
        continue;
      }
      const int qp = v.pr.pos0 + sub * kRows + r;
      const int lim = min(qp, v.kv_end[t] - 1);  // last key this row may see
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_t; ++j) {
        mbar_wait(&s_full[t], s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        float s[kKeys];
#pragma unroll
        for (int q = 0; q < kKeys / 32; ++q) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_s + q * 32, w);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) s[q * 32 + e] = __uint_as_float(w[e]);
        }
        const int k0 = (v.kb0 + j) * kKeys;
        if (!__all_sync(0xffffffffu, k0 + kKeys - 1 <= lim)) {
#pragma unroll
          for (int e = 0; e < kKeys; ++e) s[e] = (k0 + e <= lim) ? s[e] : -INFINITY;
        }
        float mx4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mx4[q] = fmax3(s[2 * q], s[2 * q + 1], -INFINITY);
#pragma unroll
        for (int e = 8; e < kKeys; e += 8) {
#pragma unroll
          for (int q = 0; q < 4; ++q) mx4[q] = fmax3(mx4[q], s[e + 2 * q], s[e + 2 * q + 1]);
        }
        const float raw_mx = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]);
        const float mx = raw_mx * sc;
        float corr = 1.f;
        bool rescale = false;
        if (mx > m_used + kRescaleThreshold || (m_used == -INFINITY && mx != -INFINITY)) {
          corr = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx);
          m_used = mx;
          rescale = true;
        }
        l *= corr;
        // S_t(j) retired => PV_t(j-1) retired (in-order issue), so O_t is final here
        if (__any_sync(0xffffffffu, rescale && j > 0)) {
#pragma unroll 1
          for (int q = 0; q < kD / 32; ++q) {
            uint32_t w[32];
            tmem_ld_32x32b_x32(t_o + q * 32, w);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(__uint_as_float(w[e]) * corr);
            tmem_st_32x32b_x32(t_o + q * 32, w);
          }
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const uint64_t sc2 = f2(sc, sc), nb2 = f2(-base, -base);
        uint64_t sum2[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
#pragma unroll
        for (int q = 0; q < kKeys / 32; ++q) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int k = q * 32 + 2 * i;
            float x0, x1, e0, e1;
            f2_split(f2_fma(f2(s[k], s[k + 1]), sc2, nb2), x0, x1);
            if ((i % POLY) == POLY - 1) {
              exp2_poly2<DEG>(x0, x1, e0, e1);
            } else {
              e0 = ex2(x0);
              e1 = ex2(x1);
            }
            sum2[i & 1] = f2_add(sum2[i & 1], f2(e0, e1));
            pk[i] = pack_bf16x2(e0, e1);
          }
          tmem_st_32x32b_x16(t_s + q * 16, pk);
          if (q == 1) {  // keys 0-63 of P_t are in TMEM: the first PV half may start
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&p_half[t]);
          }
        }
        float a0, a1, b0, b1;
        f2_split(sum2[0], a0, a1);
        f2_split(sum2[1], b0, b1);
        l += (a0 + a1) + (b0 + b1);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&p_full[t]);
      }
      // ---- epilogue: O_t -> bf16 rows (or an unnormalised partial)
      mbar_wait(&o_full[t], o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      if (v.piece < 0) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        __nv_bfloat16* out =
            p.o + static_cast<size_t>(v.pr.row0 + sub * kRows + r) * HD + v.head * kD;
#pragma unroll 1
        for (int q = 0; q < kD / 32; ++q) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_o + q * 32, w);
          tmem_wait_ld();
          if (r < nrows) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              uint4 pk;
              pk.x = pack_bf16x2(__uint_as_float(w[g * 8 + 0]) * inv, __uint_as_float(w[g * 8 + 1]) * inv);
              pk.y = pack_bf16x2(__uint_as_float(w[g * 8 + 2]) * inv, __uint_as_float(w[g * 8 + 3]) * inv);
              pk.z = pack_bf16x2(__uint_as_float(w[g * 8 + 4]) * inv, __uint_as_float(w[g * 8 + 5]) * inv);
              pk.w = pack_bf16x2(__uint_as_float(w[g * 8 + 6]) * inv, __uint_as_float(w[g * 8 + 7]) * inv);
              *reinterpret_cast<uint4*>(out + q * 32 + g * 8) = pk;
            }
          }
        }
      } else {
        uint8_t* dst = reinterpret_cast<uint8_t*>(p.partial) +
                       ((static_cast<size_t>(v.piece) * 4 + sub) * kRows + r) * kPartRowBytes;
#pragma unroll 1
        for (int q = 0; q < kD / 32; ++q) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(t_o + q * 32, w);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 pk;
            pk.x = pack_bf16x2(__uint_as_float(w[g * 8 + 0]), __uint_as_float(w[g * 8 + 1]));
            pk.y = pack_bf16x2(__uint_as_float(w[g * 8 + 2]), __uint_as_float(w[g * 8 + 3]));
            pk.z = pack_bf16x2(__uint_as_float(w[g * 8 + 4]), __uint_as_float(w[g * 8 + 5]));
            pk.w = pack_bf16x2(__uint_as_float(w[g * 8 + 6]), __uint_as_float(w[g * 8 + 7]));
            *reinterpret_cast<uint4*>(dst + q * 64 + g * 16) = pk;
          }
        }
        reinterpret_cast<float*>(dst + kD * 2)[0] = m_used;
        reinterpret_cast<float*>(dst + kD * 2)[1] = l;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&o_free[t]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 9) tmem_dealloc_pair<512>(tmem);
}

// Merge the pieces of every split (pair, head): half a warp per query row, each
// lane 8 of the 128 dims (16-byte bf16 loads); up to 4 pieces are loaded at once (one
// round trip for the usual 2-3), partial rows read coalesced (256 B per piece-row).
template <int D, int SUB = 2>
__global__ void __launch_bounds__(256)
    fa_combine_kernel(__nv_bfloat16* __restrict__ o, const FaPair* __restrict__ pairs,
                      const FaGroup* __restrict__ groups, int n_heads,
                      const float* __restrict__ partial) {
  constexpr int kD = D;
  constexpr int kPartRowBytes = D * 2 + 16;
  griddep_launch();
  griddep_wait();  // partials of the attention kernel
  // SUB 128-row sub-tiles per plan record: 2 (a pair: nrows0 / nrows1) or 4 (a
  // quad of the CTA-pair kernel: nrows0 = rows of the whole record)
  const FaGroup g = groups[blockIdx.x / (8 * SUB)];
  const int t = static_cast<int>((blockIdx.x >> 3) % SUB), rg = blockIdx.x & 7;
  const FaPair pr = pairs[g.pair];
  const int nrows = SUB == 2 ? (t ? pr.nrows1 : pr.nrows0) : max(0, min(kRows, pr.nrows0 - t * kRows));
  const int r = rg * 16 + static_cast<int>(threadIdx.x >> 4), lane = threadIdx.x & 15;
  if (r >= nrows || lane >= kD / 8) return;  // D=64: 8 lanes per row
  auto row_of = [&](int x) {
    return reinterpret_cast<const uint8_t*>(partial) +
           ((static_cast<size_t>(g.first_piece + x) * SUB + t) * kRows + r) * kPartRowBytes;
  };
  float M = -INFINITY, L = 0.f;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  for (int base = 0; base < g.n_pieces; base += 4) {
    float m[4], l[4];
    uint4 raw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + k < g.n_pieces) {
        const uint8_t* src = row_of(base + k);
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(src + kD * 2));
        m[k] = ml.x;
        l[k] = ml.y;
        raw[k] = __ldcg(reinterpret_cast<const uint4*>(src) + lane);
      } else {
        m[k] = -INFINITY;
        l[k] = 0.f;
        raw[k] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    const float Mn = fmaxf(fmaxf(M, fmaxf(m[0], m[1])), fmaxf(m[2], m[3]));
    if (Mn == -INFINITY) continue;
    const float c = (M == -INFINITY) ? 0.f : exp2f(M - Mn);
    L *= c;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] *= c;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float w = (m[k] == -INFINITY) ? 0.f : exp2f(m[k] - Mn);
      L += w * l[k];
      const uint32_t wd[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wd[j]));
        acc[2 * j] += w * f.x;
        acc[2 * j + 1] += w * f.y;
      }
    }
    M = Mn;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  uint4 pk;
  pk.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
  pk.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
  pk.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
  pk.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
  *reinterpret_cast<uint4*>(o + static_cast<size_t>(pr.row0 + t * kRows + r) * n_heads * kD +
                            g.head * kD + lane * 8) = pk;
}

// ------------------------------------------------------------------ host side
__host__ __forceinline__ static int owner_cta(long long b, long long T, int G) {
  return static_cast<int>(((b + 1) * G + T - 1) / T) - 1;
}

int fa_span(int head_dim) {
  // TK_FA_PAIR=1 selects the CTA-pair kernel for head_dim 128 (read per plan, so a
  // test can switch it).  Off by default: in situ 6% slower than the single-CTA
  // kernel (profiles/r02_experiments.md) -- the softmax chain, not the shared-memory
  // port, bounds the key-block period, and the P / O-free handshakes it waits on
  // become cross-CTA arrivals.
  const char* e = getenv("TK_FA_PAIR");
  return head_dim == 128 && e && atoi(e) != 0 ? 4 * kRows : 2 * kRows;
}

int build_fa_plan(const tk_slice* slices, int n_slices, int n_heads, int max_ctas, FaPlan* plan,
                  FaPair* pairs, int pcap, FaUnit* units, int ucap, FaGroup* groups, int gcap,
                  int32_t* cta_off, int ocap, int span) {
  // span 256: a record is a pair of 128-row tiles (nrows0 / nrows1), one CTA per
  // unit; span 512: a quad of four tiles for the CTA-pair kernel (nrows0 = the
  // quad's rows), one 2-CTA cluster per unit -- max_ctas then counts clusters and
  // every piece takes four partial tiles.
  if (span != 2 * kRows && span != 4 * kRows) return -1;
  const bool quad = span == 4 * kRows;
  const int max_pieces = quad ? kFaMaxPieces / 2 : kFaMaxPieces;
  int np = 0, row = 0;
  long long per_head = 0;
  for (int i = 0; i < n_slices; ++i) {
    const tk_slice& sl = slices[i];
    for (int r = 0; r < sl.len; r += span) {
      if (np >= pcap) return -1;
      FaPair& pr = pairs[np++];
      pr.slice = i;
      pr.row0 = row + r;
      pr.pos0 = sl.start + r;
      pr.nrows0 = quad ? std::min(span, sl.len - r) : std::min(kRows, sl.len - r);
      pr.nrows1 = quad ? 0 : std::max(0, std::min(kRows, sl.len - r - kRows));
      const int kv_end = pr.pos0 + (pr.nrows1 > 0 ? kRows + pr.nrows1 : pr.nrows0);
      pr.nblk = (kv_end + kKeys - 1) / kKeys;
      per_head += pr.nblk;
    }
    row += sl.len;
  }
  const long long T = per_head * n_heads;
  static const int min_blocks = getenv("TK_FA_MIN_BLOCKS") ? atoi(getenv("TK_FA_MIN_BLOCKS"))
                                                          : kMinBlocksPerCta;  // experiments
  int G = static_cast<int>(std::min<long long>(std::max(1, max_ctas),
                                               std::max<long long>(1, T / min_blocks)));
  // Whole units (one (head, pair) per CTA, no pieces, no combine launch) when they fit
  // one wave and the longest is at most `whole_slack` key blocks longer than the split
  // share: short prefixes, where the combine launch costs more than the imbalance
  // (512 queries at prefix 128: 21.3 -> 18.1 us, 256: 21.4 -> 19.8 us; TK_FA_WHOLE
  // overrides, -1 = never).
  static const int whole_slack = getenv("TK_FA_WHOLE") ? atoi(getenv("TK_FA_WHOLE")) : 3;
  if (whole_slack >= 0 && static_cast<long long>(np) * n_heads <= std::max(1, max_ctas)) {
    int longest = 0;
    for (int q = 0; q < np; ++q) longest = std::max(longest, pairs[q].nblk);
    if (longest <= (T + G - 1) / G + whole_slack) {
      G = np * n_heads;
      if (G + 1 > ocap) return -1;
      int nu = 0;
      for (int h = 0; h < n_heads; ++h)
        for (int q = 0; q < np; ++q) {
          if (nu >= ucap) return -1;
          units[nu] = FaUnit{q, h, 0, pairs[q].nblk, -1};
          cta_off[nu] = nu;
          ++nu;
        }
      cta_off[G] = nu;
      plan->n_pairs = np;
      plan->n_units = nu;
      plan->n_ctas = G;
      plan->n_pieces = 0;
      plan->n_groups = 0;
      plan->span = span;
      return 0;
    }
  }
  if (G + 1 > ocap) return -1;
  int nu = 0, piece = 0, n_groups = 0;
  long long cur = 0;
  for (int h = 0; h < n_heads; ++h) {
    for (int q = 0; q < np; ++q) {
      const int nb = pairs[q].nblk;
      const int first = nu;
      int s = 0;
      while (s < nb) {
        const int c = owner_cta(cur, T, G);
        const long long end_c = static_cast<long long>(c + 1) * T / G;
        const int take = static_cast<int>(std::min<long long>(nb - s, end_c - cur));
        if (nu >= ucap) return -1;
        units[nu++] = FaUnit{q, h, s, s + take, -1};
        s += take;
        cur += take;
      }
      if (nu - first > 1) {
        if (piece + (nu - first) > max_pieces || n_groups >= gcap) return -1;
        groups[n_groups++] = FaGroup{piece, nu - first, q, h};
        for (int k = first; k < nu; ++k) units[k].piece = piece++;
      }
    }
  }
  // CTA c owns the units whose first block lies in its range
  std::vector<long long> start(nu);
  {
    long long b = 0;
    for (int k = 0; k < nu; ++k) {
      start[k] = b;
      b += units[k].kb1 - units[k].kb0;
    }
  }
  int k = 0;
  for (int c = 0; c <= G; ++c) {
    while (k < nu && owner_cta(start[k], T, G) < c) ++k;
    cta_off[c] = k;
  }
  cta_off[G] = nu;
  plan->n_pairs = np;
  plan->n_units = nu;
  plan->n_ctas = G;
  plan->n_pieces = piece;
  plan->n_groups = n_groups;
  plan->span = span;
  return 0;
}

int make_tmap_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows);

int launch_chunk_attention_fa(const __nv_bfloat16* qkv, int q_rows, int q_stride,
                              __nv_bfloat16* o, const __nv_bfloat16* pool, int pool_pages,
                              KvGeom g, int layer, const FaPlan& plan, const FaPair* pairs_dev,
                              const FaUnit* units_dev, const FaGroup* groups_dev,
                              const int32_t* cta_off_dev, const tk_slice* slices_dev,
                              const int32_t* bt_dev, float scale, float* partial,
                              cudaStream_t s) {
  TK_CHECK(g.head_dim == 128 || g.head_dim == 64, TK_EUNSUPPORTED,
           "tcgen05 attention: head_dim 128 or 64");
  TK_CHECK(g.page_tokens == 16, TK_EUNSUPPORTED, "tcgen05 attention: 16-token pages");
  if (plan.n_units == 0) return TK_OK;
  CUtensorMap tq, tkv;
  int rc = make_tmap_kmajor(&tq, qkv, q_rows, q_stride, kRows);
  if (rc) return rc;
  const uint64_t blocks = static_cast<uint64_t>(pool_pages) * g.n_layers * g.n_heads * 2;
  rc = make_tmap_kmajor(&tkv, pool, blocks * g.page_tokens, g.head_dim, g.page_tokens);
  if (rc) return rc;
  // TK_FA_VARIANT (experiments): 0 degree-3 poly for 1/4 of the exponentials
  // (default), 1 MUFU only, 2 poly 1/2,
  // 3 poly 1/4 with one wait for the four S loads, 4 MUFU only + batched loads
  static const int variant = getenv("TK_FA_VARIANT") ? atoi(getenv("TK_FA_VARIANT")) : 0;
  using KernFn = void (*)(CUtensorMap, CUtensorMap, FaParams);
  KernFn kern = variant == 1 ? (KernFn)chunk_attn_fa_kernel<128, 0, false>
              : variant == 2 ? (KernFn)chunk_attn_fa_kernel<128, 2, false>
              : variant == 3 ? (KernFn)chunk_attn_fa_kernel<128, 4, true>
              : variant == 4 ? (KernFn)chunk_attn_fa_kernel<128, 0, true>
              : variant == 5 ? (KernFn)chunk_attn_fa_kernel<128, 4, false, 1>
              : variant == 6 ? (KernFn)chunk_attn_fa_kernel<128, 4, false, 2>
              : variant == 7 ? (KernFn)chunk_attn_fa_kernel<128, 4, false, 3>
              : variant == 8 ? (KernFn)chunk_attn_fa_kernel<128, 4, false, 4>
              : variant == 9 ? (KernFn)chunk_attn_fa_kernel<128, 4, false, 0, 3>
              : variant == 10 ? (KernFn)chunk_attn_fa_kernel<128, 3, false, 0, 3>
              : variant == 11 ? (KernFn)chunk_attn_fa_kernel<128, 2, false, 0, 3>
                             : (KernFn)chunk_attn_fa_kernel<128, 4, false, 0, 3>;
  if (g.head_dim == 64) {
    // its own opt-in site: TK_SMEM_OPT_IN keeps one per-device flag per call site
    kern = chunk_attn_fa_kernel<64, 4, false, 0, 3>;
    TK_SMEM_OPT_IN(kern, kSmem);
  } else {
    TK_SMEM_OPT_IN(kern, kSmem);
  }
  const bool quad = plan.span == 4 * kRows;
  TK_CHECK(!quad || g.head_dim == 128, TK_EUNSUPPORTED, "CTA-pair attention: head_dim 128");
  FaParams prm;
  prm.pairs = pairs_dev;
  prm.units = units_dev;
  prm.cta_off = cta_off_dev;
  prm.slices = slices_dev;
  prm.bt = bt_dev;
  prm.o = o;
  prm.partial = partial;
  prm.n_layers = g.n_layers;
  prm.n_heads = g.n_heads;
  prm.layer = layer;
  prm.scale_log2 = scale * 1.4426950408889634f;
  if (quad) {
    // TK_FA_PAIR_POLY (experiments): 1 of N exponential pairs by the polynomial
    static const int pair_poly = getenv("TK_FA_PAIR_POLY") ? atoi(getenv("TK_FA_PAIR_POLY")) : 4;
    auto pk = pair_poly == 2 ? chunk_attn_fa_pair_kernel<2, 3>
            : pair_poly == 3 ? chunk_attn_fa_pair_kernel<3, 3> : chunk_attn_fa_pair_kernel<4, 3>;
    if (pair_poly == 2) TK_SMEM_OPT_IN(pk, kPairSmem);
    else if (pair_poly == 3) TK_SMEM_OPT_IN(pk, kPairSmem);
    else TK_SMEM_OPT_IN(pk, kPairSmem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(plan.n_ctas * 2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kPairSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    int na = 1;
    if (pdl_enabled()) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    TK_CUDA(cudaLaunchKernelEx(&cfg, pk, tq, tkv, prm));
  } else {
    TK_CUDA(launch_pdl(kern, dim3(plan.n_ctas), dim3(kThreads), kSmem, s, tq, tkv, prm));
  }
  TK_CUDA(cudaGetLastError());
  note_launch();
  if (plan.n_groups > 0) {
    static const bool comb_pdl = !getenv("TK_COMBINE_PDL") || atoi(getenv("TK_COMBINE_PDL")) != 0;
    auto ck = quad ? fa_combine_kernel<128, 4>
            : g.head_dim == 64 ? fa_combine_kernel<64> : fa_combine_kernel<128>;
    TK_CUDA(launch_maybe_pdl(comb_pdl, ck, dim3(plan.n_groups * (quad ? 32 : 16)), dim3(256), 0, s,
                             o, pairs_dev, groups_dev, g.n_heads, partial));
    TK_CUDA(cudaGetLastError());
    note_launch();
  }
  return TK_OK;
}

}  // namespace tk

namespace tk {
int fa_debug_trace(unsigned long long* host, int n) {
  n = n < 10 * 2 * 512 ? n : 10 * 2 * 512;
  TK_CUDA(cudaMemcpyFromSymbol(host, g_fa_trace, n * sizeof(unsigned long long)));
  return TK_OK;
}
}  // namespace tk
