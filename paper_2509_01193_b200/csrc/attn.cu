// Varlen causal attention forward on tcgen05 (the decoder layer's attention;
// block-diagonal causal mask over the packed batch).  head_dim 128, bf16 in/out,
// fp32 softmax, grouped-query heads.
//
// One CTA per work item (sequence, 128-query tile, head), items ordered longest first.
//   warp 0   TMA producer: the Q tile once, then K_j and V_j tiles in separate 2-stage rings
//            (K_j is released as soon as S_j is done, V_j after P_j V_j), K_j ahead of V_{j-1}
//   warp 1   MMA issuer:   S_j = Q K_j^T into TMEM (double buffered, 2 x 128 columns) while
//                          the softmax works on S_{j-1}; O += P_j V_j (P double buffered)
//   warp 2   TMEM allocator
//   warps 4-11 softmax, a query row and 64 key columns per thread (two warps per TMEM lane
//            group, row maxima exchanged through shared memory): row max of S_j (masked:
//            key <= query and inside the sequence), p = exp2(s log2e / sqrt(D) - m), P_j to shared memory
//            in the 128-byte-swizzled K-major layout of the next MMA's A operand, running
//            sum l; O accumulates in TMEM (lazy rescale when the row max grows by > 2^8)
// Outputs: O (bf16, same layout as Q) and LSE [H, T] fp32 (natural log; FlashAttention's
// varlen layout, so its backward can consume them).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.h"
#include "lora_internal.h"
#include "ptx.cuh"

namespace lobra {
int64_t count_launch(int kind, cudaStream_t st, bool begin);   // lora_host.cu

namespace {
using namespace ptx;

constexpr int A_TILE = 128;                    // queries / keys per tile
constexpr int A_BOX = 128 * 64 * 2;            // one 64-column box of a 128-row tile: 16 KB
constexpr int A_TILE_BYTES = 2 * A_BOX;        // 128 x 128 bf16
// Q | K[2] | V[2] | P[2] | barriers | row-max exchange [2 halves][128] (the row-sum exchange
// at the end reuses it)
constexpr int A_SMEM = 7 * A_TILE_BYTES + 1024 + 256 + 2 * 128 * 4;

struct AttnItem {
  int q_row0;     // token index of the tile's first query
  int kv_row0;    // token index of the sequence start
  int len;        // sequence length
  int q_tile;     // tile index inside the sequence (its queries start at q_tile * 128)
  int head;
};

struct AttnArgs {
  const AttnItem* items;
  int nitems, H, Hkv, T;
  float scale_log2;           // log2(e) / sqrt(D)
  __nv_bfloat16* O;           // [T, H * 128]
  float* lse;                 // [H, T]
  unsigned long long* ts;     // tracing (LOBRA_TRACE_ATTN): per-phase clock64 stamps of CTA 0, else null
};
// trace slots: [event][iteration], event-major, 64 iterations
#define ATTN_TS(ev, t) \
  do { if (args.ts && blockIdx.x == 0 && (t) < 64) args.ts[(ev) * 64 + (t)] = clock64(); } while (0)
__device__ __forceinline__ float ex2(float x) {   // MUFU.EX2; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint8_t* align1024a(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__global__ void __launch_bounds__(384, 1)
    k_attn_fwd(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
               const __grid_constant__ CUtensorMap mapV, const AttnArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024a(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + A_TILE_BYTES;                        // [2]
  uint8_t* sV = sK + 2 * A_TILE_BYTES;                    // [2]
  uint8_t* sP = sV + 2 * A_TILE_BYTES;                    // [2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * A_TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;      // [2]
  uint64_t* k_empty = bars + 3;     // [2]  S_j done: K_j free (long before V_j)
  uint64_t* v_full = bars + 5;      // [2]
  uint64_t* v_empty = bars + 7;     // [2]
  uint64_t* s_full = bars + 9;      // [2]
  uint64_t* s_empty = bars + 11;    // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* pv_done = bars + 14;    // [2]  P_j V_j done (per P buffer: completes every 2nd tile)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  float* xmax = reinterpret_cast<float*>(bars + 32);     // [2 halves][128 rows]
  float* xsum = xmax;                                     // [2 halves][128 rows], after the loop

  const uint32_t warp = warp_id(), lane = lane_id();
  const AttnItem it = args.items[blockIdx.x];
  const int nkv = it.q_tile + 1;                           // causal: key tiles 0..q_tile
  const int hk = it.head / (args.H / args.Hkv);

  if (warp == 0 && lane == 0) tma_prefetch(&mapQ), tma_prefetch(&mapK), tma_prefetch(&mapV);
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1), mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 256);
      mbar_init(&pv_done[s], 1);
    }
    mbar_init(p_full, 256);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // completion of P_j V_j: its P buffer's barrier, phase j >> 1
  auto wait_pv = [&](int j) { mbar_wait(&pv_done[j & 1], (j >> 1) & 1); };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: K_j ahead of V_{j-1}
      mbar_expect_tx(q_full, A_TILE_BYTES);
      tma_load_2d(sQ, &mapQ, q_full, it.head * 128, it.q_row0);
      tma_load_2d(sQ + A_BOX, &mapQ, q_full, it.head * 128 + 64, it.q_row0);
      auto load = [&](int j, bool v) {
        const int s = j & 1;
        uint64_t* full = v ? &v_full[s] : &k_full[s];
        mbar_wait(v ? &v_empty[s] : &k_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(full, A_TILE_BYTES);
        uint8_t* dst = (v ? sV : sK) + s * A_TILE_BYTES;
        const int row = it.kv_row0 + j * A_TILE;
        tma_load_2d(dst, v ? &mapV : &mapK, full, hk * 128, row);
        tma_load_2d(dst + A_BOX, v ? &mapV : &mapK, full, hk * 128 + 64, row);
      };
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          load(j, false);
          ATTN_TS(0, j);
        }
        if (j >= 1) load(j - 1, true);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t id_s = idesc_bf16(128, 128, false, false);   // S: Q, K both K-major
      const uint32_t id_o = idesc_bf16(128, 128, false, true);    // O: P K-major, V MN-major
      const uint32_t q0 = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        mbar_wait(&k_full[s], (j >> 1) & 1);
        mbar_wait(&s_empty[s], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        ATTN_TS(1, j);
        const uint32_t k0 = smem_u32(sK + s * A_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // K = head_dim 128: 2 swizzle atoms x 4 steps of 16
          const uint32_t off = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tmem + s * 128, sdesc_sw128(q0 + off, 16, 1024), sdesc_sw128(k0 + off, 16, 1024), id_s,
                   kk ? 1u : 0u);
        }
        mma_commit(&s_full[s]);
        mma_commit(&k_empty[s]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        const int s = j & 1;
        mbar_wait(p_full, j & 1);   // P_j written (and O rescaled if the softmax had to)
        mbar_wait(&v_full[s], (j >> 1) & 1);
        tc_fence_after();
        ATTN_TS(2, j);
        const uint32_t v0 = smem_u32(sV + s * A_TILE_BYTES), p0 = smem_u32(sP + s * A_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // K = 128 keys: P (K-major) x V (MN-major)
          const uint32_t poff = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tmem + 256, sdesc_sw128(p0 + poff, 16, 1024), sdesc_sw128(v0 + kk * 2048, A_BOX, 1024), id_o,
                   (j | kk) ? 1u : 0u);   // O accumulates in TMEM over the key tiles
        }
        mma_commit(&pv_done[s]);
        mma_commit(&v_empty[s]);
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax / epilogue: 8 warps
    // Two warps per TMEM lane group (two per SM sub-partition, so the exp / max / pack chains
    // of one hide the latencies of the other): warp w owns query row r = 32 (w % 4) + lane
    // and key columns (and O columns) 64 hw .. +63, hw = (w - 4) / 4; the two halves of a row
    // exchange their maxima through shared memory once per key tile.
    // O accumulates in TMEM; P is computed against a reference max m that is raised (and O, l
    // rescaled in place) only when a tile's max exceeds it by more than 8 (log2 units, i.e.
    // p <= 256): the final O / l is exact either way.
    const int g4 = warp & 3, hw = (warp - 4) >> 2;
    const int r = g4 * 32 + lane;
    const int qpos = it.q_tile * A_TILE + r;               // position inside the sequence
    const bool qvalid = qpos < it.len;
    const uint32_t trow = (g4 * 32u) << 16;
    const uint32_t sP_a = smem_u32(sP);
    // invalid rows (past the sequence end in its last tile) keep m = 0 and only see -inf
    float m = qvalid ? -INFINITY : 0.0f, l = 0.0f;
    // per-element masks only where a tile can hold masked keys: the diagonal tile and the
    // tiles reaching past the sequence end, plus every tile of a query tile with rows past it
    const bool tail_rows = (it.q_tile + 1) * A_TILE > it.len;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      if (r == 0 && hw == 0) ATTN_TS(3, j);
      const int kbase = j * A_TILE + hw * 64;
      float sv[64];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float v[32];
        tmem_ld32(tmem + trow + sb * 128 + hw * 64 + c * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) sv[c * 32 + e] = v[e];
      }
      tc_fence_before();
      mbar_arrive(&s_empty[sb]);                             // S buffer free for S_{j+2}
      if (j == nkv - 1 || tail_rows || j * A_TILE + A_TILE > it.len) {   // warp-uniform
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const int kpos = kbase + e;
          if (!(qvalid && kpos <= qpos && kpos < it.len)) sv[e] = -INFINITY;
        }
      }
      // row max of this half as 8 independent chains, then the other half's through smem
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = sv[u];
#pragma unroll
      for (int e = 8; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], sv[e]);
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      xmax[hw * 128 + r] = mx;
      named_bar(1, 256);
      mx = fmaxf(mx, xmax[(hw ^ 1) * 128 + r]) * args.scale_log2;   // scale > 0: max commutes
      named_bar(1, 256);   // both halves read before the next tile's maxima are written
      if (r == 0 && hw == 0) ATTN_TS(4, j);
      if (r == 0 && hw == 0) ATTN_TS(5, j);
      // raise the reference max where needed (both halves decide identically); the TMEM
      // rescale is warp-collective (tcgen05.ld / st are .sync.aligned): every lane takes
      // part, alpha = 1 where unchanged
      const bool raise = qvalid && (j == 0 || mx > m + 8.0f);
      const float m_new = raise ? fmaxf(m, mx) : m;
      const float alpha = (raise && j >= 1) ? ex2(m - m_new) : 1.0f;
      if (j >= 1 && __any_sync(0xffffffffu, raise)) {
        wait_pv(j - 1);   // O quiescent before it is rescaled in place
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(tmem + trow + 256 + hw * 64 + c * 32, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] *= alpha;
          tmem_st32(tmem + trow + 256 + hw * 64 + c * 32, v);
        }
      }
      l *= alpha;
      m = m_new;
      float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (j >= 2) wait_pv(j - 2);   // P buffer j & 1 was last read by P_{j-2} V_{j-2}
      const uint32_t row = sP_a + (j & 1) * A_TILE_BYTES + hw * A_BOX + r * 128;   // 64 keys = one atom row
#pragma unroll
      for (int u = 0; u < 8; ++u) {                         // 16-byte chunk u of the row
        float p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          p[e] = ex2(fmaf(sv[u * 8 + e], args.scale_log2, -m));   // masked: ex2(-inf) = 0
          sum8[e] += p[e];
        }
        sts128(row + ((u ^ (r & 7)) << 4), pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]),
               pack_bf16x2(p[4], p[5]), pack_bf16x2(p[6], p[7]));
      }
      l += ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
      tc_fence_before();
      fence_proxy_async_smem();   // P stores visible to the tensor core
      mbar_arrive(p_full);
      if (r == 0 && hw == 0) ATTN_TS(6, j);
    }
    xsum[hw * 128 + r] = l;
    named_bar(1, 256);
    l += xsum[(hw ^ 1) * 128 + r];
    wait_pv(nkv - 1);               // the last P V (and with it every earlier one) is done
    tc_fence_after();
    const float inv = qvalid ? 1.0f / l : 0.0f;
    const size_t tok = (size_t)it.q_row0 + r;
    uint4* dst = reinterpret_cast<uint4*>(args.O + tok * (size_t)(args.H * 128) + it.head * 128 + hw * 64);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v[32];
      tmem_ld32(tmem + trow + 256 + hw * 64 + c * 32, v);   // warp-collective: every lane
      if (qvalid) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w;
          w.x = pack_bf16x2(v[u * 8 + 0] * inv, v[u * 8 + 1] * inv);
          w.y = pack_bf16x2(v[u * 8 + 2] * inv, v[u * 8 + 3] * inv);
          w.z = pack_bf16x2(v[u * 8 + 4] * inv, v[u * 8 + 5] * inv);
          w.w = pack_bf16x2(v[u * 8 + 6] * inv, v[u * 8 + 7] * inv);
          dst[c * 4 + u] = w;
        }
      }
    }
    if (qvalid && hw == 0) args.lse[(size_t)it.head * args.T + tok] = (m + log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// =====================================================================================
// Varlen causal attention BACKWARD on tcgen05 (FlashAttention's recomputation scheme: P is
// rebuilt from the forward's LSE, never stored).  Per query row q of a sequence and head h:
//   P = exp(S / sqrt(D) - LSE),  dP = dO V^T,  Dq = sum_d dO O,  dS = P (dP - Dq),
//   dV = P^T dO,  dK = dS^T Q / sqrt(D),  dQ = dS K / sqrt(D).
// One CTA per (sequence, 128-key tile j, kv head): K_j, V_j stay in shared memory; the CTA
// walks the query tiles i >= j (causal) of every query head of the kv group, so dK_j and dV_j
// accumulate in TMEM and are written once (no atomics); dQ_i partials are added into an fp32
// accumulator with red.global.add (k_attn_bwd_post scales and rounds it).  The transposed
// products put the KEY row in the TMEM lane: S^T = K Q^T and dP^T = V dO^T, so a softmax
// thread owns one key row and writes P^T / dS^T rows straight into the K-major A layouts of
// dV += P^T dO and dK += dS^T Q; the same dS^T buffer is the MN-major A operand of dQ = dS K.
//   warp 0      TMA producer: K_j, V_j once; Q_i (2 stages) and dO_i per iteration
//   warp 1      MMA issuer
//   warp 2      TMEM allocator (512 columns: R0, R1, dV, dK)
//   warps 4-11  P^T / dS^T (a key row and 64 query columns per thread: two warps per TMEM
//               lane group), the dQ drain (TMEM -> red.global.add.v4.f32 into an fp32
//               accumulator) and the final dK / dV epilogue
// TMEM roles alternate per iteration t: S^T -> R[t&1], dP^T -> R[(t+1)&1], dQ -> R[t&1], so
// the next S^T is computed while dQ_t drains.
// =====================================================================================
constexpr int B_SMEM = 7 * A_TILE_BYTES /*K V Q0 Q1 dO P dS*/ + 2 * 128 * 4 /*lse2, D*/ + 1024 + 256;

struct AttnBwdItem {
  int kv_row0;    // token index of the sequence start
  int len;        // sequence length
  int k_tile;     // key tile j
  int kv_head;
};

struct AttnBwdArgs {
  const AttnBwdItem* items;
  int H, Hkv, T;
  float scale_log2;           // log2(e) / sqrt(D)
  float scale;                // 1 / sqrt(D)
  const float* lse;           // [H, T] natural log
  const float* Dq;            // [H, T]
  float* dq_acc;              // [T, H * 128] fp32
  __nv_bfloat16* dK;          // [T, Hkv * 128]
  __nv_bfloat16* dV;
  unsigned long long* ts;     // tracing (LOBRA_TRACE_ATTN): per-phase clock64 stamps of CTA 0, else null
};

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// P^T (or dS^T) chunk c (32 query columns) of key row kr: 32 bf16 values as four 16-byte
// shared stores into the 128-byte-swizzled K-major row of the buffer at shared address `buf`.
__device__ __forceinline__ void store_row_chunk(uint32_t buf, int kr, int c, const uint32_t* pk) {
  const uint32_t row = buf + (c >> 1) * A_BOX + kr * 128;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t ch = (uint32_t)((((c & 1) * 4) + u) ^ (kr & 7)) << 4;
    sts128(row + ch, pk[u * 4], pk[u * 4 + 1], pk[u * 4 + 2], pk[u * 4 + 3]);
  }
}

__global__ void __launch_bounds__(384, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
               const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapdO,
               const AttnBwdArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024a(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + A_TILE_BYTES;
  uint8_t* sQ = sV + A_TILE_BYTES;             // [2]
  uint8_t* sdO = sQ + 2 * A_TILE_BYTES;
  uint8_t* sP = sdO + A_TILE_BYTES;            // P^T  [key rows][query cols], K-major SW128
  uint8_t* sdS = sP + A_TILE_BYTES;            // dS^T [key rows][query cols]
  float* s_lse = reinterpret_cast<float*>(sdS + A_TILE_BYTES);   // [128] lse * log2(e)
  float* s_D = s_lse + 128;                                      // [128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_D + 128);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;      // [2]
  uint64_t* q_empty = bars + 3;     // [2]
  uint64_t* do_full = bars + 5;
  uint64_t* do_empty = bars + 6;
  uint64_t* s_full = bars + 7;      // S^T in TMEM
  uint64_t* dp_full = bars + 8;     // dP^T in TMEM
  uint64_t* p_full = bars + 9;      // P^T in smem (256 arrivals)
  uint64_t* ds_full = bars + 10;    // dS^T in smem (256 arrivals)
  uint64_t* p_empty = bars + 11;    // dV (the reader of P^T) done
  uint64_t* ds_empty = bars + 12;   // dK, dQ (the readers of dS^T) done
  uint64_t* dq_full = bars + 13;
  uint64_t* dq_empty = bars + 14;   // dQ_t read out of TMEM (256 arrivals)
  uint64_t* fin = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const uint32_t warp = warp_id(), lane = lane_id();
  const AttnBwdItem it = args.items[blockIdx.x];
  const int nt = (it.len + A_TILE - 1) / A_TILE;
  const int nq = nt - it.k_tile;                     // query tiles i = j .. nt-1
  const int G = args.H / args.Hkv;
  const int niter = nq * G;                          // (head of the group, query tile)
  const int j = it.k_tile;

  if (warp == 0 && lane == 0)
    tma_prefetch(&mapQ), tma_prefetch(&mapK), tma_prefetch(&mapV), tma_prefetch(&mapdO);
  if (warp == 1 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&q_full[s], 1), mbar_init(&q_empty[s], 1);
    mbar_init(do_full, 1), mbar_init(do_empty, 1);
    mbar_init(s_full, 1), mbar_init(dp_full, 1), mbar_init(p_full, 256), mbar_init(ds_full, 256);
    mbar_init(p_empty, 1), mbar_init(ds_empty, 1), mbar_init(dq_full, 1), mbar_init(dq_empty, 256);
    mbar_init(fin, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto R = [&](int t) { return tmem + (uint32_t)(t & 1) * 128u; };
  const uint32_t tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      const int krow = it.kv_row0 + j * A_TILE;
      mbar_expect_tx(kv_full, 2 * A_TILE_BYTES);
      tma_load_2d(sK, &mapK, kv_full, it.kv_head * 128, krow);
      tma_load_2d(sK + A_BOX, &mapK, kv_full, it.kv_head * 128 + 64, krow);
      tma_load_2d(sV, &mapV, kv_full, it.kv_head * 128, krow);
      tma_load_2d(sV + A_BOX, &mapV, kv_full, it.kv_head * 128 + 64, krow);
      for (int t = 0; t < niter; ++t) {
        const int h = it.kv_head * G + t / nq, i = j + t % nq;
        const int qrow = it.kv_row0 + i * A_TILE;
        const int qb = t & 1;
        mbar_wait(&q_empty[qb], ((t >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qb], A_TILE_BYTES);
        uint8_t* q = sQ + qb * A_TILE_BYTES;
        tma_load_2d(q, &mapQ, &q_full[qb], h * 128, qrow);
        tma_load_2d(q + A_BOX, &mapQ, &q_full[qb], h * 128 + 64, qrow);
        mbar_wait(do_empty, (t & 1) ^ 1);
        mbar_expect_tx(do_full, A_TILE_BYTES);
        tma_load_2d(sdO, &mapdO, do_full, h * 128, qrow);
        tma_load_2d(sdO + A_BOX, &mapdO, do_full, h * 128 + 64, qrow);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      // Order per tile t: [S^T_t issued at the end of t-1] dP^T_t, (P^T) dV_t, (dS^T) S^T_{t+1},
      // dK_t, dQ_t -- the next tile's S^T runs while the softmax warps write dS^T, and their
      // P^T phase of t+1 overlaps dK_t / dQ_t.
      const uint32_t id_kk = idesc_bf16(128, 128, false, false);   // S^T, dP^T: both K-major
      const uint32_t id_kn = idesc_bf16(128, 128, false, true);    // dV, dK: A K-major, B MN-major
      const uint32_t id_nn = idesc_bf16(128, 128, true, true);     // dQ: A MN-major, B MN-major
      const uint32_t k0 = smem_u32(sK), v0 = smem_u32(sV), do0 = smem_u32(sdO);
      const uint32_t p0 = smem_u32(sP), ds0 = smem_u32(sdS);
      auto issue_s = [&](int t) {   // S^T_t = K Q_t^T into R[t&1]
        const int qb = t & 1;
        const uint32_t q0 = smem_u32(sQ + qb * A_TILE_BYTES);
        mbar_wait(&q_full[qb], (t >> 1) & 1);
        tc_fence_after();
        ATTN_TS(0, t);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(R(t), sdesc_sw128(k0 + off, 16, 1024), sdesc_sw128(q0 + off, 16, 1024), id_kk, kk ? 1u : 0u);
        }
        mma_commit(s_full);
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      for (int t = 0; t < niter; ++t) {
        const int qb = t & 1;
        const uint32_t q0 = smem_u32(sQ + qb * A_TILE_BYTES);
        mbar_wait(do_full, t & 1);
        ATTN_TS(8, t);
        if (t >= 1) mbar_wait(dq_empty, (t - 1) & 1);   // R[(t+1)&1] held dQ_{t-1}
        tc_fence_after();
        ATTN_TS(1, t);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // dP^T = V dO^T
          const uint32_t off = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(R(t + 1), sdesc_sw128(v0 + off, 16, 1024), sdesc_sw128(do0 + off, 16, 1024), id_kk,
                   kk ? 1u : 0u);
        }
        mma_commit(dp_full);
        mbar_wait(p_full, t & 1);   // P^T in smem
        tc_fence_after();
        ATTN_TS(2, t);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // dV += P^T dO  (K = queries)
          const uint32_t aoff = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tdV, sdesc_sw128(p0 + aoff, 16, 1024), sdesc_sw128(do0 + kk * 2048, A_BOX, 1024), id_kn,
                   (t | kk) ? 1u : 0u);
        }
        mma_commit(do_empty);
        mma_commit(p_empty);
        mbar_wait(ds_full, t & 1);  // dS^T in smem; S^T_t and dP^T_t consumed
        tc_fence_after();
        ATTN_TS(3, t);
        if (t + 1 < niter) issue_s(t + 1);   // R[(t+1)&1] (dP^T_t) is free
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // dK += dS^T Q
          const uint32_t aoff = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tdK, sdesc_sw128(ds0 + aoff, 16, 1024), sdesc_sw128(q0 + kk * 2048, A_BOX, 1024), id_kn,
                   (t | kk) ? 1u : 0u);
        }
        mma_commit(&q_empty[qb]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)     // dQ_t = dS K  (M = queries, K = keys) into R[t&1]
          mma_bf16(R(t), sdesc_sw128(ds0 + kk * 2048, A_BOX, 1024), sdesc_sw128(k0 + kk * 2048, A_BOX, 1024),
                   id_nn, kk ? 1u : 0u);
        mma_commit(dq_full);
        mma_commit(ds_empty);
      }
      mma_commit(fin);
    }
  } else if (warp >= 4) {  // ---------------- P^T / dS^T and the dQ drain: 8 warps
    // Two warps per TMEM lane group (two per SM sub-partition): warp w handles key rows
    // (lanes) 32 (w % 4) .. +31 and query columns (P^T, dS^T) or head-dim columns (dQ)
    // 64 hw .. +63, hw = (w - 4) / 4.
    const int g4 = warp & 3, hw = (warp - 4) >> 2;
    const int kr = g4 * 32 + lane;                       // key row of the tile (TMEM lane)
    const int kpos = j * A_TILE + kr;                    // position in the sequence
    const int tid = (warp - 4) * 32 + lane;              // 0 .. 255
    const uint32_t trow = (g4 * 32u) << 16;
    const uint32_t sP_a = smem_u32(sP), sdS_a = smem_u32(sdS), lse_a = smem_u32(s_lse), D_a = smem_u32(s_D);
    // the tile's lse (log2 units) and Dq, one query row per thread of the first 128; loaded
    // one iteration ahead (their global latency overlaps the wait for the next S^T)
    auto load_ld = [&](int t, float& l2, float& dd) {
      const int h = it.kv_head * G + t / nq, i = j + t % nq;
      const int qp = i * A_TILE + tid;
      const size_t tok = (size_t)it.kv_row0 + qp;
      const bool ok = tid < 128 && qp < it.len;
      l2 = ok ? __ldg(args.lse + (size_t)h * args.T + tok) * 1.4426950408889634f : 0.0f;
      dd = ok ? __ldg(args.Dq + (size_t)h * args.T + tok) : 0.0f;
    };
    // dQ_t, in two steps.  (a) TMEM -> registers (64 head-dim columns of one query row per
    // thread), the TMEM region released at once (dq_empty: dP^T_{t+1} may overwrite it).
    // (b) after the next dS^T phase, through the P^T buffer (free once dV has read it): each
    // 64-column half is written row-major (256-byte rows, 16-byte chunks XOR-swizzled by
    // row), read back two rows per warp instruction and added into the fp32 accumulator with
    // red.global.add.v4 -- 256 contiguous bytes per row and instruction instead of 32
    // scattered rows (8x fewer L2 requests).
    float dqv[64];
    auto drain_tmem = [&](int t) {
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float w[32];
        tmem_ld32(R(t) + trow + hw * 64 + c * 32, w);
#pragma unroll
        for (int e = 0; e < 32; ++e) dqv[c * 32 + e] = w[e];
      }
      tc_fence_before();
      mbar_arrive(dq_empty);
      if (tid == 0) ATTN_TS(9, t + 1);
    };
    auto drain_red = [&](int t) {   // P^T buffer must be free (dV of the current tile done)
      const int h = it.kv_head * G + t / nq, i = j + t % nq;
      const int q0 = i * A_TILE;
      const int rw = tid >> 5;                                       // 16 rows per warp
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        if (hw == half) {
          const uint32_t row = sP_a + kr * 256;                      // kr = the query row here
#pragma unroll
          for (int c = 0; c < 16; ++c)
            sts128(row + ((c ^ (kr & 15)) << 4), __float_as_uint(dqv[c * 4]), __float_as_uint(dqv[c * 4 + 1]),
                   __float_as_uint(dqv[c * 4 + 2]), __float_as_uint(dqv[c * 4 + 3]));
        }
        named_bar(1, 256);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = rw * 16 + u * 2 + (lane >> 4), c = lane & 15;
          const float4 x = lds128f(sP_a + r * 256 + ((c ^ (r & 15)) << 4));
          if (q0 + r < it.len)
            red_add_v4(args.dq_acc + ((size_t)it.kv_row0 + q0 + r) * (size_t)(args.H * 128) + h * 128 + half * 64 +
                           c * 4, x.x, x.y, x.z, x.w);
        }
        named_bar(1, 256);
      }
      if (tid == 0) ATTN_TS(10, t + 1);
    };
    float nl2, ndd;
    load_ld(0, nl2, ndd);
    for (int t = 0; t < niter; ++t) {
      const int i = j + t % nq;
      const int qpos0 = i * A_TILE;
      if (tid < 128) s_lse[tid] = nl2, s_D[tid] = ndd;
      if (t + 1 < niter) load_ld(t + 1, nl2, ndd);
      named_bar(1, 256);
      mbar_wait(s_full, t & 1);
      if (t >= 1) mbar_wait(p_empty, (t - 1) & 1);       // dV_{t-1} has read P^T
      tc_fence_after();
      if (tid == 0) ATTN_TS(4, t);
      // masks only where a tile can hold masked pairs: the diagonal and the sequence tail
      // (warp-uniform; the common unmasked tiles run without the compare / select work)
      const bool need_mask = (i == j) || (qpos0 + A_TILE > it.len);
      const int lim = need_mask ? min(it.len - qpos0, A_TILE) : A_TILE;   // valid query columns
      const int diag = kpos - qpos0;                       // masked: q < diag
      uint32_t pk[32];   // P^T row half, bf16 pairs (the rounded values the dV product uses)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cq = hw * 2 + c;                         // 32-column chunk of the 128
        float sv[32];
        tmem_ld32(R(t) + trow + cq * 32, sv);
        float l2[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 x = lds128f(lse_a + (cq * 32 + u * 4) * 4);
          l2[u * 4] = x.x, l2[u * 4 + 1] = x.y, l2[u * 4 + 2] = x.z, l2[u * 4 + 3] = x.w;
        }
        if (!need_mask) {
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            pk[(c * 32 + e) >> 1] = pack_bf16x2(ex2(fmaf(sv[e], args.scale_log2, -l2[e])),
                                                ex2(fmaf(sv[e + 1], args.scale_log2, -l2[e + 1])));
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int q = cq * 32 + e;
            float p0v = ex2(fmaf(sv[e], args.scale_log2, -l2[e]));
            float p1v = ex2(fmaf(sv[e + 1], args.scale_log2, -l2[e + 1]));
            if (q < diag || q >= lim) p0v = 0.0f;
            if (q + 1 < diag || q + 1 >= lim) p1v = 0.0f;
            pk[(c * 32 + e) >> 1] = pack_bf16x2(p0v, p1v);
          }
        }
        store_row_chunk(sP_a, kr, cq, pk + c * 16);
      }
      tc_fence_before();
      fence_proxy_async_smem();   // P^T visible to the tensor core
      mbar_arrive(p_full);
      if (tid == 0) ATTN_TS(5, t);
      if (t >= 1) drain_tmem(t - 1);   // dQ_{t-1} (issued before S^T_t, so complete by now)
      mbar_wait(dp_full, t & 1);
      if (t >= 1) mbar_wait(ds_empty, (t - 1) & 1);      // dK_{t-1}, dQ_{t-1} have read dS^T
      tc_fence_after();
      if (tid == 0) ATTN_TS(6, t);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cq = hw * 2 + c;
        float dp[32];
        tmem_ld32(R(t + 1) + trow + cq * 32, dp);
        uint32_t dk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 dd = lds128f(D_a + (cq * 32 + e) * 4);
          const float2 pa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[(c * 32 + e) >> 1]));
          const float2 pb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[((c * 32 + e) >> 1) + 1]));
          dk[e >> 1] = pack_bf16x2(pa.x * (dp[e] - dd.x), pa.y * (dp[e + 1] - dd.y));
          dk[(e >> 1) + 1] = pack_bf16x2(pb.x * (dp[e + 2] - dd.z), pb.y * (dp[e + 3] - dd.w));
        }
        store_row_chunk(sdS_a, kr, cq, dk);
      }
      tc_fence_before();
      fence_proxy_async_smem();   // dS^T visible to the tensor core
      mbar_arrive(ds_full);
      if (tid == 0) ATTN_TS(7, t);
      if (t >= 1) {
        mbar_wait(p_empty, t & 1);   // dV_t has read P^T: its buffer stages dQ_{t-1}
        drain_red(t - 1);
      } else {
        named_bar(1, 256);           // every thread is done with s_lse / s_D of this tile
      }
    }
    // the last dQ: its TMEM read, then the staging (dV of the last tile is done: fin)
    drain_tmem(niter - 1);
    mbar_wait(fin, 0);
    tc_fence_after();
    drain_red(niter - 1);
    // dK, dV of the key tile (complete: every query head of the kv group went through them)
    const bool kvalid = kpos < it.len;
    const size_t tok = (size_t)it.kv_row0 + kpos;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      __nv_bfloat16* base = which ? args.dK : args.dV;
      const float mul = which ? args.scale : 1.0f;
      uint4* dst = reinterpret_cast<uint4*>(base + tok * (size_t)(args.Hkv * 128) + it.kv_head * 128 + hw * 64);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float v[32];
        tmem_ld32((which ? tdK : tdV) + trow + hw * 64 + c * 32, v);   // warp-collective
        if (kvalid) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 w;
            w.x = pack_bf16x2(v[u * 8 + 0] * mul, v[u * 8 + 1] * mul);
            w.y = pack_bf16x2(v[u * 8 + 2] * mul, v[u * 8 + 3] * mul);
            w.z = pack_bf16x2(v[u * 8 + 4] * mul, v[u * 8 + 5] * mul);
            w.w = pack_bf16x2(v[u * 8 + 6] * mul, v[u * 8 + 7] * mul);
            dst[c * 4 + u] = w;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Dq[h][t] = sum_d dO[t][h][d] O[t][h][d] (fp32), and the dQ accumulator row zeroed: one warp
// per (token, head), 4 elements per lane.
__global__ void k_attn_bwd_pre(const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ dO,
                               int T, int H, float* __restrict__ Dq, float* __restrict__ dq_acc) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)T * H) return;
  const long long t = w / H;
  const int h = (int)(w % H);
  const size_t base = (size_t)t * H * 128 + (size_t)h * 128 + lane * 4;
  const uint2 a = *reinterpret_cast<const uint2*>(O + base);
  const uint2 b = *reinterpret_cast<const uint2*>(dO + base);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
  float s = 0.0f;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float2 x = __bfloat1622float2(a2[e]), y = __bfloat1622float2(b2[e]);
    s = fmaf(x.x, y.x, s);
    s = fmaf(x.y, y.y, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) Dq[(size_t)h * T + t] = s;
  *reinterpret_cast<float4*>(dq_acc + base) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// dQ = scale * accumulator, rounded to bf16 (8 elements per thread).
__global__ void k_attn_bwd_post(const float* __restrict__ acc, long long n8, float scale,
                                __nv_bfloat16* __restrict__ dQ) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(acc)[2 * i];
    const float4 b = reinterpret_cast<const float4*>(acc)[2 * i + 1];
    uint4 w;
    w.x = pack_bf16x2(a.x * scale, a.y * scale);
    w.y = pack_bf16x2(a.z * scale, a.w * scale);
    w.z = pack_bf16x2(b.x * scale, b.y * scale);
    w.w = pack_bf16x2(b.z * scale, b.w * scale);
    reinterpret_cast<uint4*>(dQ)[i] = w;
  }
}

}  // namespace
}  // namespace lobra

using namespace lobra;

extern "C" size_t lobra_attn_workspace_bytes(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads) {
  if (num_seqs < 1 || !seq_lens || n_heads < 1) return 0;
  size_t items = 0;
  for (int s = 0; s < num_seqs; ++s) items += (size_t)((seq_lens[s] + A_TILE - 1) / A_TILE) * n_heads;
  return std::max<size_t>(256, items * sizeof(AttnItem));
}

extern "C" lobra_status lobra_attn_fwd(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                       int32_t n_kv_heads, int32_t head_dim, const void* Q, const void* K,
                                       const void* V, void* O, float* lse, void* ws, size_t ws_bytes,
                                       lobra_stream_t stream) {
  clear_error();
  if (num_seqs < 1 || !seq_lens || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads)
    return fail(LOBRA_ERR_INPUT, "attn: need num_seqs >= 1 and n_kv_heads | n_heads");
  if (head_dim != 128) return fail(LOBRA_ERR_UNSUPPORTED, "attn: head_dim %d (only 128)", head_dim);
  if (!Q || !K || !V || !O || !lse || !ws) return fail(LOBRA_ERR_INPUT, "attn: null pointer");
  if ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(V) |
       reinterpret_cast<uintptr_t>(O)) & 15)
    return fail(LOBRA_ERR_INPUT, "attn: pointers must be 16-byte aligned");
  // work items, longest first (the number of key tiles of a query tile is its index + 1)
  std::vector<AttnItem> items;
  long long T = 0;
  for (int s = 0; s < num_seqs; ++s) {
    if (seq_lens[s] < 0) return fail(LOBRA_ERR_INPUT, "attn: negative length");
    const int nt = (seq_lens[s] + A_TILE - 1) / A_TILE;
    for (int i = 0; i < nt; ++i)
      for (int h = 0; h < n_heads; ++h)
        items.push_back({(int)(T + i * A_TILE), (int)T, seq_lens[s], i, h});
    T += seq_lens[s];
  }
  if (T > (1LL << 31) - 1) return fail(LOBRA_ERR_INPUT, "attn: too many tokens");
  if (items.empty()) return LOBRA_OK;
  if (ws_bytes < items.size() * sizeof(AttnItem)) return fail(LOBRA_ERR_INPUT, "attn: workspace too small");
  std::stable_sort(items.begin(), items.end(), [](const AttnItem& a, const AttnItem& b) { return a.q_tile > b.q_tile; });
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // metadata through the library's pinned staging ring (k_meta_copy: no copy-engine
  // transfer, no host wait per call)
  if (upload_host_meta(items.data(), items.size() * sizeof(AttnItem), ws, st) != LOBRA_OK) return LOBRA_ERR_CUDA;
  CUtensorMap mQ, mK, mV;
  lobra_status s;
  if ((s = make_tensor_map_2d(&mQ, Q, (uint64_t)n_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_tensor_map_2d(&mK, K, (uint64_t)n_kv_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_tensor_map_2d(&mV, V, (uint64_t)n_kv_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  AttnArgs a;
  a.items = static_cast<const AttnItem*>(ws);
  a.nitems = (int)items.size();
  a.H = n_heads, a.Hkv = n_kv_heads, a.T = (int)T;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  a.O = static_cast<__nv_bfloat16*>(O);
  a.lse = lse;
  a.ts = nullptr;
  static const char* trace = getenv("LOBRA_TRACE_ATTN");
  static unsigned long long* d_ts = nullptr;
  if (trace) {
    if (!d_ts && cudaMalloc(&d_ts, 16 * 64 * sizeof(unsigned long long)) != cudaSuccess) d_ts = nullptr;
    if (d_ts) cudaMemsetAsync(d_ts, 0, 16 * 64 * sizeof(unsigned long long), st);
    a.ts = d_ts;
  }
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, A_SMEM);
    init = true;
  }
  count_launch(LOBRA_K_LAYER, st, true);
  k_attn_fwd<<<a.nitems, 384, A_SMEM, st>>>(mQ, mK, mV, a);
  count_launch(LOBRA_K_LAYER, st, false);
  if (a.ts) {   // tracing only: synchronous dump of CTA 0's phase stamps
    std::vector<unsigned long long> h(16 * 64);
    cudaMemcpyAsync(h.data(), a.ts, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* f = fopen(trace, "a")) {
      fprintf(f, "fwd\n");
      for (int e = 0; e < 16; ++e) {
        for (int t = 0; t < 64; ++t) fprintf(f, "%llu ", h[e * 64 + t]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "attn: %s", cudaGetErrorString(e));
  return LOBRA_OK;
}

namespace {
size_t attn_bwd_items(int32_t num_seqs, const int32_t* seq_lens, int32_t n_kv_heads) {
  size_t n = 0;
  for (int s = 0; s < num_seqs; ++s) n += (size_t)((std::max(seq_lens[s], 0) + A_TILE - 1) / A_TILE) * n_kv_heads;
  return n;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

extern "C" size_t lobra_attn_bwd_workspace_bytes(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                                 int32_t n_kv_heads) {
  if (num_seqs < 1 || !seq_lens || n_heads < 1 || n_kv_heads < 1) return 0;
  long long T = 0;
  for (int s = 0; s < num_seqs; ++s) T += std::max(seq_lens[s], 0);
  return align256(std::max<size_t>(256, attn_bwd_items(num_seqs, seq_lens, n_kv_heads) * sizeof(AttnBwdItem))) +
         align256((size_t)T * n_heads * sizeof(float)) + (size_t)T * n_heads * 128 * sizeof(float);
}

extern "C" lobra_status lobra_attn_bwd(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                       int32_t n_kv_heads, int32_t head_dim, const void* Q, const void* K,
                                       const void* V, const void* O, const void* dO, const float* lse, void* dQ,
                                       void* dK, void* dV, void* ws, size_t ws_bytes, lobra_stream_t stream) {
  clear_error();
  if (num_seqs < 1 || !seq_lens || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads)
    return fail(LOBRA_ERR_INPUT, "attn_bwd: need num_seqs >= 1 and n_kv_heads | n_heads");
  if (head_dim != 128) return fail(LOBRA_ERR_UNSUPPORTED, "attn_bwd: head_dim %d (only 128)", head_dim);
  if (!Q || !K || !V || !O || !dO || !lse || !dQ || !dK || !dV || !ws)
    return fail(LOBRA_ERR_INPUT, "attn_bwd: null pointer");
  if ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(V) |
       reinterpret_cast<uintptr_t>(O) | reinterpret_cast<uintptr_t>(dO) | reinterpret_cast<uintptr_t>(dQ) |
       reinterpret_cast<uintptr_t>(dK) | reinterpret_cast<uintptr_t>(dV) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return fail(LOBRA_ERR_INPUT, "attn_bwd: pointers must be 16-byte aligned");
  if (ws_bytes < lobra_attn_bwd_workspace_bytes(num_seqs, seq_lens, n_heads, n_kv_heads))
    return fail(LOBRA_ERR_INPUT, "attn_bwd: workspace too small");
  // work items (sequence, key tile, kv head), most query tiles first
  std::vector<AttnBwdItem> items;
  long long T = 0;
  for (int s = 0; s < num_seqs; ++s) {
    if (seq_lens[s] < 0) return fail(LOBRA_ERR_INPUT, "attn_bwd: negative length");
    const int nt = (seq_lens[s] + A_TILE - 1) / A_TILE;
    for (int j = 0; j < nt; ++j)
      for (int h = 0; h < n_kv_heads; ++h) items.push_back({(int)T, seq_lens[s], j, h});
    T += seq_lens[s];
  }
  if (T > (1LL << 31) - 1) return fail(LOBRA_ERR_INPUT, "attn_bwd: too many tokens");
  if (items.empty()) return LOBRA_OK;
  std::stable_sort(items.begin(), items.end(), [](const AttnBwdItem& a, const AttnBwdItem& b) {
    const int na = (a.len + A_TILE - 1) / A_TILE - a.k_tile, nb = (b.len + A_TILE - 1) / A_TILE - b.k_tile;
    return na > nb;
  });
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  const size_t items_bytes = align256(std::max<size_t>(256, attn_bwd_items(num_seqs, seq_lens, n_kv_heads) *
                                                                 sizeof(AttnBwdItem)));
  float* Dq = reinterpret_cast<float*>(w + items_bytes);
  float* acc = reinterpret_cast<float*>(w + items_bytes + align256((size_t)T * n_heads * sizeof(float)));
  if (upload_host_meta(items.data(), items.size() * sizeof(AttnBwdItem), ws, st) != LOBRA_OK)
    return LOBRA_ERR_CUDA;
  CUtensorMap mQ, mK, mV, mdO;
  lobra_status s;
  if ((s = make_tensor_map_2d(&mQ, Q, (uint64_t)n_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_tensor_map_2d(&mK, K, (uint64_t)n_kv_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_tensor_map_2d(&mV, V, (uint64_t)n_kv_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_tensor_map_2d(&mdO, dO, (uint64_t)n_heads * 128, (uint64_t)T, 64, 128)) != LOBRA_OK) return s;
  AttnBwdArgs a;
  a.items = reinterpret_cast<const AttnBwdItem*>(ws);
  a.H = n_heads, a.Hkv = n_kv_heads, a.T = (int)T;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  a.scale = 1.0f / sqrtf((float)head_dim);
  a.lse = lse;
  a.Dq = Dq;
  a.dq_acc = acc;
  a.dK = static_cast<__nv_bfloat16*>(dK);
  a.dV = static_cast<__nv_bfloat16*>(dV);
  a.ts = nullptr;
  static const char* trace = getenv("LOBRA_TRACE_ATTN");
  static unsigned long long* d_ts = nullptr;
  if (trace) {
    if (!d_ts && cudaMalloc(&d_ts, 16 * 64 * sizeof(unsigned long long)) != cudaSuccess) d_ts = nullptr;
    if (d_ts) cudaMemsetAsync(d_ts, 0, 16 * 64 * sizeof(unsigned long long), st);
    a.ts = d_ts;
  }
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, B_SMEM);
    init = true;
  }
  const long long warps = T * n_heads;
  count_launch(LOBRA_K_LAYER, st, true);
  k_attn_bwd_pre<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(O),
                                                                       static_cast<const __nv_bfloat16*>(dO),
                                                                       (int)T, n_heads, Dq, acc);
  count_launch(LOBRA_K_LAYER, st, false);
  count_launch(LOBRA_K_LAYER, st, true);
  k_attn_bwd<<<(unsigned)items.size(), 384, B_SMEM, st>>>(mQ, mK, mV, mdO, a);
  count_launch(LOBRA_K_LAYER, st, false);
  if (a.ts) {   // tracing only: synchronous dump of CTA 0's phase stamps
    std::vector<unsigned long long> h(16 * 64);
    cudaMemcpyAsync(h.data(), a.ts, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* f = fopen(trace, "a")) {
      fprintf(f, "bwd\n");
      for (int e = 0; e < 16; ++e) {
        for (int t = 0; t < 64; ++t) fprintf(f, "%llu ", h[e * 64 + t]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  const long long n8 = T * n_heads * 128 / 8;
  count_launch(LOBRA_K_LAYER, st, true);
  k_attn_bwd_post<<<(unsigned)std::min<long long>((n8 + 255) / 256, 148 * 16), 256, 0, st>>>(
      acc, n8, a.scale, static_cast<__nv_bfloat16*>(dQ));
  count_launch(LOBRA_K_LAYER, st, false);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "attn_bwd: %s", cudaGetErrorString(e));
  return LOBRA_OK;
}
