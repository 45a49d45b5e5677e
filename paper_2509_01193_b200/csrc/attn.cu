// Varlen causal attention forward on tcgen05 (the decoder layer's attention;
// block-diagonal causal mask over the packed batch).  head_dim 128, bf16 in/out,
// fp32 softmax, grouped-query heads.
//
// One CTA per work item (sequence, 128-query tile, head), items ordered longest first.
//   warp 0   TMA producer: the Q tile once, then K_j / V_j tiles (2-stage ring)
//   warp 1   MMA issuer:   S_j = Q K_j^T into TMEM (double buffered, 2 x 128 columns) while
//                          the softmax works on S_{j-1}; O_j = P_j V_j into a TMEM scratch
//   warp 2   TMEM allocator
//   warps 4-7 softmax, one query row per thread: row max of S_j (masked: key <= query and
//            inside the sequence), p = exp2(s log2e / sqrt(D) - m), P_j to shared memory
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
constexpr int A_KV_STAGES = 2;
constexpr int A_SMEM = A_TILE_BYTES /*Q*/ + A_KV_STAGES * 2 * A_TILE_BYTES /*K,V*/ + A_TILE_BYTES /*P*/ + 1024 + 256;

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
};

__device__ __forceinline__ float ex2(float x) {   // MUFU.EX2; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint8_t* align1024a(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__global__ void __launch_bounds__(256, 1)
    k_attn_fwd(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
               const __grid_constant__ CUtensorMap mapV, const AttnArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024a(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + A_TILE_BYTES;                       // stage s: K at +s*2T, V at +s*2T+T
  uint8_t* sP = sKV + A_KV_STAGES * 2 * A_TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + A_TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;     // [2]
  uint64_t* kv_empty = bars + 3;    // [2]
  uint64_t* s_full = bars + 5;      // [2]
  uint64_t* s_empty = bars + 7;     // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_full = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const uint32_t warp = warp_id(), lane = lane_id();
  const AttnItem it = args.items[blockIdx.x];
  const int nkv = it.q_tile + 1;                           // causal: key tiles 0..q_tile
  const int hk = it.head / (args.H / args.Hkv);

  if (warp == 0 && lane == 0) tma_prefetch(&mapQ), tma_prefetch(&mapK), tma_prefetch(&mapV);
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1), mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_expect_tx(q_full, A_TILE_BYTES);
      tma_load_2d(sQ, &mapQ, q_full, it.head * 128, it.q_row0);
      tma_load_2d(sQ + A_BOX, &mapQ, q_full, it.head * 128 + 64, it.q_row0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        mbar_wait(&kv_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], 2 * A_TILE_BYTES);
        uint8_t* k = sKV + s * 2 * A_TILE_BYTES;
        const int row = it.kv_row0 + j * A_TILE;
        tma_load_2d(k, &mapK, &kv_full[s], hk * 128, row);
        tma_load_2d(k + A_BOX, &mapK, &kv_full[s], hk * 128 + 64, row);
        tma_load_2d(k + A_TILE_BYTES, &mapV, &kv_full[s], hk * 128, row);
        tma_load_2d(k + A_TILE_BYTES + A_BOX, &mapV, &kv_full[s], hk * 128 + 64, row);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t id_s = idesc_bf16(128, 128, false, false);   // S: Q, K both K-major
      const uint32_t id_o = idesc_bf16(128, 128, false, true);    // O: P K-major, V MN-major
      const uint32_t q0 = smem_u32(sQ), p0 = smem_u32(sP);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        mbar_wait(&kv_full[s], (j >> 1) & 1);
        mbar_wait(&s_empty[s], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(sKV + s * 2 * A_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // K = head_dim 128: 2 swizzle atoms x 4 steps of 16
          const uint32_t off = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tmem + s * 128, sdesc_sw128(q0 + off, 16, 1024), sdesc_sw128(k0 + off, 16, 1024), id_s,
                   kk ? 1u : 0u);
        }
        mma_commit(&s_full[s]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        mbar_wait(p_full, j & 1);   // P_j written (and O rescaled if the softmax had to)
        tc_fence_after();
        const uint32_t v0 = smem_u32(sKV + (j & 1) * 2 * A_TILE_BYTES + A_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // K = 128 keys: P (K-major) x V (MN-major)
          const uint32_t poff = (kk >> 2) * A_BOX + (kk & 3) * 32;
          mma_bf16(tmem + 256, sdesc_sw128(p0 + poff, 16, 1024), sdesc_sw128(v0 + kk * 2048, A_BOX, 1024), id_o,
                   (j | kk) ? 1u : 0u);   // O accumulates in TMEM over the key tiles
        }
        mma_commit(o_full);
        mma_commit(&kv_empty[j & 1]);
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax / epilogue: one query row per thread
    // O accumulates in TMEM; P is computed against a reference max m that is raised (and O, l
    // rescaled in place) only when a tile's max exceeds it by more than 8 (log2 units, i.e.
    // p <= 256): the final O / l is exact either way.
    const int r = (warp - 4) * 32 + lane;
    const int qpos = it.q_tile * A_TILE + r;               // position inside the sequence
    const bool qvalid = qpos < it.len;
    const uint32_t trow = ((warp - 4) * 32u) << 16;
    // invalid rows (past the sequence end in its last tile) keep m = 0 and only see -inf
    float m = qvalid ? -INFINITY : 0.0f, l = 0.0f;
    // per-element masks only where a tile can hold masked keys: the diagonal tile and the
    // tiles reaching past the sequence end, plus every tile of a query tile with rows past it
    const bool tail_rows = (it.q_tile + 1) * A_TILE > it.len;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      const int kbase = j * A_TILE;
      float sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(tmem + trow + sb * 128 + c * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) sv[c * 32 + e] = v[e];
      }
      tc_fence_before();
      mbar_arrive(&s_empty[sb]);                             // S buffer free for S_{j+2}
      if (j == nkv - 1 || tail_rows || kbase + A_TILE > it.len) {   // warp-uniform
#pragma unroll
        for (int e = 0; e < 128; ++e) {
          const int kpos = kbase + e;
          if (!(qvalid && kpos <= qpos && kpos < it.len)) sv[e] = -INFINITY;
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 128; ++e) mx = fmaxf(mx, sv[e]);
      mx *= args.scale_log2;                                  // scale > 0: max commutes
      // the previous P V is complete (O quiescent, P buffer free) before P_j is written
      if (j >= 1) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
      }
      // raise the reference max where needed; the TMEM rescale is warp-collective
      // (tcgen05.ld / st are .sync.aligned): every lane takes part, alpha = 1 where unchanged
      const bool raise = qvalid && (j == 0 || mx > m + 8.0f);
      const float m_new = raise ? fmaxf(m, mx) : m;
      const float alpha = (raise && j >= 1) ? ex2(m - m_new) : 1.0f;
      if (j >= 1 && __any_sync(0xffffffffu, raise)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(tmem + trow + 256 + c * 32, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] *= alpha;
          tmem_st32(tmem + trow + 256 + c * 32, v);
        }
      }
      l *= alpha;
      m = m_new;
      float sum = 0.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float p[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          p[e] = ex2(fmaf(sv[c * 32 + e], args.scale_log2, -m));   // masked: ex2(-inf) = 0
          sum += p[e];
        }
        uint8_t* atom = sP + (c >> 1) * A_BOX + r * 128;     // 64 keys per 128-byte swizzle atom row
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = (c & 1) * 4 + u;                 // 16-byte chunk within the 128-byte row
          uint4 w;
          w.x = pack_bf16x2(p[u * 8 + 0], p[u * 8 + 1]);
          w.y = pack_bf16x2(p[u * 8 + 2], p[u * 8 + 3]);
          w.z = pack_bf16x2(p[u * 8 + 4], p[u * 8 + 5]);
          w.w = pack_bf16x2(p[u * 8 + 6], p[u * 8 + 7]);
          *reinterpret_cast<uint4*>(atom + ((chunk ^ (r & 7)) << 4)) = w;
        }
      }
      l += sum;
      tc_fence_before();
      fence_proxy_async_smem();   // P stores visible to the tensor core
      mbar_arrive(p_full);
    }
    mbar_wait(o_full, (nkv - 1) & 1);
    tc_fence_after();
    const float inv = qvalid ? 1.0f / l : 0.0f;
    const size_t tok = (size_t)it.q_row0 + r;
    uint4* dst = reinterpret_cast<uint4*>(args.O + tok * (size_t)(args.H * 128) + it.head * 128);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float v[32];
      tmem_ld32(tmem + trow + 256 + c * 32, v);            // warp-collective: every lane
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
    if (qvalid) args.lse[(size_t)it.head * args.T + tok] = (m + log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
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
  // metadata through a persistent pinned staging buffer (the previous copy from it is
  // waited for before it is overwritten)
  static void* pinned = nullptr;
  static size_t pinned_bytes = 0;
  static cudaEvent_t done = nullptr;
  const size_t bytes = items.size() * sizeof(AttnItem);
  if (!done && cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "attn: event creation failed");
  cudaEventSynchronize(done);
  if (pinned_bytes < bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned_bytes = std::max<size_t>(bytes, 1 << 16);
    if (cudaMallocHost(&pinned, pinned_bytes) != cudaSuccess) {
      pinned = nullptr, pinned_bytes = 0;
      return fail(LOBRA_ERR_CUDA, "attn: pinned allocation failed");
    }
  }
  memcpy(pinned, items.data(), bytes);
  if (cudaMemcpyAsync(ws, pinned, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "attn: metadata upload failed");
  cudaEventRecord(done, st);
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
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, A_SMEM);
    init = true;
  }
  count_launch(LOBRA_K_LAYER, st, true);
  k_attn_fwd<<<a.nitems, 256, A_SMEM, st>>>(mQ, mK, mV, a);
  count_launch(LOBRA_K_LAYER, st, false);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "attn: %s", cudaGetErrorString(e));
  return LOBRA_OK;
}
