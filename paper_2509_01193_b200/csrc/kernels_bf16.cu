// bf16 kernels of the multi-LoRA hot path for sm_100a (tcgen05 + TMEM + TMA).
//
// k_gemm2    : 2-CTA (cta_group::2, 256 x 256 per CTA pair) persistent GEMM:
//              C = Z W^T (fwd) or Z W (bwd, W as an MN-major operand) with the LoRA
//              expand fused into the SAME TMEM accumulator as extra K steps over the
//              tile's adapter slots ("K-extension"): "the computation of the base
//              model can be fused into a batched operation whilst ... multiple LoRA
//              adapters ... customized operations".
// k_shrink   : the forward rank-r shrink H_s = s_t X A_t^T, HBM-bound: one CTA per slot (or
//              per tile) over the whole K, deep TMA ring, the slots of a tile as one MMA.
// k_shrink_planes: the same for wide projection groups (every projection's H_s from one X
//              pass, MMA N = np * qp), separate X / adapter rings.
// k_rowproj  : the same with split-K over CTAs (small batches; the unfused backward G_s).
// k_dypass   : the fused backward dY pass: G_s = s_t dY B_t partials and dB_t partials from
//              ONE read of dY (static schedule weighted by the measured per-entry cost);
//              k_gfin writes the G slots.
// k_segred   : the token reductions dA_t = X^T G_s (and unfused dB_t = dY^T H_s) on tensor
//              cores, Z tiles used as MN-major A operands (one HBM read of Z), static balanced
//              schedule, deterministic two-pass (segment partials + k_finalize_multi).
// See DESIGN.md "Kernels" for layouts and the roofline of each.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>
#include <cstdio>

#include "lora_internal.h"
#include "ptx.cuh"

namespace lobra {
using namespace ptx;

namespace {

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ int rpad16(int r) { return (r + 15) & ~15; }

constexpr int G_THREADS = 256;

// =====================================================================================
// 2-CTA GEMM with fused K-extension (cta_group::2): a CTA pair computes a 256 x 256 tile,
// each CTA loads its own 128 rows of A and HALF (128 columns) of B, the leader issues
// tcgen05.mma.cta_group::2 (M = 256) and each CTA drains its 128 accumulator rows.
// Per CTA and K step: 32 KB of operands for 128 x 256 outputs (a 1-CTA 128 x 256 tile needs
// 48 KB) -> two thirds of the L2->SM operand traffic.
// K-extension across the pair: the union of the two M tiles' tasks; a CTA whose tile lacks
// a task feeds the all-zero slot (index meta.nslots) for that step.
// =====================================================================================
constexpr int P_BK = 64, P_STAGES = 6;
constexpr int P_A_BYTES = 128 * P_BK * 2;    // 16 KB: this CTA's 128 rows
constexpr int P_B_BYTES = 128 * P_BK * 2;    // 16 KB: this CTA's half of the 256 B columns
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_SMEM = P_STAGES * P_STAGE_BYTES + 1024 + 256;

struct Gemm2Args {
  int T, N, K, ntm2, ntn, accumulate, group_m;
  __nv_bfloat16* C;
  Meta meta;
  TpScatter tp;   // tp.peer != nullptr: fused GEMM -> reduce-scatter over peer memory
};

__device__ __forceinline__ int tile_slot_begin(const Meta& m, int tile) {
  return tile < m.ntiles ? m.tile_slot_off[tile] : 0;
}
__device__ __forceinline__ int tile_slot_end(const Meta& m, int tile) {
  return tile < m.ntiles ? m.tile_slot_off[tile + 1] : 0;
}
// slot of `task` in `tile`, or the zero slot
__device__ __forceinline__ int find_slot(const Meta& m, int tile, int task) {
  for (int s = tile_slot_begin(m, tile); s < tile_slot_end(m, tile); ++s)
    if (m.slot_task[s] == task) return s;
  return m.nslots;
}

// Calls f(task, my_slot) for the union of the pair's tasks (tile A's order, then tile B's
// new tasks); identical sequence in both CTAs.
template <typename F>
__device__ __forceinline__ void for_union(const Meta& m, int tA, int tB, uint32_t rank, F&& f) {
  for (int s = tile_slot_begin(m, tA); s < tile_slot_end(m, tA); ++s) {
    const int t = m.slot_task[s];
    f(t, rank == 0 ? s : find_slot(m, tB, t));
  }
  for (int s = tile_slot_begin(m, tB); s < tile_slot_end(m, tB); ++s) {
    const int t = m.slot_task[s];
    if (find_slot(m, tA, t) != m.nslots) continue;
    f(t, rank == 1 ? s : m.nslots);
  }
}

// Pair-tile order: groups of `group_m` pair-M blocks, N-major inside a group, so that the
// concurrently running clusters share a few X panels AND a few W panels (both stay in L2).
// group_m < 0: the transpose -- groups of -group_m N blocks, M-major inside a group.
__device__ __forceinline__ void pair_tile(int pt, int ntm2, int ntn, int group_m, int& mp, int& n) {
  if (group_m < -1) {
    const int gn_ = -group_m;
    const int per_group = gn_ * ntm2;
    const int g = pt / per_group, r = pt % per_group;
    const int gn = min(gn_, ntn - g * gn_);
    n = g * gn_ + r % gn;
    mp = r / gn;
    return;
  }
  if (group_m <= 1) {
    mp = pt / ntn, n = pt % ntn;
    return;
  }
  const int per_group = group_m * ntn;
  const int g = pt / per_group, r = pt % per_group;
  const int gm = min(group_m, ntm2 - g * group_m);   // the last group may be short
  mp = g * group_m + r % gm;
  n = r / gm;
}

template <bool kBMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G_THREADS, 1)
    k_gemm2(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW,
            const __grid_constant__ CUtensorMap mapSlot, const __grid_constant__ CUtensorMap mapV,
            const Gemm2Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + P_STAGES * P_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + P_STAGES * P_B_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapZ);
    tma_prefetch(&mapW);
    tma_prefetch(&mapSlot);
    tma_prefetch(&mapV);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < P_STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 8);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  const int npt = args.ntm2 * args.ntn;
  const int nk = (args.K + P_BK - 1) / P_BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const Meta& meta = args.meta;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int pt = cid; pt < npt; pt += ncl) {
        int mp, n;
        pair_tile(pt, args.ntm2, args.ntn, args.group_m, mp, n);
        const int m = 2 * mp + rank;
        const int ncol = n * 256 + rank * 128;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = mapa(smem_u32(&full[stage]), 0);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
          tma_load_2d_pair(sA + stage * P_A_BYTES, &mapZ, fb, kb * P_BK, m * 128);
          if (!kBMN) {
            tma_load_2d_pair(sB + stage * P_B_BYTES, &mapW, fb, kb * P_BK, ncol);
          } else {
            tma_load_2d_pair(sB + stage * P_B_BYTES, &mapW, fb, ncol, kb * P_BK);
            tma_load_2d_pair(sB + stage * P_B_BYTES + 8192, &mapW, fb, ncol + 64, kb * P_BK);
          }
          if (++stage == P_STAGES) stage = 0, phase ^= 1;
        }
        for_union(meta, 2 * mp, 2 * mp + 1, rank, [&](int t, int my_slot) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = mapa(smem_u32(&full[stage]), 0);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
          tma_load_2d_pair(sA + stage * P_A_BYTES, &mapSlot, fb, 0, my_slot * kTileM);
          if (!kBMN) {
            tma_load_2d_pair(sB + stage * P_B_BYTES, &mapV, fb, meta.boff[t], ncol);
          } else {
            tma_load_2d_pair(sB + stage * P_B_BYTES, &mapV, fb, ncol, meta.roff[t]);
            tma_load_2d_pair(sB + stage * P_B_BYTES + 8192, &mapV, fb, ncol + 64, meta.roff[t]);
          }
          if (++stage == P_STAGES) stage = 0, phase ^= 1;
        });
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader CTA only)
      const uint32_t id = idesc_bf16(256, 256, false, kBMN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int pt = cid; pt < npt; pt += ncl, ++it) {
        int mp, n_unused;
        pair_tile(pt, args.ntm2, args.ntn, args.group_m, mp, n_unused);
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * P_A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * P_B_BYTES);
#pragma unroll
          for (int k = 0; k < P_BK / 16; ++k) {
            const uint64_t bd = kBMN ? sdesc_sw128(b0 + k * 2048, 8192, 1024)
                                     : sdesc_sw128(b0 + k * 32, 16, 1024);
            mma_bf16_pair(d, sdesc_sw128(a0 + k * 32, 16, 1024), bd, id, (kb | k) != 0);
          }
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == P_STAGES) stage = 0, phase ^= 1;
        }
        for_union(meta, 2 * mp, 2 * mp + 1, 0, [&](int t, int) {
          const int nk16 = rpad16(meta.ranks[t]) / 16;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * P_A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * P_B_BYTES);
          for (int k = 0; k < nk16; ++k) {
            const uint64_t bd = kBMN ? sdesc_sw128(b0 + k * 2048, 8192, 1024)
                                     : sdesc_sw128(b0 + k * 32, 16, 1024);
            // the slot's columns [band, band + 16 nk16) hold this projection's H_s / G_s
            mma_bf16_pair(d, sdesc_sw128(a0 + (meta.band / 16 + k) * 32, 16, 1024), bd, id, 1u);
          }
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == P_STAGES) stage = 0, phase ^= 1;
        });
        mma_commit_pair(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs): own 128 rows
    const uint32_t q = warp - 4;
    int it = 0;
    for (int pt = cid; pt < npt; pt += ncl, ++it) {
      int mp, n;
      pair_tile(pt, args.ntm2, args.ntn, args.group_m, mp, n);
      const int m = 2 * mp + rank;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = m * 128 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        float v[32];
        tmem_ld32(tmem + ((q * 32u) << 16) + acc * 256 + c * 32, v);
        const int col0 = n * 256 + c * 32;
        if (row < args.T && col0 < args.N) {
          // fused TP reduce-scatter: row r goes to its owner rank (r / chunk) into the slot of
          // this rank -- a store over NVLink that overlaps the next tile's MMAs
          __nv_bfloat16* crow =
              args.tp.peer ? reinterpret_cast<__nv_bfloat16*>(args.tp.peer[row / args.tp.chunk_rows] + args.tp.data_off) +
                                 ((size_t)args.tp.rank * args.tp.chunk_rows + row % args.tp.chunk_rows) * args.N
                           : args.C + (size_t)row * args.N;
          uint4* dst = reinterpret_cast<uint4*>(crow + col0);
          if (args.accumulate) {
            // accumulate onto the LOCAL partial in C (with the fused reduce-scatter the
            // accumulated row then goes to its owner)
            const uint4* src = reinterpret_cast<const uint4*>(args.C + (size_t)row * args.N + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 o = src[j];
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                v[j * 8 + 2 * e] += f.x;
                v[j * 8 + 2 * e + 1] += f.y;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 o;
            o.x = pack_bf16x2(v[j * 8 + 0], v[j * 8 + 1]);
            o.y = pack_bf16x2(v[j * 8 + 2], v[j * 8 + 3]);
            o.z = pack_bf16x2(v[j * 8 + 4], v[j * 8 + 5]);
            o.w = pack_bf16x2(v[j * 8 + 6], v[j * 8 + 7]);
            dst[j] = o;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa(smem_u32(&tempty[acc]), 0));
    }
  }
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// =====================================================================================
// Row projection (shrink): slot[s][row][q] = s_t * sum_k Z[row][k] V_t(q, k)
//   kVmn = false: V_t rows of A_cat [rsum, K] (K-major; forward H_s = s X A_t^T)
//   kVmn = true : V_t = columns of B_cat [K, rsum8] (MN-major; backward G_s = s dY B_t)
// The 64-wide operand box starts at the task's roff; columns q >= r_t (other tasks'
// data or OOB zeros) are masked to exact zeros in the epilogue.  HBM-bound: split-K
// over `nsplit` CTAs per tile when the tile count cannot fill the GPU, partials reduced
// in fixed split order by the last CTA to arrive (deterministic).
// =====================================================================================
constexpr int R_A_BYTES = 128 * 64 * 2;          // 16 KB
constexpr int R_V_BYTES = 64 * 64 * 2;           // 8 KB per slot
template <int STAGES, int P, int KB = 1>
constexpr int r_smem() { return STAGES * KB * (R_A_BYTES + P * R_V_BYTES) + 1024 + 256; }

struct RowArgs {
  int K, nsplit, kb_per_split, dbg_no_mma, prefetch, interleave;
  __nv_bfloat16* out;
  float* partial;     // [nsplit][nslots][128][64] fp32 (only when nsplit > 1)
  int* counters;      // [ntiles], zero on entry; reset by the last CTA
  Meta meta;
};

__device__ __forceinline__ void store_slot_row(__nv_bfloat16* out, int s, int lrow, const float* v,
                                               float sc, int rp) {
  uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)s * kTileM + lrow) * kSlotW);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = (j * 8 + e < rp) ? v[j * 8 + e] * sc : 0.0f;
    uint4 o;
    o.x = pack_bf16x2(w[0], w[1]);
    o.y = pack_bf16x2(w[2], w[3]);
    o.z = pack_bf16x2(w[4], w[5]);
    o.w = pack_bf16x2(w[6], w[7]);
    dst[j] = o;
  }
}

template <bool kVmn, int R_STAGES, int R_P, int R_KB>
__global__ void __launch_bounds__(256, 1)
    k_rowproj(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapV,
              const RowArgs args) {
  // one stage = R_KB consecutive 64-column K blocks: [Z box x R_KB][V slot i box x R_KB]...
  constexpr int R_STAGE_BYTES = R_KB * (R_A_BYTES + R_P * R_V_BYTES);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + R_STAGES * R_STAGE_BYTES);
  uint64_t* empty = full + R_STAGES;
  uint64_t* tfull = empty + R_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;
  const int m = blockIdx.x / args.nsplit, split = blockIdx.x % args.nsplit;
  const int s_begin = meta.tile_slot_off[m], s_end = meta.tile_slot_off[m + 1];
  const int npass = (s_end - s_begin + R_P - 1) / R_P;
  const int nk = (args.K + 63) / 64;
  const int kb0 = split * args.kb_per_split, kb1 = min(nk, kb0 + args.kb_per_split);

  if (warp == 0 && lane == 0) tma_prefetch(&mapZ), tma_prefetch(&mapV);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < R_STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int p = 0; p < npass; ++p) {
        const int s0 = s_begin + p * R_P;
        const int ns = min(R_P, s_end - s0);
        for (int kk = kb0; kk < kb1; kk += R_KB) {
          // interleaved: this split takes K blocks split, split + nsplit, ... so that the
          // CTAs of one tile read adjacent column blocks of the same rows concurrently
          const int kb = args.interleave ? split + (kk - kb0) * args.nsplit : kk;
          if (kb >= nk) break;
          const int nkb = args.interleave ? 1 : min(R_KB, kb1 - kk);
          mbar_wait(&empty[stage], phase ^ 1);
          const bool nov = (args.dbg_no_mma & 2) != 0;   // probe: skip the adapter boxes
          mbar_expect_tx(&full[stage], nkb * (R_A_BYTES + (nov ? 0 : ns) * R_V_BYTES));
          uint8_t* st = smem + stage * R_STAGE_BYTES;
          if (args.prefetch && !args.interleave)   // stream the Z tile into L2 ahead
            for (int j = 0; j < nkb; ++j)
              if (kb + j + args.prefetch < kb1)
                tma_prefetch_2d(&mapZ, (kb + j + args.prefetch) * 64, m * kTileM);
          for (int j = 0; j < nkb; ++j)
            tma_load_2d(st + j * R_A_BYTES, &mapZ, &full[stage], (kb + j) * 64, m * kTileM);
          for (int i = 0; i < (nov ? 0 : ns); ++i) {
            const int t = meta.slot_task[s0 + i];
            for (int j = 0; j < nkb; ++j) {
              uint8_t* vd = st + R_KB * R_A_BYTES + (i * R_KB + j) * R_V_BYTES;
              if (kVmn)   // B operand [out, ld8], columns boff..boff+63 (MN-major)
                tma_load_2d(vd, &mapV, &full[stage], meta.boff[t], (kb + j) * 64);
              else        // A_cat [rsum, in], rows roff..roff+63 (K-major)
                tma_load_2d(vd, &mapV, &full[stage], (kb + j) * 64, meta.roff[t]);
            }
          }
          if (++stage == R_STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = idesc_bf16(128, 64, false, kVmn);
      int stage = 0;
      uint32_t phase = 0;
      for (int p = 0; p < npass; ++p) {
        const int s0 = s_begin + p * R_P;
        const int ns = min(R_P, s_end - s0);
        mbar_wait(tempty, (p & 1) ^ 1);
        tc_fence_after();
        for (int kk = kb0; kk < kb1; kk += R_KB) {
          const int kb = args.interleave ? split + (kk - kb0) * args.nsplit : kk;
          if (kb >= nk) break;
          const int nkb = args.interleave ? 1 : min(R_KB, kb1 - kk);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st0 = smem_u32(smem + stage * R_STAGE_BYTES);
          if (args.dbg_no_mma & 1) {   // tuning probe: pure TMA streaming, no tensor work
            mbar_arrive(&empty[stage]);
            if (++stage == R_STAGES) stage = 0, phase ^= 1;
            continue;
          }
          for (int i = 0; i < ns; ++i) {
            for (int j = 0; j < nkb; ++j) {
              const uint32_t a0 = st0 + j * R_A_BYTES;
              const uint32_t b0 = st0 + R_KB * R_A_BYTES + (i * R_KB + j) * R_V_BYTES;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t bd = kVmn ? sdesc_sw128(b0 + k * 2048, 8192, 1024)
                                         : sdesc_sw128(b0 + k * 32, 16, 1024);
                mma_bf16(tmem + i * 64, sdesc_sw128(a0 + k * 32, 16, 1024), bd, id,
                         (kk != kb0 || j != 0 || k != 0) ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty[stage]);
          if (++stage == R_STAGES) stage = 0, phase ^= 1;
        }
        mma_commit(tfull);
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;
    const int lrow = q * 32 + lane;
    const int row = m * kTileM + lrow;
    const int my_task = row < meta.T ? row_task(meta, row) : -1;
    if (blockIdx.x == 0) {   // the all-zero slot (index nslots) used by the 2-CTA GEMM
      float z[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) z[j] = 0.0f;
      store_slot_row(args.out, meta.nslots, lrow, z, 0.0f, 0);
    }
    for (int p = 0; p < npass; ++p) {
      const int s0 = s_begin + p * R_P;
      const int ns = min(R_P, s_end - s0);
      mbar_wait(tfull, p & 1);
      tc_fence_after();
      for (int i = 0; i < ((args.dbg_no_mma & 4) ? 0 : ns); ++i) {   // bit 2: probe, no output
        const int s = s0 + i;
        const int ts = meta.slot_task[s];
        float v[64];
        tmem_ld32(tmem + ((q * 32u) << 16) + i * 64, *reinterpret_cast<float(*)[32]>(v));
        tmem_ld32(tmem + ((q * 32u) << 16) + i * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
        if (args.nsplit == 1) {
          const bool mine = ts == my_task;
          store_slot_row(args.out, s, lrow, v, mine ? meta.scales[ts] : 0.0f, mine ? meta.ranks[ts] : 0);
        } else {
          const int rp = rpad16(meta.ranks[ts]);
          float4* dst = reinterpret_cast<float4*>(
              args.partial + (((size_t)split * meta.nslots + s) * kTileM + lrow) * 64);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (4 * j < rp) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
    if (args.nsplit > 1 && !(args.dbg_no_mma & 4)) {
      // deterministic split-K reduction by the last CTA of this tile to finish
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lrow == 0) *last_flag = (atomicAdd(&args.counters[m], 1) == args.nsplit - 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int s = s_begin; s < s_end; ++s) {
          const int ts = meta.slot_task[s];
          const int rp = rpad16(meta.ranks[ts]);
          float v[64];
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] = 0.0f;
          for (int sp = 0; sp < args.nsplit; ++sp) {
            const float4* src = reinterpret_cast<const float4*>(
                args.partial + (((size_t)sp * meta.nslots + s) * kTileM + lrow) * 64);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (4 * j >= rp) break;
              const float4 f = __ldcg(src + j);
              v[4 * j] += f.x, v[4 * j + 1] += f.y, v[4 * j + 2] += f.z, v[4 * j + 3] += f.w;
            }
          }
          const bool mine = ts == my_task;
          store_slot_row(args.out, s, lrow, v, mine ? meta.scales[ts] : 0.0f, mine ? meta.ranks[ts] : 0);
        }
        if (lrow == 0) args.counters[m] = 0;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// =====================================================================================
// Row projection with an LDGSTS producer: 4 producer warps stream Z with 16-byte cp.async,
// each warp reading KB x 128 contiguous bytes of a row per instruction and writing the
// 128-byte-swizzled K-major UMMA layout directly; the adapter operand (K-major, qp rows:
// A_cat for the forward, B^T for the backward) comes by TMA.  Same math, epilogue and
// split-K reduction as k_rowproj.  Warps: 0-3 producers, 4-7 epilogue, 8 MMA + TMEM.
// =====================================================================================
struct RowLdArgs {
  const __nv_bfloat16* Z;
  int K, nsplit, kb_per_split, qp;
  __nv_bfloat16* out;
  float* partial;
  int* counters;
  Meta meta;
};

template <int STAGES, int KB>
__global__ void __launch_bounds__(288, 1)
    k_rowproj_ld(const __grid_constant__ CUtensorMap mapV, const RowLdArgs args) {
  constexpr int P = 2;                           // slots per pass
  constexpr int ZB = KB * R_A_BYTES;             // Z bytes per stage
  const int vbox = args.qp * 128;                // one K block of one slot's operand
  const int stage_bytes = ZB + P * KB * vbox;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;
  const int m = blockIdx.x / args.nsplit, split = blockIdx.x % args.nsplit;
  const int s_begin = meta.tile_slot_off[m], s_end = meta.tile_slot_off[m + 1];
  const int npass = (s_end - s_begin + P - 1) / P;
  const int nk = (args.K + 63) / 64;
  const int kb0 = split * args.kb_per_split, kb1 = min(nk, kb0 + args.kb_per_split);

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mapV);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 128 + 1), mbar_init(&empty[s], 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp < 4) {  // ---------------- LDGSTS producers (128 threads)
    constexpr int LPR = KB * 8 < 32 ? KB * 8 : 32;   // lanes per row
    constexpr int RPI = 32 / LPR;                    // rows per instruction
    const int pt = threadIdx.x;
    const int c = lane % LPR;                        // 16-byte chunk within the row segment
    const int b = c >> 3, j = c & 7;                 // K block, chunk in 128 B
    int stage = 0;
    uint32_t phase = 0;
    int g = 0;                                       // stages issued
    for (int p = 0; p < npass; ++p) {
      const int s0 = s_begin + p * P;
      const int ns = min(P, s_end - s0);
      for (int kb = kb0; kb < kb1; kb += KB, ++g) {
        const int nkb = min(KB, kb1 - kb);
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * stage_bytes;
        const uint32_t zb = smem_u32(st);
        for (int it = 0; it < 32 / RPI; ++it) {
          const int r = warp * 32 + it * RPI + lane / LPR;
          const int row = m * kTileM + r;
          const int col = (kb + b) * 64 + j * 8;
          const bool ok = row < meta.T && b < nkb && col < args.K;
          const __nv_bfloat16* src = args.Z + (ok ? (size_t)row * args.K + col : 0);
          cp_async16(zb + b * R_A_BYTES + r * 128 + ((j ^ (r & 7)) << 4), src, ok ? 16u : 0u);
        }
        cp_async_commit();
        if (pt == 0) {   // adapter operand by TMA, counted on the same barrier
          mbar_expect_tx(&full[stage], ns * nkb * vbox);
          for (int i = 0; i < ns; ++i) {
            const int t = meta.slot_task[s0 + i];
            for (int q = 0; q < nkb; ++q)
              tma_load_2d(st + ZB + (i * KB + q) * vbox, &mapV, &full[stage], (kb + q) * 64,
                          meta.roff[t]);
          }
        }
        if (g >= STAGES - 1) {   // the stage issued STAGES-1 steps ago has landed
          cp_async_wait<STAGES - 1>();
          fence_proxy_async_smem();
          const int sd = (stage + 1) % STAGES;   // == (g - (STAGES - 1)) % STAGES
          mbar_arrive(&full[sd]);
        }
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
    }
    // drain: signal the last min(g, STAGES-1) stages
    cp_async_wait<0>();
    fence_proxy_async_smem();
    const int pending = g < STAGES - 1 ? g : STAGES - 1;
    for (int k = pending; k >= 1; --k) mbar_arrive(&full[(stage - k + STAGES) % STAGES]);
  } else if (warp == 8) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t id = idesc_bf16(128, args.qp, false, false);
      int stage = 0;
      uint32_t phase = 0;
      for (int p = 0; p < npass; ++p) {
        const int s0 = s_begin + p * P;
        const int ns = min(P, s_end - s0);
        mbar_wait(tempty, (p & 1) ^ 1);
        tc_fence_after();
        for (int kb = kb0; kb < kb1; kb += KB) {
          const int nkb = min(KB, kb1 - kb);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st0 = smem_u32(smem + stage * stage_bytes);
          for (int i = 0; i < ns; ++i)
            for (int q = 0; q < nkb; ++q) {
              const uint32_t a0 = st0 + q * R_A_BYTES;
              const uint32_t b0 = st0 + ZB + (i * KB + q) * vbox;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16(tmem + i * 64, sdesc_sw128(a0 + k * 32, 16, 1024),
                         sdesc_sw128(b0 + k * 32, 16, 1024), id,
                         (kb != kb0 || q != 0 || k != 0) ? 1u : 0u);
            }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        mma_commit(tfull);
      }
    }
  } else {  // ---------------- epilogue (warps 4-7)
    const uint32_t q = warp - 4;
    const int lrow = q * 32 + lane;
    const int row = m * kTileM + lrow;
    const int my_task = row < meta.T ? row_task(meta, row) : -1;
    if (blockIdx.x == 0) {
      float z[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) z[i] = 0.0f;
      store_slot_row(args.out, meta.nslots, lrow, z, 0.0f, 0);
    }
    for (int p = 0; p < npass; ++p) {
      const int s0 = s_begin + p * P;
      const int ns = min(P, s_end - s0);
      mbar_wait(tfull, p & 1);
      tc_fence_after();
      for (int i = 0; i < ns; ++i) {
        const int s = s0 + i;
        const int ts = meta.slot_task[s];
        float v[64];
        tmem_ld32(tmem + ((q * 32u) << 16) + i * 64, *reinterpret_cast<float(*)[32]>(v));
        tmem_ld32(tmem + ((q * 32u) << 16) + i * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
        if (args.nsplit == 1) {
          const bool mine = ts == my_task;
          store_slot_row(args.out, s, lrow, v, mine ? meta.scales[ts] : 0.0f, mine ? meta.ranks[ts] : 0);
        } else {
          const int rp = rpad16(meta.ranks[ts]);
          float4* dst = reinterpret_cast<float4*>(
              args.partial + (((size_t)split * meta.nslots + s) * kTileM + lrow) * 64);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (4 * jj < rp) dst[jj] = make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
    if (args.nsplit > 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lrow == 0) *last_flag = (atomicAdd(&args.counters[m], 1) == args.nsplit - 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int s = s_begin; s < s_end; ++s) {
          const int ts = meta.slot_task[s];
          const int rp = rpad16(meta.ranks[ts]);
          float v[64];
#pragma unroll
          for (int jj = 0; jj < 64; ++jj) v[jj] = 0.0f;
          for (int sp = 0; sp < args.nsplit; ++sp) {
            const float4* src = reinterpret_cast<const float4*>(
                args.partial + (((size_t)sp * meta.nslots + s) * kTileM + lrow) * 64);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              if (4 * jj >= rp) break;
              const float4 f = __ldcg(src + jj);
              v[4 * jj] += f.x, v[4 * jj + 1] += f.y, v[4 * jj + 2] += f.z, v[4 * jj + 3] += f.w;
            }
          }
          const bool mine = ts == my_task;
          store_slot_row(args.out, s, lrow, v, mine ? meta.scales[ts] : 0.0f, mine ? meta.ranks[ts] : 0);
        }
        if (lrow == 0) args.counters[m] = 0;
      }
    }
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// =====================================================================================
// Forward shrink, one CTA per 128-row tile and the whole K (no split-K, no partials):
// slot[s][row][q] = s_t sum_k X[row][k] A(q, k).  Persistent over tiles when there are more
// tiles than SMs.  A stage is SH_KB adjacent 64-column K blocks of the X tile (2 x 16 KB
// boxes) plus, per slot of the pass, the matching qv-row boxes of the adapter operand
// (qv = rows the tile's tasks need: the padded rank, or np*qp for a projection group; rows
// past a task's rank are masked in the epilogue).  The stage count fills the shared memory
// (one CTA per SM), so ~200 KB of X is in flight per SM: HBM-bound streaming at the copy
// roofline needs bytes in flight, not more CTAs (profiles/r1e_shrink.md).
// Accumulators: two TMEM buffers of SH_P x 64 columns, so the epilogue of one tile overlaps
// the streaming of the next.
// =====================================================================================
constexpr int SH_KB = 2, SH_P = 4;
struct ShrinkArgs {
  int K, qv, stages, stage_bytes, P;
  int kb;          // 64-column K blocks per stage (2; 1 when the adapter operand is wide)
  // planes mode (a projection group whose bands exceed the 64-wide slot, np * qp > 64): the
  // accumulator's columns [p pq, p pq + pq) go to plane p (out + p * plane_stride), each plane
  // an ordinary single-projection slot buffer; rk / sc = the tasks' real ranks / scales
  int nplanes, pq;
  long long plane_stride;
  const int* rk;
  const float* sc;
  int per_slot;   // 1: one work item per slot (X tile re-read for every task of a mixed tile;
                  //    equal work per CTA, used when the slots fit in one wave), 0: per tile
  __nv_bfloat16* out;
  unsigned long long* ts;   // probe (LOBRA_DBG_SHRINK_TS): per CTA globaltimer stamps, else null
  Meta meta;
};
// work item w -> tile m and its slot range
__device__ __forceinline__ void shrink_item(const Meta& meta, int per_slot, int w, int& m, int& s_begin,
                                            int& s_end) {
  if (per_slot) {
    m = meta.slot_tile[w], s_begin = w, s_end = w + 1;
  } else {
    m = w, s_begin = meta.tile_slot_off[w], s_end = meta.tile_slot_off[w + 1];
  }
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256, 1)
    k_shrink(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapV,
             const ShrinkArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = args.stages, SB = args.stage_bytes, P = args.P, qv = args.qv, KB = args.kb;
  const int vbox = qv * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SB);
  uint64_t* empty = full + 8;
  uint64_t* tfull = empty + 8;      // [2]
  uint64_t* tempty = tfull + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;
  const int nk = (args.K + 63) / 64;
  const int nitems = args.per_slot ? meta.nslots : meta.ntiles;

  if (warp == 0 && lane == 0) tma_prefetch(&mapZ), tma_prefetch(&mapV);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&tfull[b], 1), mbar_init(&tempty[b], 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (args.ts && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    args.ts[blockIdx.x * 8 + 0] = gtimer();
    args.ts[blockIdx.x * 8 + 5] = smid;
    args.ts[blockIdx.x * 8 + 6] = args.per_slot ? 1 : meta.tile_slot_off[blockIdx.x + 1] - meta.tile_slot_off[blockIdx.x];
  }

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        int m, s_begin, s_end;
        shrink_item(meta, args.per_slot, w, m, s_begin, s_end);
        for (int s0 = s_begin; s0 < s_end; s0 += P) {
          const int ns = min(P, s_end - s0);
          for (int kb = 0; kb < nk; kb += KB) {
            const int nkb = min(KB, nk - kb);
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], nkb * (R_A_BYTES + ns * vbox));
            uint8_t* st = smem + stage * SB;
            for (int j = 0; j < nkb; ++j)
              tma_load_2d(st + j * R_A_BYTES, &mapZ, &full[stage], (kb + j) * 64, m * kTileM);
            // V of K block j: the ns slots' qv-row boxes back to back = ONE K-major operand
            // of ns*qv rows (8-row groups 1024 B apart), so one MMA covers every slot
            for (int i = 0; i < ns; ++i) {
              const int row0 = meta.roff[meta.slot_task[s0 + i]];
              for (int j = 0; j < nkb; ++j)
                tma_load_2d(st + KB * R_A_BYTES + (j * P + i) * vbox, &mapV, &full[stage],
                            (kb + j) * 64, row0);
            }
            if (++stage == S) stage = 0, phase ^= 1;
          }
        }
      }
      if (args.ts) args.ts[blockIdx.x * 8 + 1] = gtimer();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;   // (tile, pass) counter -> accumulator buffer it & 1
      for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        int m, s_begin, s_end;
        shrink_item(meta, args.per_slot, w, m, s_begin, s_end);
        for (int s0 = s_begin; s0 < s_end; s0 += P, ++it) {
          const int ns = min(P, s_end - s0);
          const uint32_t id = idesc_bf16(128, ns * qv, false, false);   // slot i: columns [i qv, (i+1) qv)
          const int b = it & 1;
          mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t acc = tmem + b * 256;
          for (int kb = 0; kb < nk; kb += KB) {
            const int nkb = min(KB, nk - kb);
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t st0 = smem_u32(smem + stage * SB);
            for (int j = 0; j < nkb; ++j) {
              const uint32_t a0 = st0 + j * R_A_BYTES;
              const uint32_t b0 = st0 + KB * R_A_BYTES + j * P * vbox;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16(acc, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), id,
                         (kb != 0 || j != 0 || k != 0) ? 1u : 0u);
            }
            mma_commit(&empty[stage]);
            if (++stage == S) stage = 0, phase ^= 1;
          }
          mma_commit(&tfull[b]);
        }
      }
      if (args.ts) args.ts[blockIdx.x * 8 + 2] = gtimer();
    }
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;
    const int lrow = q * 32 + lane;
    if (blockIdx.x == 0) {   // the all-zero slot (index nslots) used by the 2-CTA GEMM
      float z[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) z[j] = 0.0f;
      for (int pl = 0; pl < args.nplanes; ++pl)
        store_slot_row(args.out + pl * args.plane_stride, meta.nslots, lrow, z, 0.0f, 0);
    }
    int it = 0;
    bool first = true;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
      int m, s_begin, s_end;
      shrink_item(meta, args.per_slot, w, m, s_begin, s_end);
      const int row = m * kTileM + lrow;
      const int my_task = row < meta.T ? row_task(meta, row) : -1;
      for (int s0 = s_begin; s0 < s_end; s0 += P, ++it) {
        const int ns = min(P, s_end - s0);
        const int b = it & 1;
        mbar_wait(&tfull[b], (it >> 1) & 1);
        tc_fence_after();
        if (args.ts && first && lrow == 0) args.ts[blockIdx.x * 8 + 3] = gtimer();
        first = false;
        for (int i = 0; i < ns; ++i) {
          const int s = s0 + i;
          const int ts = meta.slot_task[s];
          float v[64];
          if (args.nplanes > 1) {   // planes mode (P = 1): plane pl <- columns [pl pq, pl pq + pq)
            const bool mine = ts == my_task;
            for (int pl = 0; pl < args.nplanes; ++pl) {
              const uint32_t ta = tmem + ((q * 32u) << 16) + b * 256 + pl * args.pq;
              tmem_ld32(ta, *reinterpret_cast<float(*)[32]>(v));
              if (args.pq > 32) tmem_ld32(ta + 32, *reinterpret_cast<float(*)[32]>(v + 32));
              else {
#pragma unroll
                for (int j = 32; j < 64; ++j) v[j] = 0.0f;
              }
              store_slot_row(args.out + pl * args.plane_stride, s, lrow, v, mine ? args.sc[ts] : 0.0f,
                             mine ? args.rk[ts] : 0);
            }
            continue;
          }
          const uint32_t ta = tmem + ((q * 32u) << 16) + b * 256 + i * qv;
          tmem_ld32(ta, *reinterpret_cast<float(*)[32]>(v));
          if (qv > 32) tmem_ld32(ta + 32, *reinterpret_cast<float(*)[32]>(v + 32));
          else {
#pragma unroll
            for (int j = 32; j < 64; ++j) v[j] = 0.0f;
          }
          const bool mine = ts == my_task;
          store_slot_row(args.out, s, lrow, v, mine ? meta.scales[ts] : 0.0f, mine ? meta.ranks[ts] : 0);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
      }
    }
  }
  __syncthreads();
  if (args.ts && threadIdx.x == 0) args.ts[blockIdx.x * 8 + 4] = gtimer();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// =====================================================================================
// Planes shrink (a projection group whose bands exceed the 64-wide slot, e.g. q/k/v with
// rank-64 tasks): H_s of every projection of the group from ONE pass over X, the adapter
// operand being the task's np * qp packed rows (MMA N = np * qp, plane p = columns
// [p qp, (p+1) qp)).  Its adapter slice (24 KB per 64-column K block at np * qp = 192) is
// bigger than the X block (16 KB), so X and the adapter get separate rings: X 8 deep (128 KB
// in flight per SM, the amount the single-projection shrink streams at 0.8 of HBM) and the
// L2-resident adapter 4 deep, the X loads running 4 K blocks ahead of the adapter loads.
// (In k_shrink's shared stages only 5 x 16 KB of X were in flight: 0.55-0.60 of HBM.)
// Work item = tile (persistent over tiles), one pass per slot of the tile.
// =====================================================================================
constexpr int SP_NX = 8, SP_NV = 4, SP_LEAD = 4;

struct PlanesCursor {   // walks the (tile, slot, K block) steps of one CTA
  int w, s, s_end, kb, nk, nitems, stride;
  const Meta* meta;
  __device__ bool valid() const { return w < nitems; }
  __device__ void init(const Meta& m, int w0, int stride_, int nk_, int nitems_) {
    meta = &m, stride = stride_, nk = nk_, nitems = nitems_, kb = 0;
    for (w = w0; w < nitems; w += stride)
      if (m.tile_slot_off[w] < m.tile_slot_off[w + 1]) break;
    if (w < nitems) s = m.tile_slot_off[w], s_end = m.tile_slot_off[w + 1];
  }
  __device__ void next() {
    if (++kb < nk) return;
    kb = 0;
    if (++s < s_end) return;
    for (w += stride; w < nitems; w += stride)
      if (meta->tile_slot_off[w] < meta->tile_slot_off[w + 1]) break;
    if (w < nitems) s = meta->tile_slot_off[w], s_end = meta->tile_slot_off[w + 1];
  }
};

__global__ void __launch_bounds__(256, 1)
    k_shrink_planes(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapV,
                    const ShrinkArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int qv = args.qv, vbox = qv * 128;
  uint8_t* sX = smem;                                   // [SP_NX][16 KB]
  uint8_t* sV = sX + SP_NX * R_A_BYTES;                 // [SP_NV][vbox]
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sV + SP_NV * vbox);
  uint64_t* xempty = xfull + SP_NX;
  uint64_t* vfull = xempty + SP_NX;
  uint64_t* vempty = vfull + SP_NV;
  uint64_t* tfull = vempty + SP_NV;     // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;
  const int nk = (args.K + 63) / 64;

  if (warp == 0 && lane == 0) tma_prefetch(&mapZ), tma_prefetch(&mapV);
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < SP_NX; ++i) mbar_init(&xfull[i], 1), mbar_init(&xempty[i], 1);
    for (int i = 0; i < SP_NV; ++i) mbar_init(&vfull[i], 1), mbar_init(&vempty[i], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&tfull[b], 1), mbar_init(&tempty[b], 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: X of step g + SP_LEAD, then V of step g
      PlanesCursor cx, cv;
      cx.init(meta, blockIdx.x, gridDim.x, nk, meta.ntiles);
      cv.init(meta, blockIdx.x, gridDim.x, nk, meta.ntiles);
      int gx = 0, gv = 0;
      auto issue_x = [&]() {
        const int i = gx % SP_NX;
        mbar_wait(&xempty[i], ((gx / SP_NX) & 1) ^ 1);
        mbar_expect_tx(&xfull[i], R_A_BYTES);
        tma_load_2d(sX + i * R_A_BYTES, &mapZ, &xfull[i], cx.kb * 64, cx.w * kTileM);
        cx.next();
        ++gx;
      };
      for (int l = 0; l < SP_LEAD && cx.valid(); ++l) issue_x();
      while (cv.valid()) {
        if (cx.valid()) issue_x();
        const int i = gv % SP_NV;
        mbar_wait(&vempty[i], ((gv / SP_NV) & 1) ^ 1);
        mbar_expect_tx(&vfull[i], vbox);
        tma_load_2d(sV + i * vbox, &mapV, &vfull[i], cv.kb * 64, meta.roff[meta.slot_task[cv.s]]);
        cv.next();
        ++gv;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t id = idesc_bf16(128, qv, false, false);
      int g = 0, it = 0;
      for (int w = blockIdx.x; w < meta.ntiles; w += gridDim.x) {
        for (int s = meta.tile_slot_off[w]; s < meta.tile_slot_off[w + 1]; ++s, ++it) {
          const int b = it & 1;
          mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t acc = tmem + b * 256;
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int ix = g % SP_NX, iv = g % SP_NV;
            mbar_wait(&xfull[ix], (g / SP_NX) & 1);
            mbar_wait(&vfull[iv], (g / SP_NV) & 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sX + ix * R_A_BYTES), b0 = smem_u32(sV + iv * vbox);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16(acc, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), id,
                       (kb | k) ? 1u : 0u);
            mma_commit(&xempty[ix]);
            mma_commit(&vempty[iv]);
          }
          mma_commit(&tfull[b]);
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue: plane p <- columns [p pq, p pq + pq)
    const uint32_t q = warp - 4;
    const int lrow = q * 32 + lane;
    if (blockIdx.x == 0) {   // the all-zero slot (index nslots) used by the 2-CTA GEMM
      float z[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) z[j] = 0.0f;
      for (int pl = 0; pl < args.nplanes; ++pl)
        store_slot_row(args.out + pl * args.plane_stride, meta.nslots, lrow, z, 0.0f, 0);
    }
    int it = 0;
    for (int w = blockIdx.x; w < meta.ntiles; w += gridDim.x) {
      const int row = w * kTileM + lrow;
      const int my_task = row < meta.T ? row_task(meta, row) : -1;
      for (int s = meta.tile_slot_off[w]; s < meta.tile_slot_off[w + 1]; ++s, ++it) {
        const int b = it & 1;
        mbar_wait(&tfull[b], (it >> 1) & 1);
        tc_fence_after();
        const int ts = meta.slot_task[s];
        const bool mine = ts == my_task;
        float v[64];
        for (int pl = 0; pl < args.nplanes; ++pl) {
          const uint32_t ta = tmem + ((q * 32u) << 16) + b * 256 + pl * args.pq;
          tmem_ld32(ta, *reinterpret_cast<float(*)[32]>(v));
          if (args.pq > 32) tmem_ld32(ta + 32, *reinterpret_cast<float(*)[32]>(v + 32));
          else {
#pragma unroll
            for (int j = 32; j < 64; ++j) v[j] = 0.0f;
          }
          store_slot_row(args.out + pl * args.plane_stride, s, lrow, v, mine ? args.sc[ts] : 0.0f,
                         mine ? args.rk[ts] : 0);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// B [out, rsum] -> Bt [rsum, out] (the backward projection's K-major operand)
__global__ void k_transpose_b(const __nv_bfloat16* __restrict__ B, __nv_bfloat16* __restrict__ Bt,
                              int out, int rsum) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ __nv_bfloat16 tile[32][33];
  const int o0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int o = o0 + i, r = r0 + threadIdx.x;
    tile[i][threadIdx.x] = (o < out && r < rsum) ? B[(size_t)o * rsum + r] : __float2bfloat16(0.0f);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, o = o0 + threadIdx.x;
    if (r < rsum && o < out) Bt[(size_t)r * out + o] = tile[threadIdx.x][i];
  }
}

// =====================================================================================
// Segmented token reduction: partial[u][c][q][i] = sum_{slots of unit u} sum_rows
//      Z[row][c*128 + i] * Slot[row][q]          (Z^T as an MN-major A operand)
// =====================================================================================
constexpr int S_STAGES = 4;
constexpr int S_A_BYTES = 2 * 128 * 64 * 2;  // two 64-col boxes of 128 rows: 32 KB
constexpr int S_B_BYTES = 128 * 64 * 2;      // one slot: 16 KB
constexpr int S_STAGE_BYTES = S_A_BYTES + S_B_BYTES;
constexpr int S_SMEM = S_STAGES * S_STAGE_BYTES + 1024 + 256;

struct SegArgs {
  int width, nchunks, nitems;
  float* partial;
  Meta meta;
};

__global__ void __launch_bounds__(256, 1)
    k_segred(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapSlot,
             const SegArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_STAGES * S_STAGE_BYTES);
  uint64_t* empty = full + S_STAGES;
  uint64_t* tfull = empty + S_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;

  if (warp == 0 && lane == 0) tma_prefetch(&mapZ), tma_prefetch(&mapSlot);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S_STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&tfull[a], 1), mbar_init(&tempty[a], 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = meta.sr_cta_off[blockIdx.x]; u < meta.sr_cta_off[blockIdx.x + 1]; ++u) {
        const int c = meta.sr_chunk[u];
        for (int k = meta.sr_s0[u]; k < meta.sr_s1[u]; ++k) {
          const int sl = meta.task_slots[k];
          const int tile = meta.slot_tile[sl];
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], S_STAGE_BYTES);
          uint8_t* st = smem + stage * S_STAGE_BYTES;
          tma_load_2d(st, &mapZ, &full[stage], c * 128, tile * kTileM);
          tma_load_2d(st + 16384, &mapZ, &full[stage], c * 128 + 64, tile * kTileM);
          tma_load_2d(st + S_A_BYTES, &mapSlot, &full[stage], 0, sl * kTileM);
          if (++stage == S_STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = idesc_bf16(128, 64, true, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = meta.sr_cta_off[blockIdx.x]; u < meta.sr_cta_off[blockIdx.x + 1]; ++u, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 64;
        bool first = true;
        for (int k = meta.sr_s0[u]; k < meta.sr_s1[u]; ++k) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * S_STAGE_BYTES);
          const uint32_t b0 = a0 + S_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            mma_bf16(d, sdesc_sw128(a0 + kk * 2048, 16384, 1024),
                     sdesc_sw128(b0 + kk * 2048, 8192, 1024), id, first ? 0u : 1u);
            first = false;
          }
          mma_commit(&empty[stage]);
          if (++stage == S_STAGES) stage = 0, phase ^= 1;
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;
    int it = 0;
    for (int u = meta.sr_cta_off[blockIdx.x]; u < meta.sr_cta_off[blockIdx.x + 1]; ++u, ++it) {
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int rp = rpad16(meta.ranks[meta.sr_task[u]]);
      float* dst = args.partial + ((size_t)u * meta.qp) * 128 + q * 32 + lane;   // [seg][qp][128]
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        if (h * 32 >= rp) break;
        float v[32];
        tmem_ld32(tmem + ((q * 32u) << 16) + acc * 64 + h * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (h * 32 + j < rp) dst[(size_t)(h * 32 + j) * 128] = v[j];
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// =====================================================================================
// Fused backward dY pass: ONE HBM read of dY computes both
//   G_s  = s_t dY B_t        (per row: reduction over `out`)   -> fp32 partials per
//                                                                (slot, 512-col chunk)
//   dB_t = H_s^T dY          (per column: reduction over tokens) -> fp32 partials per
//                                                                (unit, 128-col block)
// Work item = (dy unit u: consecutive slots of one task, 512-column chunk c).  Per slot and
// 128-column sub-block b the stage holds the dY tile (2 boxes, K-major for G / MN-major for
// dB), the H slot (MN-major B for dB) and 2 boxes of the caller's B (64 q x 64 o rows,
// MN-major B for G: no transpose copy).  TMEM: four dB
// accumulators (4 x 64 cols) kept across the unit's slots + two G accumulators (2 x 64).
// k_gfin then sums the G chunk partials in fixed order, scales by s_t, masks and writes
// the bf16 G slots; the dB partials go through k_finalize_multi (fixed order).
// =====================================================================================
// The H slot and B_t operands are MN-major (q contiguous) boxes only as wide as the rank needs:
// `hrow` = 32 / 64 / 128 bytes (16 / 32 / 64 q, TMA and UMMA swizzle of that span), MMA N = nq.
// A stage is [dY 2 x 16 KB][B 2 x 64 o x hrow]; the H slot (128 tokens x hrow) is loaded
// ONCE per (slot, chunk) into a 2-entry ring beside the stages and serves the chunk's four
// sub-blocks (it used to ride in every stage): 6 / 5 / 4 stages (192 / 160 / 128 KB of dY in
// flight) for hrow 32 / 64 / 128 instead of 5 / 4 / 3.
constexpr int Y_Z_BYTES = 2 * 128 * 64 * 2;   // dY tile: 2 boxes of 64 cols x 128 rows
constexpr int Y_SMEM = 232448;                // stages fill the shared memory (one CTA per SM)

struct DyArgs {
  int width, nchunks, nitems, n128, qp;
  int hrow, nq, stages, stage_bytes;
  int dbg_dy_only;   // tuning probe (LOBRA_DBG_DY_ONLY=1): stream dY only, skip H / B loads
  unsigned long long* ts;   // tracing (LOBRA_TRACE_DY): per CTA {start, end, smid} globaltimer, else null
  float* gpart;    // [nslots][nchunks][128][qp]
  float* bpart;    // [segments][4][qp][128]
  Meta meta;
};

__global__ void __launch_bounds__(256, 1)
    k_dypass(const __grid_constant__ CUtensorMap mapDY, const __grid_constant__ CUtensorMap mapH,
             const __grid_constant__ CUtensorMap mapBt, const DyArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int NS = args.stages, SB = args.stage_bytes, hrow = args.hrow;
  const int hbytes = 128 * hrow;          // H region (128 tokens)
  const int bbox = 64 * hrow;             // one B box (64 o rows)
  uint8_t* hbuf = smem + NS * SB;         // [2][hbytes]: the H ring
  uint64_t* full = reinterpret_cast<uint64_t*>(hbuf + 2 * hbytes);
  uint64_t* empty = full + 8;
  uint64_t* gfull = empty + 8;           // [2]
  uint64_t* gempty = gfull + 2;          // [2]
  uint64_t* bfull = gempty + 2;          // [1]
  uint64_t* bempty = bfull + 1;          // [1]
  uint64_t* hfull = bempty + 1;          // [2]
  uint64_t* hempty = hfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const Meta& meta = args.meta;

  if (warp == 0 && lane == 0) tma_prefetch(&mapDY), tma_prefetch(&mapH), tma_prefetch(&mapBt);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&gfull[a], 1), mbar_init(&gempty[a], 128);
    mbar_init(bfull, 1);
    mbar_init(bempty, 128);
    for (int a = 0; a < 2; ++a) mbar_init(&hfull[a], 1), mbar_init(&hempty[a], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (args.ts && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    args.ts[blockIdx.x * 3 + 0] = gtimer();
    args.ts[blockIdx.x * 3 + 2] = smid;
  }

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      int hcount = 0;
      for (int u = meta.dy_cta_off[blockIdx.x]; u < meta.dy_cta_off[blockIdx.x + 1]; ++u) {
        const int c = meta.dy_unit_chunk[u];
        const int t = meta.dy_unit_task[u];
        const int nb = min(4, args.n128 - c * 4);
        if (nb <= 0) continue;   // a chunk past this projection's width (group of unequal outs)
        for (int k = meta.dy_unit_s0[u]; k < meta.dy_unit_s1[u]; ++k, ++hcount) {
          const int sl = meta.task_slots[k];
          const int tile = meta.slot_tile[sl];
          // the slot's H (this projection's band only, or all 64 columns for hrow 128), once
          // for the chunk's sub-blocks
          const int hb = hcount & 1;
          mbar_wait(&hempty[hb], ((hcount >> 1) & 1) ^ 1);
          mbar_expect_tx(&hfull[hb], (args.dbg_dy_only & 1) ? 0 : hbytes);
          if (!(args.dbg_dy_only & 1))
            tma_load_2d(hbuf + hb * hbytes, &mapH, &hfull[hb], hrow == 128 ? 0 : meta.band, sl * kTileM);
          for (int b = 0; b < nb; ++b) {
            const int col = c * 512 + b * 128;
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], (args.dbg_dy_only & 1) ? Y_Z_BYTES : Y_Z_BYTES + 2 * bbox);
            uint8_t* st = smem + stage * SB;
            tma_load_2d(st, &mapDY, &full[stage], col, tile * kTileM);
            tma_load_2d(st + 16384, &mapDY, &full[stage], col + 64, tile * kTileM);
            if (!(args.dbg_dy_only & 1)) {
              // B_t straight from the caller's B (MN-major: q contiguous, rows = o = K)
              tma_load_2d(st + Y_Z_BYTES, &mapBt, &full[stage], meta.boff[t], col);
              tma_load_2d(st + Y_Z_BYTES + bbox, &mapBt, &full[stage], meta.boff[t], col + 64);
            }
            if (++stage == NS) stage = 0, phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t id_b = idesc_bf16(128, args.nq, true, true);     // dB: both MN-major
      const uint32_t id_g = idesc_bf16(128, args.nq, false, true);    // G: A K-major, B MN-major
      // stage-0 descriptors of the H and B regions; per K step (16 rows) + hstep, per B box
      // + bstep4 (address field units of 16 bytes)
      const uint32_t s0 = smem_u32(smem);
      const uint64_t hdesc0 = sdesc_sw(smem_u32(hbuf), hbytes, 8 * hrow, hrow);
      const uint64_t tdesc0 = sdesc_sw(s0 + Y_Z_BYTES, bbox, 8 * hrow, hrow);
      const int hstep = hrow;            // 16 rows x hrow bytes >> 4
      const int bstep4 = bbox >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int gcount = 0, it = 0;
      for (int u = meta.dy_cta_off[blockIdx.x]; u < meta.dy_cta_off[blockIdx.x + 1]; ++u) {
        const int c = meta.dy_unit_chunk[u];
        const int nb = min(4, args.n128 - c * 4);
        if (nb <= 0) continue;
        mbar_wait(bempty, (it & 1) ^ 1);
        tc_fence_after();
        bool first_slot = true;
        for (int k = meta.dy_unit_s0[u]; k < meta.dy_unit_s1[u]; ++k, ++gcount) {
          const int gb = gcount & 1;
          mbar_wait(&gempty[gb], ((gcount >> 1) & 1) ^ 1);
          mbar_wait(&hfull[gb], (gcount >> 1) & 1);   // the H ring advances with the slots
          tc_fence_after();
          const uint32_t dg = tmem + 256 + gb * 64;
          const uint64_t dh = hdesc0 + ((uint64_t)(gb * hbytes) >> 4);
          for (int b = 0; b < nb; ++b) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            // descriptors built once per stage; a K step adds its byte offset >> 4 to the
            // start-address field (the single issuing thread must keep up with the stream)
            const uint32_t z0 = smem_u32(smem + stage * SB);
            const uint64_t dz_mn = sdesc_sw128(z0, 16384, 1024);
            const uint64_t dz_k = sdesc_sw128(z0, 16, 1024);
            const uint64_t dt = tdesc0 + ((uint64_t)(stage * SB) >> 4);
            if (!(args.dbg_dy_only & 2)) {   // probe bit 1: skip the dB MMAs
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)   // dB[b] += dY^T H   (K = 128 tokens)
                mma_bf16(tmem + b * 64, dz_mn + (uint64_t)(kk * 128), dh + (uint64_t)(kk * hstep),
                         id_b, (first_slot && kk == 0) ? 0u : 1u);
            }
            if (!(args.dbg_dy_only & 4)) {   // probe bit 2: skip the G MMAs
#pragma unroll
              for (int j = 0; j < 2; ++j)      // G += dY[:, 64 cols] B^T[qp, 64 cols]^T
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_bf16(dg, dz_k + (uint64_t)(j * 1024 + kk * 2),
                           dt + (uint64_t)(j * bstep4 + kk * hstep), id_g,
                           (b == 0 && j == 0 && kk == 0) ? 0u : 1u);
            }
            mma_commit(&empty[stage]);
            if (++stage == NS) stage = 0, phase ^= 1;
          }
          mma_commit(&gfull[gb]);
          mma_commit(&hempty[gb]);
          first_slot = false;
        }
        mma_commit(bfull);
        ++it;
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    const uint32_t q = warp - 4;
    const int lr = q * 32 + lane;    // row of the tile (G) / column of the sub-block (dB)
    int gcount = 0, it = 0;
    for (int u = meta.dy_cta_off[blockIdx.x]; u < meta.dy_cta_off[blockIdx.x + 1]; ++u) {
      const int c = meta.dy_unit_chunk[u];
      const int nb = min(4, args.n128 - c * 4);
      if (nb <= 0) continue;
      const int t = meta.dy_unit_task[u];
      const int rp = rpad16(meta.ranks[t]);
      for (int k = meta.dy_unit_s0[u]; k < meta.dy_unit_s1[u]; ++k, ++gcount) {
        const int gb = gcount & 1;
        const int sl = meta.task_slots[k];
        mbar_wait(&gfull[gb], (gcount >> 1) & 1);
        tc_fence_after();
        float* dst = args.gpart + (((size_t)sl * args.nchunks + c) * kTileM + lr) * args.qp;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (h * 32 >= rp) break;
          float v[32];
          tmem_ld32(tmem + ((q * 32u) << 16) + 256 + gb * 64 + h * 32, v);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            if (h * 32 + j < rp)
              *reinterpret_cast<float4*>(dst + h * 32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
        tc_fence_before();
        mbar_arrive(&gempty[gb]);
      }
      mbar_wait(bfull, it & 1);
      tc_fence_after();
      for (int b = 0; b < nb; ++b) {
        float* dst = args.bpart + ((size_t)(u * 4 + b) * meta.qp) * 128 + lr;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (h * 32 >= rp) break;
          float v[32];
          tmem_ld32(tmem + ((q * 32u) << 16) + b * 64 + (hrow == 128 ? meta.band : 0) + h * 32, v);   // dB vs H band
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (h * 32 + j < rp) dst[(size_t)(h * 32 + j) * 128] = v[j];
        }
      }
      tc_fence_before();
      mbar_arrive(bempty);
      ++it;
    }
  }
  __syncthreads();
  if (args.ts && threadIdx.x == 0) args.ts[blockIdx.x * 3 + 1] = gtimer();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// G slots from the chunk partials: slot[s][row][q] = s_t * sum_c gpart[s][c][row][q] for
// rows of the slot's task and q < r_t, zero otherwise; also the all-zero slot nslots.
// One thread per (slot row, 8 output columns of this projection's band): float4 loads of the
// chunk partials, summed in chunk order, scaled, masked, one 16-byte store at column
// band + 8 g (a projection group's other bands are left untouched).
constexpr int GF_BATCH = 8;
constexpr int GF_CTAS_PER_SM = 4;   // chunk partials loaded per batch (independent loads in flight)
__global__ void k_gfin(const float* __restrict__ gpart, int nchunks, int qp, Meta meta,
                       __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  const int ng = qp / 8;
  const int total = (meta.nslots + 1) * kTileM * ng;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % ng, r = i / ng;
    const int s = r / kTileM, lrow = r % kTileM;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 0.0f;
    int rp = 0;
    float sc = 0.0f;
    if (s < meta.nslots && g * 8 < meta.ranks[meta.slot_task[s]]) {   // columns < r_t only
      const int t = meta.slot_task[s];
      // the chunk partials are loaded (4 chunks at a time, independent loads) while the
      // row's task is looked up; rows of other tasks are masked afterwards
      const float* src = gpart + ((size_t)s * nchunks * kTileM + lrow) * qp + g * 8;
      const size_t cstride = (size_t)kTileM * qp;
      for (int c = 0; c < nchunks; c += GF_BATCH) {
        float4 a[GF_BATCH], b[GF_BATCH];
#pragma unroll
        for (int j = 0; j < GF_BATCH; ++j) {
          const bool ok = c + j < nchunks;
          a[j] = ok ? __ldg(reinterpret_cast<const float4*>(src + (c + j) * cstride)) : make_float4(0, 0, 0, 0);
          b[j] = ok ? __ldg(reinterpret_cast<const float4*>(src + (c + j) * cstride) + 1) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < GF_BATCH; ++j) {   // chunk order, as before
          if (c + j >= nchunks) break;
          v[0] += a[j].x; v[1] += a[j].y; v[2] += a[j].z; v[3] += a[j].w;
          v[4] += b[j].x; v[5] += b[j].y; v[6] += b[j].z; v[7] += b[j].w;
        }
      }
      const int row = meta.slot_tile[s] * kTileM + lrow;
      if (row < meta.T && row_task(meta, row) == t) {
        rp = meta.ranks[t] - g * 8;
        sc = meta.scales[t];
      }
    }
    float w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = e < rp ? v[e] * sc : 0.0f;
    uint4 o;
    o.x = pack_bf16x2(w[0], w[1]);
    o.y = pack_bf16x2(w[2], w[3]);
    o.z = pack_bf16x2(w[4], w[5]);
    o.w = pack_bf16x2(w[6], w[7]);
    reinterpret_cast<uint4*>(out + ((size_t)s * kTileM + lrow) * kSlotW + meta.band)[g] = o;
  }
}

// Projection group: A_grp[(t * np + p) * qp + j, :] = A_p[roff[t] + j, :] for j < r_t, zero
// rows for r_t <= j < qp (the band layout of the shared H/G slots).
struct GroupA {
  const __nv_bfloat16* A[4];
};
__global__ void k_pack_a_group(GroupA src, int np, int qp, int in, Meta meta,
                               __nv_bfloat16* __restrict__ dst) {
  pdl_wait();
  pdl_launch_dependents();
  const int vpr = in / 8;   // uint4 per row
  const long long total = (long long)meta.ntasks * np * qp * vpr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i % vpr);
    const long long row = i / vpr;
    const int j = (int)(row % qp), p = (int)((row / qp) % np), t = (int)(row / ((long long)qp * np));
    uint4 val = make_uint4(0, 0, 0, 0);
    if (j < meta.ranks[t])
      val = __ldg(reinterpret_cast<const uint4*>(src.A[p] + (size_t)(meta.roff[t] + j) * in) + v);
    reinterpret_cast<uint4*>(dst + (size_t)row * in)[v] = val;
  }
}

// =====================================================================================
// small helper kernels
// =====================================================================================
// B_cat [out, rsum] -> Bp [out, ld8]: task t's r_t columns at boff[t], zero padding.
__global__ void k_pad_cols(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                           int out, int ld8, Meta meta) {
  pdl_wait();
  pdl_launch_dependents();
  const int total = out * ld8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int o = i / ld8, c = i - o * ld8;
    int t = 0;
    while (t + 1 < meta.ntasks && meta.boff[t + 1] <= c) ++t;
    const int q = c - meta.boff[t];
    dst[i] = q < meta.ranks[t] ? src[(size_t)o * meta.rsum + meta.roff[t] + q] : __float2bfloat16(0.0f);
  }
}

// out[(t,q), col] (+)= sum over the task's units / segments (fixed order) of the partials.
// Several finalizations in ONE launch (blockIdx.z = job): the dA and dB of a projection, or
// of every projection of a group.  Same fixed summation order as k_finalize; the unit loads
// are issued 8 at a time (independent) before the in-order sum.
__global__ void __launch_bounds__(256) k_finalize_multi(const FinJobs jobs, const Meta meta) {
  // block = 8 adapter rows (rq, one per warp) x one 128-column chunk of one job; a lane sums
  // 4 columns (lane + 32 k: 128-byte coalesced partial loads, 4 independent chains).  dA
  // (mode 0, row-major [r, width]) is stored directly; dB (mode 1, PEFT [width, rsum]) goes
  // through a shared-memory transpose so that 8 threads store 8 consecutive rq of one column
  // (32 B) instead of 8 scattered words.
  __shared__ float tile[8][129];
  pdl_wait();
  pdl_launch_dependents();
  const FinJob& J = jobs.j[blockIdx.z];
  const int col0 = blockIdx.x * 128;
  if (col0 >= J.width) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rq = blockIdx.y * 8 + w;
  const int c = blockIdx.x;                       // 128-column chunk
  float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (rq < meta.rsum) {
    int lo = 0, hi = meta.ntasks - 1;             // task of row rq: last t with roff[t] <= rq
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (meta.roff[mid] <= rq) lo = mid; else hi = mid - 1;
    }
    const int t = lo, q = rq - meta.roff[t];
    int u0, u1;
    size_t base, ustride;
    if (J.dy) {   // segments of (t, J.sub 128-column blocks): [seg][sub][qp][128]
      const int tc = t * J.dy_nch + c / J.sub;
      u0 = J.uoff[tc], u1 = J.uoff[tc + 1];
      base = ((size_t)(c % J.sub) * J.qp + J.band + q) * 128 + lane;
      ustride = (size_t)J.sub * J.qp * 128;
    } else {
      u0 = J.uoff[t], u1 = J.uoff[t + 1];
      base = ((size_t)c * J.qp + J.band + q) * 128 + lane;
      ustride = (size_t)J.nchunks * J.qp * 128;
    }
    for (int u = u0; u < u1; u += 2) {
      float v[2][4];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[a][k] = (u + a < u1 && col0 + lane + 32 * k < J.width)
                        ? __ldg(J.partial + base + (size_t)(u + a) * ustride + 32 * k) : 0.0f;
#pragma unroll
      for (int a = 0; a < 2; ++a)
        if (u + a < u1)
#pragma unroll
          for (int k = 0; k < 4; ++k) s[k] += v[a][k];
    }
    if (J.mode == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int col = col0 + lane + 32 * k;
        if (col < J.width) {
          float* dst = J.out + (long long)rq * J.ld + col;
          *dst = J.accumulate ? *dst + s[k] : s[k];
        }
      }
    }
  }
  if (J.mode == 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[w][lane + 32 * k] = s[k];
    __syncthreads();
    const int r = threadIdx.x & 7;
    const int rq2 = blockIdx.y * 8 + r;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int cc = (threadIdx.x >> 3) + 32 * k, cl = col0 + cc;
      if (rq2 < meta.rsum && cl < J.width) {
        float* dst = J.out + (long long)cl * meta.rsum + rq2;
        const float v = tile[r][cc];
        *dst = J.accumulate ? *dst + v : v;
      }
    }
  }
}

__global__ void k_zero(float* p, long long n) {
  pdl_wait();
  pdl_launch_dependents();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0f;
}

}  // namespace

// =====================================================================================
// launchers (programmatic dependent launch unless LOBRA_NO_PDL=1)
// =====================================================================================
namespace {
bool use_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  note_launch();
}
}  // namespace
void launch_pad_cols(const __nv_bfloat16* src, __nv_bfloat16* dst, int out, int ld8,
                     const Meta& meta, cudaStream_t st) {
  launch_k(k_pad_cols, dim3(592), dim3(256), 0, st, src, dst, out, ld8, meta);
}

// rank-r projection configuration (split-K k_rowproj for batches whose tiles cannot fill
// the GPU): 3 stages, 2 slots per pass, 1 K block per stage, 2 resident CTAs per SM
// (the best of the six configurations measured in round 1, profiles/r1_skinny_probes.md).
constexpr int kRpPerSm = 2;

bool rowproj_uses_ld() {   // opt-in (LOBRA_RP_LD=1): measured slower than TMA on B200
  const char* e = getenv("LOBRA_RP_LD");
  return e && e[0] == '1';
}

int rowproj_splits(int ntiles, int K) {
  // one wave of similar-size CTAs: HBM-bound, so what matters is that every resident CTA
  // streams the same number of bytes
  const int nk = (K + 63) / 64;
  const int per_sm = rowproj_uses_ld() ? 1 : kRpPerSm;
  const int slots = per_sm * 148;
  int s = ntiles > 0 ? slots / ntiles : 1;
  if (const char* fs = getenv("LOBRA_RP_SPLITS")) {   // tuning override
    const int v = atoi(fs);
    if (v >= 1 && v <= 8) s = v;
  }
  s = s < 1 ? 1 : s;
  s = s > 8 ? 8 : s;
  s = s > nk ? nk : s;
  return s;
}

template <bool V, int ST, int P, int KB>
void launch_rp(int grid, const CUtensorMap& mapZ, const CUtensorMap& mapV, const RowArgs& a,
               cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_rowproj<V, ST, P, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         r_smem<ST, P, KB>());
    init = true;
  }
  launch_k(k_rowproj<V, ST, P, KB>, dim3(grid), dim3(256), r_smem<ST, P, KB>(), st, mapZ, mapV, a);
}

void launch_rowproj(bool v_mn, const CUtensorMap& mapZ, const CUtensorMap& mapV, int K,
                    const Meta& meta, __nv_bfloat16* slots, float* partial, int* counters,
                    cudaStream_t st) {
  RowArgs a;
  a.K = K;
  {
    a.dbg_no_mma = 0;
#ifdef LOBRA_PROBES   // work-skipping probes: never compiled into the product library
    const char* e = getenv("LOBRA_DBG_RP_NOMMA");
    a.dbg_no_mma = (e && e[0] == '1') ? 1 : 0;
    // LOBRA_DBG_RP: probe bit mask (1 no MMA, 2 no adapter boxes, 4 no output / reduction)
    if (const char* d = getenv("LOBRA_DBG_RP")) a.dbg_no_mma = atoi(d);
#endif
    const char* f = getenv("LOBRA_RP_PREFETCH");
    a.prefetch = f ? atoi(f) : 0;
    const char* g = getenv("LOBRA_RP_INTERLEAVE");
    a.interleave = (g && g[0] == '1') ? 1 : 0;
  }
  a.nsplit = rowproj_splits(meta.ntiles, K);
  const int nk = (K + 63) / 64;
  a.kb_per_split = (nk + a.nsplit - 1) / a.nsplit;
  a.nsplit = (nk + a.kb_per_split - 1) / a.kb_per_split;
  a.out = slots;
  a.partial = partial;
  a.counters = counters;
  a.meta = meta;
  if (a.nsplit > 1) cudaMemsetAsync(counters, 0, sizeof(int) * meta.ntiles, st);
  const int grid = meta.ntiles * a.nsplit;
  if (v_mn)
    launch_rp<true, 3, 2, 1>(grid, mapZ, mapV, a, st);
  else
    launch_rp<false, 3, 2, 1>(grid, mapZ, mapV, a, st);
}

bool shrink_applies(int ntiles, int num_sms) {
  // enough tiles to keep >= 3/4 of the SMs streaming; else the split-K k_rowproj
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_SHRINK");   // 0: always k_rowproj (A/B)
    v = e ? atoi(e) : 1;
  }
  return v != 0 && 4 * ntiles >= 3 * num_sms;
}

void launch_shrink(const CUtensorMap& mapZ, const CUtensorMap& mapV, int K, const Meta& meta,
                   __nv_bfloat16* slots, int num_sms, cudaStream_t st, const ShrinkPlanes* planes) {
  constexpr int kMaxSmem = 232448;
  ShrinkArgs a;
  a.K = K;
  a.qv = meta.qp;
  a.nplanes = 1, a.pq = 0, a.plane_stride = 0, a.rk = nullptr, a.sc = nullptr;
  if (planes) {
    a.nplanes = planes->np, a.pq = planes->pq, a.plane_stride = planes->plane_stride;
    a.rk = planes->ranks, a.sc = planes->scales;
  }
  a.per_slot = meta.nslots <= num_sms ? 1 : 0;
  if (const char* e = getenv("LOBRA_SHRINK_PER_TILE")) a.per_slot = (e[0] == '1') ? 0 : a.per_slot;
  a.P = (a.per_slot || planes) ? 1 : std::max(1, std::min(SH_P, meta.max_slots_per_tile));
  a.kb = a.qv > 64 ? 1 : SH_KB;   // a wide adapter operand: 1 K block per stage, more stages
  a.stage_bytes = a.kb * (R_A_BYTES + a.P * a.qv * 128);
  a.stages = std::min(8, (kMaxSmem - 1024 - 256) / a.stage_bytes);
  a.out = slots;
  a.meta = meta;
  a.ts = nullptr;
  {
    static unsigned long long* ts = nullptr;
    static int dbg = -1;
    if (dbg < 0) {
      dbg = 0;
#ifdef LOBRA_PROBES
      const char* e = getenv("LOBRA_DBG_SHRINK_TS");
      dbg = (e && e[0] == '1') ? 1 : 0;
      if (dbg) cudaMalloc(&ts, 8 * 1024 * sizeof(unsigned long long));
#endif
    }
    a.ts = ts;
  }
  const int smem = a.stages * a.stage_bytes + 1024 + 256;
  static int init = 0;
  if (init < smem) {
    cudaFuncSetAttribute(k_shrink, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    init = kMaxSmem;
  }
  if (planes && !getenv("LOBRA_PLANES_SHARED_STAGES")) {   // separate X / adapter rings
    const int psmem = SP_NX * R_A_BYTES + SP_NV * a.qv * 128 + 1024 + 256;
    static bool pinit = false;
    if (!pinit) {
      cudaFuncSetAttribute(k_shrink_planes, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
      pinit = true;
    }
    const int pgrid = std::max(1, std::min(meta.ntiles, num_sms));
    launch_k(k_shrink_planes, dim3(pgrid), dim3(256), psmem, st, mapZ, mapV, a);
    return;
  }
  const int grid = std::max(1, std::min(a.per_slot ? meta.nslots : meta.ntiles, num_sms));
  launch_k(k_shrink, dim3(grid), dim3(256), smem, st, mapZ, mapV, a);
  if (a.ts) {   // probe: per-CTA phase times (us from the earliest CTA start)
    std::vector<unsigned long long> h(8 * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), a.ts, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[8 * c]);
    double mx[5] = {0}, sm[5] = {0};
    for (int c = 0; c < grid; ++c)
      for (int k = 0; k < 5; ++k) {
        const double v = (h[8 * c + k] - t0) * 1e-3;
        mx[k] = std::max(mx[k], v);
        sm[k] += v / grid;
      }
    static int dumped = 0;
    if (dumped++ == 5) {
      fprintf(stderr, "shrink per-CTA: cta smid done_us\n");
      for (int c = 0; c < grid; ++c)
        fprintf(stderr, "CTA %d sm %llu ns %llu start %.1f prod %.1f mma %.1f epi %.1f end %.1f\n", c, h[8 * c + 5],
                h[8 * c + 6], (h[8 * c] - t0) * 1e-3, (h[8 * c + 1] - t0) * 1e-3, (h[8 * c + 2] - t0) * 1e-3,
                (h[8 * c + 3] - t0) * 1e-3, (h[8 * c + 4] - t0) * 1e-3);
    }
    fprintf(stderr, "shrink ts (us; avg/max over %d CTAs): start %.1f/%.1f producer-done %.1f/%.1f "
            "mma-done %.1f/%.1f epi-start %.1f/%.1f end %.1f/%.1f\n", grid, sm[0], mx[0], sm[1], mx[1],
            sm[2], mx[2], sm[3], mx[3], sm[4], mx[4]);
  }
}

void launch_pack_a_group(const __nv_bfloat16* const* A, int np, int qp, int in, const Meta& meta,
                         __nv_bfloat16* dst, cudaStream_t st) {
  GroupA g{};
  for (int p = 0; p < np && p < 4; ++p) g.A[p] = A[p];
  const long long total = (long long)meta.ntasks * np * qp * (in / 8);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  launch_k(k_pack_a_group, dim3(std::max(blocks, 1)), dim3(256), 0, st, g, np, qp, in, meta, dst);
}

void launch_transpose_b(const __nv_bfloat16* B, __nv_bfloat16* Bt, int out, int rsum, cudaStream_t st) {
  launch_k(k_transpose_b, dim3((out + 31) / 32, (rsum + 31) / 32), dim3(32, 8), 0, st, B, Bt, out, rsum);
}

template <int ST, int KB>
void launch_rpld(int grid, const CUtensorMap& mapV, const RowLdArgs& a, cudaStream_t st) {
  const int smem = ST * (KB * R_A_BYTES + 2 * KB * a.qp * 128) + 1024 + 256;
  static int init = 0;
  if (init < smem) {
    cudaFuncSetAttribute(k_rowproj_ld<ST, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = smem;
  }
  launch_k(k_rowproj_ld<ST, KB>, dim3(grid), dim3(288), smem, st, mapV, a);
}

void launch_rowproj_ld(const __nv_bfloat16* Z, int K, const CUtensorMap& mapVk, int qp,
                       const Meta& meta, __nv_bfloat16* slots, float* partial, int* counters,
                       cudaStream_t st) {
  RowLdArgs a;
  a.Z = Z;
  a.K = K;
  a.qp = qp;
  a.nsplit = rowproj_splits(meta.ntiles, K);
  const int nk = (K + 63) / 64;
  a.kb_per_split = (nk + a.nsplit - 1) / a.nsplit;
  a.nsplit = (nk + a.kb_per_split - 1) / a.kb_per_split;
  a.out = slots;
  a.partial = partial;
  a.counters = counters;
  a.meta = meta;
  if (a.nsplit > 1) cudaMemsetAsync(counters, 0, sizeof(int) * meta.ntiles, st);
  const int grid = meta.ntiles * a.nsplit;
  launch_rpld<3, 2>(grid, mapVk, a, st);
}

int dypass_span(int qp) {
  static int force = -1;   // LOBRA_DY_SPAN=32|64|128 (tuning; never narrower than the rank)
  if (force < 0) {
    const char* e = getenv("LOBRA_DY_SPAN");
    force = e ? atoi(e) : 0;
  }
  const int need = qp <= 16 ? 32 : qp <= 32 ? 64 : 128;
  return force > need ? force : need;
}

void launch_dypass(const CUtensorMap& mapDY, const CUtensorMap& mapH, const CUtensorMap& mapBt,
                   int width, int qp, const Meta& meta, float* gpart, float* bpart,
                   __nv_bfloat16* gslots, int num_sms, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_dypass, cudaFuncAttributeMaxDynamicSharedMemorySize, Y_SMEM);
    init = true;
  }
  DyArgs a;
  a.hrow = dypass_span(qp);
  a.nq = a.hrow / 2;
  a.stage_bytes = Y_Z_BYTES + 2 * 64 * a.hrow;
  a.stages = std::min(8, (Y_SMEM - 1024 - 256 - 2 * 128 * a.hrow) / a.stage_bytes);
  if (const char* e = getenv("LOBRA_DY_STAGES")) a.stages = std::max(2, std::min(a.stages, atoi(e)));
  a.width = width;
  a.n128 = (width + 127) / 128;
  a.nchunks = (width + 511) / 512;
  a.nitems = meta.ndyunits * a.nchunks;
  a.qp = qp;
  a.gpart = gpart;
  a.bpart = bpart;
  a.meta = meta;
  {
    static int dbg = -1;
    if (dbg < 0) {
      dbg = 0;
#ifdef LOBRA_PROBES
      const char* e = getenv("LOBRA_DBG_DY_ONLY");
      dbg = (e && e[0] == '1') ? 1 : 0;
      // LOBRA_DBG_DY: probe bit mask (1 dY only, 2 no dB MMAs, 4 no G MMAs)
      if (const char* f = getenv("LOBRA_DBG_DY")) dbg = atoi(f);
#endif
    }
    a.dbg_dy_only = dbg;
  }
  a.ts = nullptr;
  static const char* trace = getenv("LOBRA_TRACE_DY");
  static unsigned long long* d_ts = nullptr;
  if (trace && meta.ndyunits > 0) {
    if (!d_ts && cudaMalloc(&d_ts, 3 * 4096 * sizeof(unsigned long long)) != cudaSuccess) d_ts = nullptr;
    if (d_ts && meta.ndycta <= 4096) a.ts = d_ts;
  }
  if (meta.ndyunits > 0) launch_k(k_dypass, dim3(meta.ndycta), dim3(256), Y_SMEM, st, mapDY, mapH, mapBt, a);
  if (a.ts) {   // tracing only: per-CTA times with the CTA's entry ranges, one JSON line per launch
    std::vector<unsigned long long> h(3 * meta.ndycta);
    std::vector<int> off(meta.ndycta + 1), ut(meta.ndyunits), u0(meta.ndyunits), u1(meta.ndyunits),
        uc(meta.ndyunits), rk(meta.ntasks);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), a.ts, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(off.data(), meta.dy_cta_off, off.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ut.data(), meta.dy_unit_task, ut.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(u0.data(), meta.dy_unit_s0, u0.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(u1.data(), meta.dy_unit_s1, u1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(uc.data(), meta.dy_unit_chunk, uc.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(rk.data(), meta.ranks, rk.size() * 4, cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace, "a")) {
      fprintf(f, "{\"width\": %d, \"qp\": %d, \"ranks\": [", width, qp);
      for (int t = 0; t < meta.ntasks; ++t) fprintf(f, "%s%d", t ? ", " : "", rk[t]);
      fprintf(f, "], \"cta\": [");
      for (int b = 0; b < meta.ndycta; ++b) {
        fprintf(f, "%s[%llu, %llu, %llu, [", b ? ", " : "", h[3 * b], h[3 * b + 1], h[3 * b + 2]);
        for (int u = off[b]; u < off[b + 1]; ++u)
          fprintf(f, "%s[%d, %d, %d, %d]", u > off[b] ? ", " : "", ut[u], uc[u], u0[u], u1[u]);
        fprintf(f, "]]");
      }
      fprintf(f, "]}\n");
      fclose(f);
    }
  }
  launch_k(k_gfin, dim3(num_sms * GF_CTAS_PER_SM), dim3(256), 0, st, (const float*)gpart, a.nchunks, qp, meta, gslots);
}

// Tile order of the 2-CTA GEMM per shape class (pair_tile).  Measured defaults
// (profiles/r1_gemm_raster.md, r2_gemm_raster.md); tuning overrides, read per launch:
// LOBRA_GEMM_GM_SMALL (weight <= 48 MB), LOBRA_GEMM_GM_NBIG (large weight, N >= K),
// LOBRA_GEMM_GM_KBIG (large weight, K > N).
int gemm_group_m(int N, int K) {
  const bool big = (double)N * K * 2 > 48e6;
  const char* key = !big ? "LOBRA_GEMM_GM_SMALL" : (K > N ? "LOBRA_GEMM_GM_KBIG" : "LOBRA_GEMM_GM_NBIG");
  if (const char* e = getenv(key)) return atoi(e);
  // N = 11008 (gate/up fwd, down bwd): 16-block groups; K = 11008 (down fwd, gate/up bwd):
  // N-fastest -- C3 DRAM bytes per launch 6.5 / 10.3 GB vs 10-18 / 12-20 GB for the other
  // orders tried, 2-5% shorter launches (profiles/r2_gemm_raster.md)
  return !big ? 1 : (K > N ? 1 : 16);
}


void launch_gemm(bool b_mn, const CUtensorMap& mapZ, const CUtensorMap& mapW,
                 const CUtensorMap& mapSlot, const CUtensorMap& mapVext, int T, int N, int K,
                 __nv_bfloat16* C, int accumulate, const Meta& meta, int num_sms,
                 cudaStream_t st, const TpScatter* tp) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_gemm2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM);
    cudaFuncSetAttribute(k_gemm2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM);
    init = true;
  }
  Gemm2Args a;
  a.T = T;
  a.N = N;
  a.K = K;
  a.ntm2 = (T + 255) / 256;
  a.ntn = (N + 255) / 256;
  a.accumulate = accumulate;
  a.C = C;
  a.meta = meta;
  a.tp = tp ? *tp : TpScatter{};
  a.group_m = gemm_group_m(N, K);
  const int tiles = a.ntm2 * a.ntn;
  int clusters = num_sms / 2;
  if (tiles < clusters) clusters = tiles;
  if (b_mn)
    launch_k(k_gemm2<true>, dim3(2 * clusters), dim3(G_THREADS), P_SMEM, st, mapZ, mapW, mapSlot, mapVext, a);
  else
    launch_k(k_gemm2<false>, dim3(2 * clusters), dim3(G_THREADS), P_SMEM, st, mapZ, mapW, mapSlot, mapVext, a);
}

void launch_segred(const CUtensorMap& mapZ, const CUtensorMap& mapSlot, int width,
                   const Meta& meta, float* partial, int num_sms, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_segred, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
    init = true;
  }
  SegArgs a;
  a.width = width;
  a.nchunks = (width + 127) / 128;
  a.nitems = meta.nsrseg;
  a.partial = partial;
  a.meta = meta;
  if (a.nitems == 0 || meta.nsrcta == 0) return;
  launch_k(k_segred, dim3(meta.nsrcta), dim3(256), S_SMEM, st, mapZ, mapSlot, a);
}

void launch_finalize_multi(const FinJob* jobs, int n, const Meta& meta, cudaStream_t st) {
  if (meta.rsum == 0 || n <= 0) return;
  FinJobs J{};
  int wmax = 1;
  for (int i = 0; i < n && i < kMaxFinJobs; ++i) J.j[i] = jobs[i], wmax = std::max(wmax, jobs[i].width);
  J.n = std::min(n, kMaxFinJobs);
  launch_k(k_finalize_multi, dim3((wmax + 127) / 128, (meta.rsum + 7) / 8, J.n), dim3(256), 0, st, J, meta);
}

void launch_zero_f32(float* p, long long n, cudaStream_t st) {
  if (n > 0) launch_k(k_zero, dim3(296), dim3(256), 0, st, p, n);
}

}  // namespace lobra
