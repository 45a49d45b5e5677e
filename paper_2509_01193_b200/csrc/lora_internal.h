// Internal (non-ABI) declarations shared by the host planner and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lobra.h"

namespace lobra {

constexpr int kTileM = 128;     // rows (tokens) per M tile == rows per adapter "slot"
constexpr int kSlotW = 64;      // slot width: ranks padded to 64 columns (r_t <= 64)

// Batch metadata resident in the workspace (int32 unless noted).  Built on the host
// from (seq_lens, seq_task, ranks) and copied once per call.
//   segments: maximal runs of equal task in packing order, rows [seg_off[i], seg_off[i+1])
//   slots:    one per (M tile, task present in the tile), tile-major; slot s holds the
//             128 x 64 block of H_s (or G_s) rows of that tile for that task, zeros in the
//             rows of other tasks (the block-stacked K-extension layout)
//   units:    split of each task's slot list into contiguous ranges for the token
//             reductions dA/dB (deterministic two-pass reduction)
struct Meta {
  int T, nseg, ntiles, nslots, ntasks, nunits, rsum, max_slots_per_tile;
  int qp;                    // max over tasks of rank padded to 16 (partials' q stride)
  int band;                  // projection group: this projection's first column in the 64-wide
                             // H/G slots (0 for a single projection); multiple of 16
  const int* seg_off;        // [nseg+1]
  const int* seg_task;       // [nseg]
  const int* tile_slot_off;  // [ntiles+1]
  const int* slot_task;      // [nslots]
  const int* slot_tile;      // [nslots]
  const int* task_slot_off;  // [ntasks+1]
  const int* task_slots;     // [nslots]
  const int* unit_task;      // [nunits]
  const int* unit_s0;        // [nunits] range into task_slots
  const int* unit_s1;        // [nunits]
  const int* task_unit_off;  // [ntasks+1]
  // segments of the fused dY pass (task, 512-column chunk, range [s0, s1) of the task's slot
  // list); CTA b runs segments [dy_cta_off[b], dy_cta_off[b+1]) (static balanced schedule,
  // ndycta CTAs); the segments of (task t, chunk c) are [dy_task_unit_off[t*dy_nch + c],
  // dy_task_unit_off[t*dy_nch + c + 1]) (k_finalize_multi sums them in order)
  int ndyunits, use_dy_units, ndycta, dy_nch;
  const int* dy_unit_task;
  const int* dy_unit_s0;
  const int* dy_unit_s1;
  const int* dy_unit_chunk;
  const int* dy_cta_off;
  const int* dy_task_unit_off;
  // token-reduction (k_segred) schedule: the same static balanced cut as the dY pass over
  // (task, 128-column chunk, slot) entries; CTA b runs segments [sr_cta_off[b], sr_cta_off[b+1])
  // (nsrcta CTAs), segment partials [seg][qp][128]; the segments of (t, c) are
  // [sr_tc_off[t*sr_nch + c], sr_tc_off[t*sr_nch + c + 1])
  int nsrseg, nsrcta, sr_nch;
  const int* sr_task;
  const int* sr_s0;
  const int* sr_s1;
  const int* sr_chunk;
  const int* sr_cta_off;
  const int* sr_tc_off;
  const int* ranks;          // [ntasks]
  const int* roff;           // [ntasks+1]
  const int* boff;           // [ntasks+1] task column offset in the B operand the kernels read
                             // (== roff when every rank is a multiple of 8, else the padded copy's)
  const float* scales;       // [ntasks]
};

__device__ __forceinline__ int row_task(const Meta& m, int row) {
  int lo = 0, hi = m.nseg - 1;
  while (lo < hi) {  // last segment with seg_off <= row
    const int mid = (lo + hi + 1) >> 1;
    if (m.seg_off[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return m.seg_task[lo];
}

// ---- bf16 launchers (kernels_bf16.cu) ---------------------------------------------
// B_cat [out, rsum] -> Bp [out, ld8] with task t's columns at boff[t] (8-aligned, zero
// padded): only when some rank is not a multiple of 8 (TMA needs 16-byte aligned inner
// coordinates and strides).
// one library kernel launch (lora_host.cu): every launcher calls it after enqueueing
void note_launch();

void launch_pad_cols(const __nv_bfloat16* src, __nv_bfloat16* dst, int out, int ld8,
                     const Meta& meta, cudaStream_t st);
// Split factor of the rank-r projection for `ntiles` tiles and reduction length K.
int rowproj_splits(int ntiles, int K);
// slot[s] = s_t * Z[rows of tile] V_t for every slot of every tile (zeros in rows of other
// tasks and in columns q >= r_t).  v_mn = false: V = A_cat [rsum, K] (forward shrink);
// v_mn = true: V = B_cat [K, ld8] (backward G).  partial/counters: split-K scratch.
void launch_rowproj(bool v_mn, const CUtensorMap& mapZ, const CUtensorMap& mapV, int K,
                    const Meta& meta, __nv_bfloat16* slots, float* partial, int* counters,
                    cudaStream_t st);
// Forward shrink without split-K (one CTA per tile, persistent, whole K): used when the
// tiles fill >= 3/4 of the SMs (LOBRA_SHRINK=0 disables).  mapV: the adapter operand
// (A_cat, or the packed group A) with box {64, meta.qp}.
bool shrink_applies(int ntiles, int num_sms);
// planes: a projection group whose bands do not fit one 64-wide slot (np * pq > 64, <= 256):
// ONE pass over X (meta.qp = np * pq rows of the packed group A per task), projection p's H_s
// written to its own single-projection slot buffer `slots + p * plane_stride` (elements).
struct ShrinkPlanes {
  int np, pq;
  long long plane_stride;
  const int* ranks;     // device: the tasks' ranks / scales (meta of the single projections)
  const float* scales;
};
void launch_shrink(const CUtensorMap& mapZ, const CUtensorMap& mapV, int K, const Meta& meta,
                   __nv_bfloat16* slots, int num_sms, cudaStream_t st,
                   const ShrinkPlanes* planes = nullptr);
// LDGSTS-producer variant (default; LOBRA_RP_TMA=1 selects the TMA-producer kernel):
// Z raw [T, K]; mapVk K-major adapter operand, box {64, qp} (A_cat forward, B^T backward).
bool rowproj_uses_ld();
void launch_rowproj_ld(const __nv_bfloat16* Z, int K, const CUtensorMap& mapVk, int qp,
                       const Meta& meta, __nv_bfloat16* slots, float* partial, int* counters,
                       cudaStream_t st);
// Projection group (np <= 4 projections sharing X and the task ranks): A_grp rows
// (t * np + p) * qp + j = A_p[roff[t] + j] for j < r_t, zero otherwise.
void launch_pack_a_group(const __nv_bfloat16* const* A, int np, int qp, int in, const Meta& meta,
                         __nv_bfloat16* dst, cudaStream_t st);
// B [out, rsum] -> Bt [rsum, out]
void launch_transpose_b(const __nv_bfloat16* B, __nv_bfloat16* Bt, int out, int rsum, cudaStream_t st);
// C[T, N] (+)= Z[T,K] . Wop  +  sum over tile slots: Slot[128, r] . Vext_t
//   b_mn = false: Wop = W^T with W [N, K] K-major (forward, X W^T); Vext = B_cat [N, ld8]
//   b_mn = true : Wop = W   with W [K, N] (MN-major B operand; backward, dY W);
//                 Vext = A_cat [rsum, N] (MN-major)
// true: the 2-CTA (cta_group::2) GEMM is used; its B boxes are 128 rows/columns per CTA
// (env LOBRA_GEMM_1CTA=1 selects the 1-CTA kernel with 256-wide boxes).
// bf16 2D TMA map, 128-byte swizzle (lora_host.cu)
lobra_status make_tensor_map_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                                uint32_t box_inner, uint32_t box_outer);
// host metadata -> device (`bytes` % 4 == 0, dst 16-byte aligned) through the library's
// pinned staging ring and k_meta_copy, in stream order on st (lora_host.cu)
lobra_status upload_host_meta(const void* src, size_t bytes, void* dst, cudaStream_t st);
// Fused GEMM -> TP reduce-scatter (symm.cu): output row r is stored into rank
// (r / chunk_rows)'s symmetric buffer, slot `rank`, row r % chunk_rows (bf16 [chunk_rows, N]
// per slot) instead of C (with accumulate, the row of C is added first: C holds the local
// partial).  peer == nullptr: plain C.  2-CTA GEMM only.
struct TpScatter {
  uint8_t* const* peer = nullptr;   // device table of the group's buffer bases
  long long data_off = 0;           // bytes from a base to its data area
  int rank = 0, chunk_rows = 1;
};
void launch_gemm(bool b_mn, const CUtensorMap& mapZ, const CUtensorMap& mapW,
                 const CUtensorMap& mapSlot, const CUtensorMap& mapVext, int T, int N, int K,
                 __nv_bfloat16* C, int accumulate, const Meta& meta, int num_sms, cudaStream_t st,
                 const TpScatter* tp = nullptr);
// partial[seg][q][128] = sum over the segment's slots: Z[tile rows, chunk cols]^T Slot, for the
// segments of meta's k_segred schedule (set for this width)
void launch_segred(const CUtensorMap& mapZ, const CUtensorMap& mapSlot, int width,
                   const Meta& meta, float* partial, int num_sms, cudaStream_t st);
// Fused dY pass (G slots + dB partials in one dY read) followed by the G finalize.
// mapH / mapBt: boxes {dypass_span(qp) / 2, 128 tokens} over the H slots and
// {dypass_span(qp) / 2, 64 o} over B, swizzled with span dypass_span(qp) bytes.
int dypass_span(int qp);
void launch_dypass(const CUtensorMap& mapDY, const CUtensorMap& mapH, const CUtensorMap& mapBt,
                   int width, int qp, const Meta& meta, float* gpart, float* bpart,
                   __nv_bfloat16* gslots, int num_sms, cudaStream_t st);
// One launch for several finalizations: mode 0 dA [r, width] rows with stride ld, mode 1 dB
// [width, rsum] (PEFT layout); out = (accumulate ? out : 0) + sum of the partials in fixed order.
// uoff: the task's unit offsets (meta.task_unit_off) or, with dy = 1, (task, chunk) segment
// offsets (meta.dy_task_unit_off of the dY pass with sub = 4 blocks of 128 columns per segment,
// or meta.sr_tc_off of k_segred with sub = 1), dy_nch chunks per task.
struct FinJob {
  const float* partial;
  float* out;
  long long ld;
  const int* uoff;
  int mode, width, nchunks, band, qp, dy, dy_nch, accumulate;
  int sub = 4;   // with dy = 1: 128-column blocks per segment (4: fused dY pass, 1: k_segred)
};
constexpr int kMaxFinJobs = 8;
struct FinJobs {
  FinJob j[kMaxFinJobs];
  int n;
};
void launch_finalize_multi(const FinJob* jobs, int n, const Meta& meta, cudaStream_t st);
// Zero (or leave) the dA/dB of every task when the batch has no tokens.
void launch_zero_f32(float* p, long long n, cudaStream_t st);

// ---- fp32 SIMT launchers (kernels_fp32.cu) ----------------------------------------
// fwd (dir 0): H [T,64] = s_t X A_t^T;   bwd (dir 1): G [T,64] = s_t dY B_t
void launch_f32_rowproj(int dir, const float* Z, const float* A, const float* B, int in, int out,
                        const Meta& meta, float* H, cudaStream_t st);
// fwd: Y = X W^T + H B_t^T ; bwd: dX (+)= dY W + G A_t
void launch_f32_gemm(int dir, const float* Z, const float* W, const float* A, const float* B,
                     const float* H, int in, int out, const Meta& meta, float* C, int accumulate,
                     cudaStream_t st);
// dA_t (dir 0) = sum G^T X  (rows stride ld) ; dB_t (dir 1) = sum dY^T H
void launch_f32_segred(int dir, const float* Z, const float* H, int width, const Meta& meta,
                       float* out, long long ld, int accumulate, cudaStream_t st);

}  // namespace lobra
