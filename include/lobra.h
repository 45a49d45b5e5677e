/*
 * lobra.h -- C ABI of the B200-native LobRA multi-LoRA hot path.
 *
 * Paper: "LobRA: Multi-tenant Fine-tuning over Heterogeneous Data" (arXiv 2509.01193),
 * /root/reference/PAPER.md, cited as P:<line> with its section / equation.
 *
 * The library computes, for a packed batch of variable-length sequences of many
 * fine-tuning tasks ("fuse the input data from different tasks so that the
 * computation of the base model can be fused into a batched operation whilst the
 * computation of multiple LoRA adapters can be supported by customized operations";
 * packing P:261-266), the forward and backward of ONE frozen base projection plus the
 * tasks' LoRA adapters (§2.1 "computes XW + XBA"):
 *
 *     for every token row x of a sequence of task t:
 *        y  = x W^T + s_t (x A_t^T) B_t^T                       (forward)
 *        dx = dy W  + s_t (dy B_t) A_t                           (backward, W frozen
 *        dA_t += s_t sum_rows (dy B_t)^T x                        P:74: no dW)
 *        dB_t += s_t sum_rows dy^T (x A_t^T)
 *
 * Names: A_t is the "shrink" (paper's B), B_t the "expand" (paper's A); storage is
 * PyTorch/PEFT style (reading Q24):
 *     W   [out, in]    row-major (torch Linear.weight; a TP rank passes its local shard)
 *     A   [sum_t r_t, in]   task t's rows start at roff[t] = sum_{u<t} r_u   (lora_A)
 *     B   [out, sum_t r_t]  task t's columns start at roff[t]               (lora_B)
 *     X   [T, in], Y [T, out], dY [T, out], dX [T, in]  row-major, T = sum seq_lens
 *     dA  [sum_t r_t, in] fp32 (row stride problem.dA_ld), dB [out, sum_t r_t] fp32
 *
 * It also implements the per-step workload-balanced dispatch (Eq. 3 and
 * dynamic bucketing) and the adapter-gradient all-reduce across FT replicas (P:170,
 * P:306 "must synchronize the parameters of LoRA adapters for every training step").
 *
 * Conventions (all entry points):
 *  - Every function returns lobra_status; nothing throws across the ABI.
 *  - All host-side checks run BEFORE any device work is enqueued; on error nothing is
 *    enqueued and lobra_last_error() says why (thread-local string, valid until the
 *    next call on the same thread).
 *  - Device work is enqueued on the caller's stream in stream order; there is no
 *    implicit device synchronisation.  Asynchronous CUDA faults surface at the
 *    caller's next synchronisation.
 *  - The caller allocates and owns every device buffer (X, W, A, B, Y, Hs, dX, dA, dB,
 *    workspace).  The library never allocates device memory on the hot path.  Host
 *    arrays are only read during the call.  A lazily created per-device context
 *    (SM count, a small ring of pinned host staging buffers) is freed by
 *    lobra_shutdown().
 *  - Calls on different streams are safe if their workspaces do not alias.
 *  - Requires an sm_100 (B200) device for the compute entry points
 *    (LOBRA_ERR_UNSUPPORTED otherwise).
 */
#ifndef LOBRA_H_
#define LOBRA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LOBRA_API __attribute__((visibility("default")))
#else
#define LOBRA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lobra_stream_t;   /* == cudaStream_t */

/* Status codes; 1-3 reuse SPEC.md's CLI exit codes. */
typedef enum {
  LOBRA_OK = 0,
  LOBRA_ERR_INPUT = 1,        /* bad argument: shape, alignment, rank, task id, ...    */
  LOBRA_ERR_INFEASIBLE = 2,   /* dispatch: a sequence fits no deployed replica, or     */
                              /* exceeds the grid ("re-plan required")          */
  LOBRA_ERR_BUDGET = 3,       /* dispatch: Eq. 3 solver node cap hit; the best         */
                              /* incumbent found is returned                   */
  LOBRA_ERR_CUDA = 4,         /* a CUDA runtime/driver call failed                     */
  LOBRA_ERR_NCCL = 5,         /* an NCCL call failed, or NCCL could not be loaded      */
  LOBRA_ERR_UNSUPPORTED = 6   /* device is not sm_100, or configuration not supported  */
} lobra_status;

/* Human-readable reason for the last non-OK status on this thread. */
LOBRA_API const char* lobra_last_error(void);

/* Library version string, e.g. "lobra-b200 0.1 (sm_100a)". */
LOBRA_API const char* lobra_version(void);

typedef enum { LOBRA_BF16 = 0, LOBRA_FP32 = 1 } lobra_dtype;

/* Megatron tensor parallelism of the base projection inside one FT replica
 * (§2.2).  COLUMN: W sharded along `out` (q,k,v,gate,up); the backward
 * all-reduces dX over the TP group.  ROW: W sharded along `in` (o,down); the forward
 * all-reduces Y over the TP group.  The LoRA adapters add no collective (DESIGN.md
 * "Multi-GPU").  NONE: unsharded, no collective. */
typedef enum { LOBRA_TP_NONE = 0, LOBRA_TP_COLUMN = 1, LOBRA_TP_ROW = 2 } lobra_tp_kind;

/* The packed batch (host arrays).  Sequence k occupies rows [off_k, off_k + seq_lens[k])
 * of X/Y/dY/dX, off_k = sum_{j<k} seq_lens[j]; its task is seq_task[k] in
 * [0, num_tasks).  P:256-266 (packing, block-diagonal: rows of different sequences never
 * interact in a projection).  Any order is accepted; grouping sequences by task (what
 * lobra_dispatch emits) minimises mixed-task tiles.  num_seqs >= 1, seq_lens[k] >= 0. */
typedef struct {
  int32_t num_seqs;
  const int32_t* seq_lens;
  const int32_t* seq_task;
} lobra_batch;

/* The tasks' adapters for this projection.  ranks/scales are host arrays of length
 * num_tasks; 1 <= ranks[t] <= 64 (reading Q4); scales are s_t (reading Q2,
 * the paper has no scale).  A and B are DEVICE pointers in the dtype of the problem,
 * laid out as described at the top of this file (for a TP rank: its local shard, i.e.
 * COLUMN: B holds the rank's `out` rows; ROW: A holds the rank's `in` columns,
 * contiguous [sum r, in_local]). */
typedef struct {
  int32_t num_tasks;
  const int32_t* ranks;
  const float* scales;
  const void* A;
  const void* B;
} lobra_adapters;

typedef struct lobra_comm_s* lobra_comm;   /* opaque: NCCL world comm + TP sub-comm */

/* One projection.  in/out are the LOCAL (per-rank) widths.  bf16: in and out must be
 * multiples of 64.  fp32: any positive sizes.  dA_ld: row stride (elements) of the dA
 * output (0 = in); lets a ROW-parallel rank write its column slice of a full-size flat
 * gradient buffer.  tp may be NULL when tp_kind == LOBRA_TP_NONE. */
typedef struct {
  lobra_dtype dtype;
  int64_t in;
  int64_t out;
  lobra_tp_kind tp_kind;
  lobra_comm tp;
  int64_t dA_ld;
} lobra_problem;

/* Bytes of device workspace lobra_lora_fwd / lobra_lora_bwd need for this problem and
 * batch (both directions; 256-byte aligned pointer required).  Returns 0 and sets the
 * last error on invalid input. */
LOBRA_API size_t lobra_lora_workspace_bytes(const lobra_problem* prob, const lobra_batch* batch,
                                  const lobra_adapters* ad);

/* Bytes of the opaque saved state `Hs` (the pre-scaled shrink H_s = s_t X A_t^T in the
 * library's per-row-tile layout) that lobra_lora_fwd writes and lobra_lora_bwd reads. */
LOBRA_API size_t lobra_lora_saved_bytes(const lobra_problem* prob, const lobra_batch* batch,
                              const lobra_adapters* ad);

/* Forward: Y = X W^T + s_t (X A_t^T) B_t^T per task segment.
 * X [T,in], W [out,in], Y [T,out] device; Hs (saved for bwd) and ws device scratch.
 * ROW-parallel with a comm: Y is summed over the TP group (ncclAllReduce, in place).
 * Errors: LOBRA_ERR_INPUT (shapes/alignment/ranks/task ids/workspace too small),
 * LOBRA_ERR_UNSUPPORTED (not sm_100), LOBRA_ERR_CUDA, LOBRA_ERR_NCCL. */
LOBRA_API lobra_status lobra_lora_fwd(const lobra_problem* prob, const lobra_batch* batch,
                            const lobra_adapters* ad, const void* X, const void* W, void* Y,
                            void* Hs, void* ws, size_t ws_bytes, lobra_stream_t stream);

/* Backward (W frozen: P:74):
 *   dX  = dY W + s_t (dY B_t) A_t             (written, or added to dX if accumulate_dx)
 *   dA_t = s_t sum (dY B_t)^T X  [r_t, in]     fp32 (written, or added if accumulate_dadb)
 *   dB_t = s_t sum dY^T (X A_t^T) [out, r_t]   fp32 (same)
 * Gradient sums are plain sums over the call's tokens (reading Q7); a task with no
 * tokens leaves its dA/dB untouched when accumulating and writes zeros otherwise
 * (reading Q10).  Hs must come from lobra_lora_fwd on the same batch/adapters.
 * COLUMN-parallel with a comm: dX is summed over the TP group (in place).
 * dA_t/dB_t reductions are deterministic (fixed order; no atomics). */
LOBRA_API lobra_status lobra_lora_bwd(const lobra_problem* prob, const lobra_batch* batch,
                            const lobra_adapters* ad, const void* X, const void* W,
                            const void* Hs, const void* dY, void* dX, int accumulate_dx,
                            float* dA, float* dB, int accumulate_dadb, void* ws,
                            size_t ws_bytes, lobra_stream_t stream);

/* ------------------------------------------------------------------------------
 * Projection groups ("inputs sharing X are done in one pass: {q,k,v}
 * uses A_cat = [A_q; A_k; A_v] of width 3r; {gate,up} uses width 2r").
 * num_proj (1..4) projections that read the same X [T, in] and share the task set, the
 * ranks and the scales (one LoRA configuration per task).  Projection p has
 * W_p [out_p, in], A_p [sum r, in], B_p [out_p, sum r] in the single-projection layouts
 * above.  Results equal num_proj lobra_lora_fwd / lobra_lora_bwd calls (backward:
 * dX (+)= sum_p dX_p, i.e. the single calls with accumulate_dx = 1 after the first), but
 * X is read ONCE for all the shrinks H_s,p and ONCE for all the dA_p reductions: the
 * H_s / G_s slots hold one qp-column band per projection (qp = max rank padded to 16;
 * bands used when num_proj * qp <= 64 and dtype is bf16).  Otherwise the call runs the
 * num_proj single-projection sequences internally (same results); for bf16 with
 * 64 < num_proj * qp <= 256 and a batch that fills >= 3/4 of the SMs with 128-token tiles,
 * the forward still reads X once: one shrink pass writes every projection's H_s into its
 * own single-projection slot buffer inside Hs (the dA reductions stay per projection).
 * TP: all projections of a group have tp_kind; a COLUMN group all-reduces dX once at the
 * end of the backward; a ROW group all-reduces every Y_p in the forward.
 * Hs: one buffer of lobra_lora_group_saved_bytes bytes, written by the forward, read by
 * the backward.  Host arrays (out, A, B, W, Y, dY, dA, dB pointer arrays) are read during
 * the call only.  Errors as for the single-projection calls (checked for every p).
 * ------------------------------------------------------------------------------ */
typedef struct {
  lobra_dtype dtype;
  int64_t in;                  /* shared input width                                      */
  int32_t num_proj;            /* 1..4                                                    */
  const int64_t* out;          /* [num_proj] host: out_p (this rank's shard)              */
  lobra_tp_kind tp_kind;       /* same for every projection of the group                  */
  lobra_comm tp;
  int64_t dA_ld;               /* row stride of every dA_p (0 = in)                       */
} lobra_group_problem;

typedef struct {
  int32_t num_tasks;
  const int32_t* ranks;        /* [num_tasks] host, shared by the group                   */
  const float* scales;         /* [num_tasks] host, shared by the group                   */
  const void* const* A;        /* [num_proj] host array of device pointers: A_p            */
  const void* const* B;        /* [num_proj] host array of device pointers: B_p            */
} lobra_group_adapters;

LOBRA_API size_t lobra_lora_group_workspace_bytes(const lobra_group_problem* prob,
                                                  const lobra_batch* batch,
                                                  const lobra_group_adapters* ad);
LOBRA_API size_t lobra_lora_group_saved_bytes(const lobra_group_problem* prob,
                                              const lobra_batch* batch,
                                              const lobra_group_adapters* ad);
LOBRA_API lobra_status lobra_lora_group_fwd(const lobra_group_problem* prob,
                                            const lobra_batch* batch,
                                            const lobra_group_adapters* ad, const void* X,
                                            const void* const* W, void* const* Y, void* Hs,
                                            void* ws, size_t ws_bytes, lobra_stream_t stream);
LOBRA_API lobra_status lobra_lora_group_bwd(const lobra_group_problem* prob,
                                            const lobra_batch* batch,
                                            const lobra_group_adapters* ad, const void* X,
                                            const void* const* W, const void* Hs,
                                            const void* const* dY, void* dX, int accumulate_dx,
                                            float* const* dA, float* const* dB,
                                            int accumulate_dadb, void* ws, size_t ws_bytes,
                                            lobra_stream_t stream);

/* ------------------------------------------------------------------------------
 * Decoder-layer operations around the LoRA projections (one Llama layer,
 * the unit the paper's cost model profiles, App. D).  Public Llama-2 definitions
 * (reading Q27); bf16 tensors, fp32 arithmetic, one rounding per output.
 * Device pointers 16-byte aligned; widths multiples of 8.  Host-side checks run before any
 * launch (LOBRA_ERR_INPUT); launch failures -> LOBRA_ERR_CUDA.
 *
 * lobra_rmsnorm_fwd: S = X + R (R may be NULL: S = X; when R != NULL S is written to S_out),
 *   Y = S / sqrt(mean_row(S^2) + eps) * g, rstd[row] = 1 / sqrt(mean_row(S^2) + eps) (fp32,
 *   saved for the backward).  X, R, S_out, Y [T, h]; g [h]; h <= 16384.
 * lobra_rmsnorm_bwd: with u = g * dY (g frozen, no dg):
 *   dS = rstd u - S rstd^3 (u . S) / h  (+ dRes when dRes != NULL: the residual stream's
 *   gradient, fused), written to dS [T, h].
 * ------------------------------------------------------------------------------ */
LOBRA_API lobra_status lobra_rmsnorm_fwd(int64_t T, int64_t h, const void* X, const void* R,
                                         void* S_out, const void* g, float eps, void* Y,
                                         float* rstd, lobra_stream_t stream);
LOBRA_API lobra_status lobra_rmsnorm_bwd(int64_t T, int64_t h, const void* dY, const void* S,
                                         const void* g, const float* rstd, const void* dRes,
                                         void* dS, lobra_stream_t stream);
/* lobra_rope: rotary position embedding IN PLACE on Q [T, n_heads * head_dim] (row stride
 *   ldq elements) and, if K != NULL, on K (stride ldk): the position of a token is its index
 *   inside its own packed sequence (restarts at 0, cu_seqlens: device int32 [num_seqs + 1]
 *   prefix offsets), angle_j = pos * theta^(-2j / head_dim) for j < head_dim / 2, pairs
 *   (j, j + head_dim/2): (a, b) -> (a cos - b sin, b cos + a sin); inverse != 0 rotates by
 *   -angle (the backward).  head_dim % 16 == 0. */
LOBRA_API lobra_status lobra_rope(int32_t num_seqs, const int32_t* cu_seqlens, int64_t T,
                                  int32_t n_heads, int32_t head_dim, float theta, void* Q,
                                  int64_t ldq, void* K, int64_t ldk, int inverse,
                                  lobra_stream_t stream);
/* lobra_swiglu_fwd: act = silu(gate) * up, elementwise over n (n % 8 == 0).
 * lobra_swiglu_bwd: with s = sigmoid(gate): d_gate = d up s (1 + gate (1 - s)),
 *   d_up = d gate s. */
LOBRA_API lobra_status lobra_swiglu_fwd(int64_t n, const void* gate, const void* up, void* act,
                                        lobra_stream_t stream);
LOBRA_API lobra_status lobra_swiglu_bwd(int64_t n, const void* d, const void* gate, const void* up,
                                        void* d_gate, void* d_up, lobra_stream_t stream);
/* lobra_attn_fwd: causal attention inside every packed sequence (block-diagonal mask over
 *   the pack; seq_lens host [num_seqs]), tcgen05 kernel.  Q [T, n_heads * 128],
 *   K, V [T, n_kv_heads * 128] bf16 row-major (n_kv_heads | n_heads: grouped-query heads);
 *   O [T, n_heads * 128] bf16; lse [n_heads, T] fp32 = natural-log softmax normaliser per
 *   query (FlashAttention's varlen layout).  scale 1 / sqrt(128).  head_dim must be 128
 *   (else LOBRA_ERR_UNSUPPORTED).  ws >= lobra_attn_workspace_bytes device bytes. */
LOBRA_API size_t lobra_attn_workspace_bytes(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads);
LOBRA_API lobra_status lobra_attn_fwd(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                      int32_t n_kv_heads, int32_t head_dim, const void* Q, const void* K,
                                      const void* V, void* O, float* lse, void* ws, size_t ws_bytes,
                                      lobra_stream_t stream);
/* lobra_attn_bwd: gradients of lobra_attn_fwd (FlashAttention's recomputation: P is rebuilt
 *   from Q, K and the forward's lse, never stored).  Per query row: Dq = sum_d dO O,
 *   P = exp(Q K^T / sqrt(128) - lse) under the same causal, per-sequence mask,
 *   dS = P (dO V^T - Dq); dQ = dS K / sqrt(128), dK = dS^T Q / sqrt(128), dV = P^T dO, summed
 *   over the query heads of each kv head.  Layouts as lobra_attn_fwd; O, dO, dQ
 *   [T, n_heads * 128] bf16; dK, dV [T, n_kv_heads * 128] bf16 (overwritten; rows of every
 *   sequence written, padding none).  P and dS are rounded to bf16 before their products
 *   (as FlashAttention does), accumulation in fp32 (TMEM; dQ through an fp32 buffer in ws).
 *   ws >= lobra_attn_bwd_workspace_bytes device bytes, 16-byte aligned pointers, head_dim
 *   128 (else LOBRA_ERR_UNSUPPORTED).  Three launches (pre: Dq + zeroed dQ accumulator;
 *   main; post: dQ scale + bf16). */
LOBRA_API size_t lobra_attn_bwd_workspace_bytes(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                                int32_t n_kv_heads);
LOBRA_API lobra_status lobra_attn_bwd(int32_t num_seqs, const int32_t* seq_lens, int32_t n_heads,
                                      int32_t n_kv_heads, int32_t head_dim, const void* Q, const void* K,
                                      const void* V, const void* O, const void* dO, const float* lse,
                                      void* dQ, void* dK, void* dV, void* ws, size_t ws_bytes,
                                      lobra_stream_t stream);
/* lobra_add: C = A + B elementwise over n bf16 (n % 8 == 0; C may alias A or B): the
 * layer's last residual add. */
LOBRA_API lobra_status lobra_add(int64_t n, const void* A, const void* B, void* C, lobra_stream_t stream);

/* ------------------------------------------------------------------------------
 * Per-step dispatch (host only, deterministic; every rank may compute it locally).
 * Implements P:591-619 (dynamic bucketing DP over the grid u_k = k*grid_step,
 * k = 1..grid_max/grid_step, empty intervals ignored, lexicographically smallest optimal
 * boundary list), r_i = #{j : s_j <= M_i} (Table tab:notations), Eq. 3
 * solved exactly with the App. D cost T_i = sum_j c_ij ceil(d_ij / p_i)
 * and the canonical tie-break "lexicographically smallest d in (group, bucket)
 * order", then: bucket j's sequences in ascending index go to groups in order; within a
 * group a per-bucket round robin starting at the replica with the smallest running
 * cost; chunks of floor(M_i / s_j) sequences ordered by descending cost;
 * inside a chunk sequences ordered by (task id, index).  See DESIGN.md "Dispatch".
 * ------------------------------------------------------------------------------ */
typedef struct {
  int32_t num_groups;          /* G; groups ordered by (tp asc, max_tokens asc)        */
  const int32_t* tp;           /* [G] n_i: GPUs per replica (TP degree)                 */
  const int32_t* replicas;     /* [G] p_i >= 0 (0 = configuration not deployed)         */
  const int32_t* max_tokens;   /* [G] M_i: max tokens per chunk, multiple of grid_step  */
  const int64_t* cost;         /* [G * U] integer cost of ONE sequence padded to grid   */
                               /* value u_k = (k+1)*grid_step, k = 0..U-1 (reading Q15) */
} lobra_deployment;

typedef struct {
  int32_t num_buckets;         /* out: R' <= R buckets actually formed                   */
  int32_t* boundaries;         /* [R] out: s_1 < ... < s_R'                               */
  int64_t* d;                  /* [G * R] out: d_ij, row-major with row stride R          */
  int32_t* seq_bucket;         /* [n] out: bucket index of every sequence                 */
  int32_t* seq_replica;        /* [n] out: global replica id (group-major numbering)      */
  int32_t* seq_chunk;          /* [n] out: chunk (micro-batch) index within the replica   */
  int32_t* pack_order;         /* [n] out: position of the sequence inside its chunk      */
  int64_t* replica_cost;       /* [sum p_i] out: assigned cost per replica                */
  int64_t t_hat;               /* out: Eq. 3 objective max_i sum_j c_ij ceil(d_ij/p_i)    */
  int64_t nodes;               /* out: branch-and-bound nodes explored                    */
} lobra_dispatch_out;

/* mode: 0 = balanced (Eq. 3), 1 = length-based (Fig. 4(c): every bucket to the
 * supporting group with the smallest c_ij * n_i, ties to the earlier group), 2 = uniform
 * (Task-Fused baseline: exactly one deployed homogeneous group, the k-th
 * sequence goes to replica k mod p).
 * chunking: 0 = padded micro-batches of App. D (per bucket, b_j = floor(M_i / s_j)
 * sequences); 1 = packed micro-batches ("can also be applied when
 * packing is employed"; reading Q6b): the replica's sequences in (bucket desc, index)
 * order filled next-fit into chunks of at most M_i REAL tokens.
 * Eq. 3 (mode 0) is solved exactly: 1 group trivially, 2 groups by a pseudo-polynomial DP,
 * >= 3 groups by branch-and-bound over the replica rounds q_ij = ceil(d_ij / p_i) (LP and
 * per-bucket integer-covering Lagrangian bounds) followed by the lexicographic
 * canonicalisation of reading Q12 (csrc/eq3_bb.cpp).
 * node_cap: branch-and-bound node budget for >= 3 groups (<= 0: default 1e6 nodes, ~5-10 s);
 * when it is exhausted the call returns LOBRA_ERR_BUDGET with the LENGTH-BASED d (mode 1's)
 * in `out` -- never a silent substitute: the status says the Eq. 3 optimum was not reached.
 * With >= 3 deployed groups the branch-and-bound subtrees run on a thread pool created for
 * the call (LOBRA_DISPATCH_THREADS, default hardware threads - 1, at most 16); the result
 * does not depend on the thread count.
 * Errors: LOBRA_ERR_INPUT, LOBRA_ERR_INFEASIBLE, LOBRA_ERR_BUDGET.  Host only; thread-safe
 * (no global state). */
LOBRA_API lobra_status lobra_dispatch(const lobra_deployment* dep, const lobra_batch* batch,
                            int32_t grid_step, int32_t grid_max, int32_t R, int32_t mode,
                            int32_t chunking, int64_t node_cap, lobra_dispatch_out* out);

/* ------------------------------------------------------------------------------
 * Stage-1 deployment planning (§4.2 Eq. 2, App. A, PP = 1).
 *  1. bucket a length sample with the dynamic-bucketing DP ("randomly sample a
 *     large number (100 x B by default) of training data and perform the bucketing");
 *  2. demands B_j = ceil(batch_size * f_j), f_j = sample fraction of bucket j (reading
 *     Q22); batch_size = 0 uses the sample's bucket counts as the demands (Eq. 1 with a
 *     concrete batch);
 *  3. configuration proposal (App. A Observation 1): a candidate is dropped when another
 *     with the same GPU count supports at least as long sequences at no higher cost;
 *  4. enumerate the maximal plans sum_i p_i n_i <= N covering every demanded bucket
 *     (App. A "integer partition problem");
 *  5. Theorem-1 lower bound (App. A): length-based dispatch times t_i, bound
 *     sum_i N_i t_i / sum_i N_i; keep plans within (1 + threshold) of the minimum bound
 *     (threshold < 0: keep all; 0.15 in the paper);
 *  6. solve Eq. 3 exactly for every kept plan; return the best (ties: fewer GPUs, fewer
 *     replicas, lexicographically smaller p).
 * Host only, deterministic.  Errors: LOBRA_ERR_INPUT, LOBRA_ERR_INFEASIBLE (no plan covers
 * the longest bucket), LOBRA_ERR_BUDGET (a per-plan solve hit node_cap; best incumbent).
 * ------------------------------------------------------------------------------ */
typedef struct {
  int32_t num_configs;         /* S candidate configurations                             */
  const int32_t* tp;           /* [S] n_i GPUs per replica                                */
  const int32_t* max_tokens;   /* [S] M_i, multiple of grid_step                         */
  const int64_t* cost;         /* [S * U] integer cost of one sequence at grid value u_k */
} lobra_candidates;

typedef struct {
  int32_t* replicas;           /* [S] out: p_i (0 = not deployed)                         */
  int32_t* boundaries;         /* [R] out: bucket boundaries                              */
  int64_t* demands;            /* [R] out: B_j                                            */
  int32_t num_buckets;         /* out                                                     */
  int32_t plans_total;         /* out: maximal covering plans                             */
  int32_t plans_solved;        /* out: plans kept by the Theorem-1 filter (each decided exactly: solved, or proven worse than the best by its Eq. 3 lower bound) */
  int32_t gpus_used;           /* out                                                     */
  int64_t t_hat;               /* out: Eq. 3 objective of the chosen plan                 */
} lobra_plan_out;

LOBRA_API lobra_status lobra_plan_deployment(const lobra_candidates* cand, int32_t n_gpus,
                                             const int32_t* lens, int32_t n_lens,
                                             int32_t batch_size, int32_t grid_step,
                                             int32_t grid_max, int32_t R, double threshold,
                                             int64_t node_cap, lobra_plan_out* out);

/* ------------------------------------------------------------------------------
 * Configuration proposal from a profiled throughput table (App. A "Configuration
 * Proposal": "SELECT config, MAX(thruput) FROM thruput_table GROUP BY
 * num_gpus, seq_len"; Table tb:parallel_config_thruputs).
 * Reading Q26: a configuration with n_c = tp * pp GPUs per replica competes in
 * every group (g = gpu_counts[k], seq_len[l]) with n_c <= g and g % n_c == 0, as g / n_c
 * replicas at its own per-GPU throughput (the table's "-": "the throughput remains the same
 * after model replication").  The group winner has the maximum throughput; ties go to fewer
 * GPUs per replica, then smaller TP, then smaller PP, then lower index.  Exact double
 * comparisons (no tolerance).
 *   thruput : [C * L] row-major, tokens per GPU per second of one replica of config c at
 *             seq_len[l]; <= 0 (or NaN) = cannot run that length (out of memory)
 *   winner  : [K * L] out, config index of each group, -1 when no configuration runs it
 *   keep    : [C] out, 1 for the proposed configurations (winners of at least one group)
 * Host only.  Errors: LOBRA_ERR_INPUT (null/empty arrays, tp or pp < 1, gpu_counts < 1).
 * ------------------------------------------------------------------------------ */
typedef struct {
  int32_t num_configs;         /* C                                                       */
  const int32_t* tp;           /* [C] TP degree                                           */
  const int32_t* pp;           /* [C] PP degree (GPUs per replica = tp * pp)              */
  int32_t num_lens;            /* L                                                       */
  const int32_t* seq_len;      /* [L] profiled sequence lengths                           */
  const double* thruput;       /* [C * L]                                                 */
  int32_t num_gpu_counts;      /* K                                                       */
  const int32_t* gpu_counts;   /* [K] the table's num_gpus columns                        */
} lobra_thruput_table;

LOBRA_API lobra_status lobra_propose_configs(const lobra_thruput_table* table, int32_t* winner,
                                             int32_t* keep);

/* ------------------------------------------------------------------------------
 * Replica time cost model, App. D, with 1F1B pipeline parallel.
 * Bucket j holds d[j] >= 0 sequences of (padded) length s[j], 1 <= s[j] <= max_tokens (M,
 * the configuration's maximum supportable length); full micro-batches hold
 * b_j = floor(M / s_j) sequences: d_j = m_j b_j + r_j.  With the fitted per-chunk time
 * t(b, s) = c0 + c1 b s + c2 b s^2 (b >= 1; t(0, s) = 0; reading Q28):
 *   *out = sum_j (m_j t(b_j, s_j) + t(r_j, s_j)) + (pp_stages - 1) x (longest existing chunk)
 * (Eq. appendix_cost_model_pp_varlen; pp_stages = 1 is the no-PP equation; reading Q29: the
 * max ranges over the chunks that exist).  Host only, no device work.
 * Errors: LOBRA_ERR_INPUT for num_buckets < 1, pp_stages < 1, max_tokens < 1, a null pointer,
 * d[j] < 0 or s[j] outside [1, max_tokens]. */
LOBRA_API lobra_status lobra_replica_time(int32_t num_buckets, const int32_t* d, const int32_t* s,
                                          int64_t max_tokens, int32_t pp_stages, double c0,
                                          double c1, double c2, double* out);

/* ------------------------------------------------------------------------------
 * Communication (NCCL over NVLink/NVSwitch).  One process per GPU.
 * ------------------------------------------------------------------------------ */
/* Rank 0 creates a 128-byte NCCL unique id; the caller broadcasts it (e.g. with
 * torch.distributed.broadcast_object_list) to all ranks. */
LOBRA_API lobra_status lobra_nccl_unique_id(void* out128);

/* World communicator over all `world` ranks plus the TP sub-communicator of this
 * rank's FT replica: ncclCommSplit(color = replica_id, key = rank).  Collective: every
 * rank must call it.  The current CUDA device must be set by the caller. */
LOBRA_API lobra_status lobra_comm_init(const void* id128, int32_t world, int32_t rank,
                             int32_t replica_id, lobra_comm* out);
LOBRA_API lobra_status lobra_comm_destroy(lobra_comm comm);
/* TP group size / rank of this process inside its replica. */
LOBRA_API lobra_status lobra_comm_tp_info(lobra_comm comm, int32_t* tp_size, int32_t* tp_rank);

/* Adapter-gradient synchronisation across FT replicas: in-place SUM of
 * the flat fp32 buffer over the WORLD communicator (reading Q7: sum, not mean).  Every
 * rank passes a buffer with the identical full-size layout holding its partial sums
 * (zeros where it owns nothing). */
/* ------------------------------------------------------------------------------
 * Own TP collective over peer memory (Megatron row-parallel Y and
 * column-parallel dX all-reduces).  Every rank of a group allocates one
 * symmetric device buffer of `bytes` data bytes (lobra_symm_create returns its 64-byte CUDA
 * IPC handle), the caller exchanges the handles (any transport, e.g. torch.distributed) and
 * lobra_symm_open maps the peers' buffers (NVLink / NVSwitch peer access inside a node).
 * lobra_symm_allreduce: dst = sum over ranks of src, two-shot (reduce-scatter in rank order
 *   0..P-1 with fp32 accumulation, then all-gather) with epoch-flag barriers, so every rank
 *   gets bitwise the same result; src / dst local device buffers (src may be the data area:
 *   lobra_symm_data, then no staging copy), count * sizeof(dtype) <= bytes, multiple of 16.
 *   Every rank must call it with the same count, in the same order.
 * lobra_comm_from_symm: a comm whose TP group (and world) is the symmetric group (no NCCL);
 * lobra_comm_attach_symm: route an NCCL comm's TP all-reduces through the symmetric group.
 * The TP all-reduces of lobra_lora_fwd/bwd (and the group calls) then run on these kernels.
 * ------------------------------------------------------------------------------ */
typedef struct lobra_symm_s* lobra_symm;
LOBRA_API lobra_status lobra_symm_create(int32_t rank, int32_t world, size_t bytes, lobra_symm* out,
                                         void* ipc_handle_out);
LOBRA_API lobra_status lobra_symm_open(lobra_symm s, const void* handles /* world x 64 bytes */);
LOBRA_API lobra_status lobra_symm_destroy(lobra_symm s);
LOBRA_API void* lobra_symm_data(lobra_symm s);
LOBRA_API lobra_status lobra_symm_allreduce(lobra_symm s, int32_t dtype, const void* src, void* dst,
                                            size_t count, lobra_stream_t stream);
LOBRA_API lobra_status lobra_comm_from_symm(lobra_symm s, lobra_comm* out);
LOBRA_API lobra_status lobra_comm_attach_symm(lobra_comm comm, lobra_symm s);

LOBRA_API lobra_status lobra_adapter_allreduce(lobra_comm comm, float* flat_grads, size_t count,
                                     lobra_stream_t stream);

/* ------------------------------------------------------------------------------
 * Adapter optimizer: one AdamW step ("We use the Adam optimizer
 * [adam, adamw]"; decoupled weight decay):
 *     g = grad_scale * grad;  m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
 *     p = p - lr * ( (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps) + wd * p )
 * over a flat fp32 master-parameter buffer with per-group hyper-parameters (multi-tenant:
 * one group per task).  params/m/v are updated in place; grads are read.  group: device
 * uint8 [count] group id per element, or NULL (every element in group 0); elements whose
 * id is >= num_groups are left untouched.  hp: host array [num_groups], 1 <= num_groups
 * <= 64.  hp[k].step is group k's own step count t >= 1 in the bias corrections (a task
 * that joined later has taken fewer steps than the others); 0 = use `step`.
 * params_bf16: optional device bf16 [count] copy of the updated parameters (what the LoRA
 * kernels read), or NULL.  All device pointers 16-byte aligned.  Errors: LOBRA_ERR_INPUT,
 * LOBRA_ERR_CUDA.
 * ------------------------------------------------------------------------------ */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int64_t step;
} lobra_adamw_hparams;
LOBRA_API lobra_status lobra_adamw_step(float* params, void* params_bf16, const float* grads,
                                        float* m, float* v, const uint8_t* group, size_t count,
                                        const lobra_adamw_hparams* hp, int32_t num_groups,
                                        int64_t step, float grad_scale, lobra_stream_t stream);

/* ------------------------------------------------------------------------------
 * Tracing: per-kernel-class device times (CUDA events recorded on the launching
 * stream around every kernel the library enqueues, only while enabled) and a launch
 * counter (always on).  The paper's cost model is fitted from such single-layer
 * profiles (App. D).
 * ------------------------------------------------------------------------------ */
enum {
  LOBRA_K_GEMM_FWD = 0,   /* fused base GEMM + LoRA expand, forward            */
  LOBRA_K_GEMM_BWD = 1,   /* fused dY W + G_s A_t, backward                     */
  LOBRA_K_ROWPROJ = 2,    /* rank-r shrink H_s / G_s                            */
  LOBRA_K_SEGRED = 3,     /* token reductions dA_t / dB_t (partials)            */
  LOBRA_K_FINALIZE = 4,   /* fixed-order partial sums                           */
  LOBRA_K_PAD = 5,        /* adapter operand packing                            */
  LOBRA_K_FP32 = 6,       /* fp32 SIMT path kernels                             */
  LOBRA_K_OPT = 7,        /* adapter optimizer (AdamW)                          */
  LOBRA_K_LAYER = 8,      /* decoder-layer elementwise ops (RMSNorm, RoPE, SwiGLU) */
  LOBRA_K_COMM = 9,       /* own peer-memory collectives (lobra_symm_*)          */
  LOBRA_K_NUM = 10
};
typedef struct {
  int64_t count[LOBRA_K_NUM];   /* launches per class since the last reset        */
  double ms[LOBRA_K_NUM];       /* summed device milliseconds per class           */
} lobra_profile;
/* Enables/disables event timing of every launch (off by default). */
LOBRA_API lobra_status lobra_profile_enable(int on);
/* Synchronises the recorded events, fills `out`, and (if reset) clears the counters. */
LOBRA_API lobra_status lobra_profile_read(lobra_profile* out, int reset);
/* Total kernels launched by the library in this process (never reset). */
LOBRA_API int64_t lobra_launch_count(void);

/* Frees the lazily created per-device context(s). */
LOBRA_API lobra_status lobra_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* LOBRA_H_ */
