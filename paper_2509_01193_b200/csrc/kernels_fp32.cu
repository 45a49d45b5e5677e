// fp32 SIMT path (FFMA, fp32 accumulation) of the multi-LoRA forward/backward.
// Used for the 1e-5 parity configuration (BASELINE config 1): TF32 tensor cores cannot
// meet 1e-5, so this path stays on CUDA cores.  Same math and
// same block-diagonal packing semantics as the bf16 path.
#include "lora_internal.h"

namespace lobra {
namespace {

// H[row][q] = s_t * sum_k Z[row][k] * V(t,q,k); zeros for q >= r_t.
// dir 0: Z = X [T,in], V(t,q,k) = A[roff+q][k];  dir 1: Z = dY [T,out], V = B[k][roff+q]
__global__ void k32_rowproj(int dir, const float* __restrict__ Z, const float* __restrict__ A,
                            const float* __restrict__ B, int in, int out, Meta meta,
                            float* __restrict__ H) {
  const int row = blockIdx.x;
  const int q = threadIdx.x;  // 64 threads
  if (row >= meta.T) return;
  const int t = row_task(meta, row);
  float acc = 0.0f;
  if (q < meta.ranks[t]) {
    if (dir == 0) {
      const float* z = Z + (size_t)row * in;
      const float* a = A + (size_t)(meta.roff[t] + q) * in;
      for (int k = 0; k < in; ++k) acc = fmaf(z[k], a[k], acc);
    } else {
      const float* z = Z + (size_t)row * out;
      for (int k = 0; k < out; ++k) acc = fmaf(z[k], B[(size_t)k * meta.rsum + meta.roff[t] + q], acc);
    }
    acc *= meta.scales[t];
  }
  H[(size_t)row * kSlotW + q] = acc;
}

// 16x16 tiled: C[row][n] = sum_k Z[row][k] Wop(k,n) + sum_q H[row][q] E(t,q,n)
//  dir 0: Z = X, K = in, N = out, Wop(k,n) = W[n][k], E = B[n][roff+q]
//  dir 1: Z = dY, K = out, N = in, Wop(k,n) = W[k][n], E = A[roff+q][n]
__global__ void k32_gemm(int dir, const float* __restrict__ Z, const float* __restrict__ W,
                         const float* __restrict__ A, const float* __restrict__ B,
                         const float* __restrict__ H, int in, int out, Meta meta,
                         float* __restrict__ C, int accumulate) {
  __shared__ float sZ[16][17], sW[16][17];
  const int K = dir == 0 ? in : out;
  const int N = dir == 0 ? out : in;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty;
  const int col = blockIdx.x * 16 + tx;
  float acc = 0.0f;
  for (int k0 = 0; k0 < K; k0 += 16) {
    const int zr = blockIdx.y * 16 + ty, zk = k0 + tx;
    sZ[ty][tx] = (zr < meta.T && zk < K) ? Z[(size_t)zr * K + zk] : 0.0f;
    const int wk = k0 + ty, wn = blockIdx.x * 16 + tx;
    float w = 0.0f;
    if (wk < K && wn < N) w = dir == 0 ? W[(size_t)wn * in + wk] : W[(size_t)wk * in + wn];
    sW[ty][tx] = w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = fmaf(sZ[ty][k], sW[k][tx], acc);
    __syncthreads();
  }
  if (row >= meta.T || col >= N) return;
  const int t = row_task(meta, row);
  const float* h = H + (size_t)row * kSlotW;
  for (int q = 0; q < meta.ranks[t]; ++q) {
    const float e = dir == 0 ? B[(size_t)col * meta.rsum + meta.roff[t] + q]
                             : A[(size_t)(meta.roff[t] + q) * in + col];
    acc = fmaf(h[q], e, acc);
  }
  float* c = C + (size_t)row * N + col;
  *c = accumulate ? *c + acc : acc;
}

// dir 0: dA[roff+q][col] = sum_{rows of t} H[row][q] * X[row][col]   (H = G_s)
// dir 1: dB[col][roff+q] = sum_{rows of t} dY[row][col] * H[row][q]   (H = H_s)
// One thread per output element; rows of task t visited segment by segment in packing
// order -> deterministic.
__global__ void k32_segred(int dir, const float* __restrict__ Z, const float* __restrict__ H,
                           int width, Meta meta, float* __restrict__ out, long long ld,
                           int accumulate) {
  const long long total = (long long)meta.rsum * width;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(i % width);
    const int rq = (int)(i / width);
    int t = 0;
    while (meta.roff[t + 1] <= rq) ++t;
    const int q = rq - meta.roff[t];
    float acc = 0.0f;
    for (int sg = 0; sg < meta.nseg; ++sg) {
      if (meta.seg_task[sg] != t) continue;
      for (int row = meta.seg_off[sg]; row < meta.seg_off[sg + 1]; ++row)
        acc = fmaf(H[(size_t)row * kSlotW + q], Z[(size_t)row * width + col], acc);
    }
    float* dst = dir == 0 ? out + (long long)rq * ld + col : out + (long long)col * meta.rsum + rq;
    *dst = accumulate ? *dst + acc : acc;
  }
}

}  // namespace

void launch_f32_rowproj(int dir, const float* Z, const float* A, const float* B, int in, int out,
                        const Meta& meta, float* H, cudaStream_t st) {
  if (meta.T > 0) { k32_rowproj<<<meta.T, kSlotW, 0, st>>>(dir, Z, A, B, in, out, meta, H); note_launch(); }
}

void launch_f32_gemm(int dir, const float* Z, const float* W, const float* A, const float* B,
                     const float* H, int in, int out, const Meta& meta, float* C, int accumulate,
                     cudaStream_t st) {
  const int N = dir == 0 ? out : in;
  dim3 grid((N + 15) / 16, (meta.T + 15) / 16);
  if (meta.T > 0) { k32_gemm<<<grid, dim3(16, 16), 0, st>>>(dir, Z, W, A, B, H, in, out, meta, C, accumulate); note_launch(); }
}

void launch_f32_segred(int dir, const float* Z, const float* H, int width, const Meta& meta,
                       float* out, long long ld, int accumulate, cudaStream_t st) {
  k32_segred<<<592, 256, 0, st>>>(dir, Z, H, width, meta, out, ld, accumulate);
  note_launch();
}

}  // namespace lobra
