// Streaming-read probe for the skinny (rank-r) kernels: how fast can a [T, K] bf16 row-major
// activation be read tile by tile (128-row M tiles, split-K over CTAs) with different
// producers?  No tensor work: each stage is consumed by one warp arriving on the empty
// barrier.  Output: one line per configuration with the achieved read bandwidth.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_01193_b200/csrc \
//        tools/probe_stream.cu -o /tmp/probe_stream && /tmp/probe_stream
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"
using namespace lobra::ptx;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 g_encode;

struct Cfg {
  int box_rows, box_cols, swz, nb, stages, nsplit, mfast, pad_kb, spin, mma_n, vrows;
};

// TMA producer: stage = nb adjacent boxes of box_rows x box_cols along K
__global__ void __launch_bounds__(256, 1) k_tma(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap mapv, int T, int K,
                                               Cfg c, int ntiles, unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = c.box_rows * c.box_cols * 2;
  const int stage_bytes = c.nb * box_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + c.stages * stage_bytes);   // bars in the first 1 KB after stages
  uint64_t* empty = full + 16;
  uint64_t* done = empty + 16;
  const int m = c.mfast ? blockIdx.x % ntiles : blockIdx.x / c.nsplit;
  const int split = c.mfast ? blockIdx.x / ntiles : blockIdx.x % c.nsplit;
  const int ncb = K / c.box_cols;                         // column boxes per row
  const int per = (ncb + c.nsplit - 1) / c.nsplit;
  const int cb0 = split * per, cb1 = min(ncb, cb0 + per);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < c.stages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 96) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int cb = cb0; cb < cb1; cb += c.nb) {
      const int n = min(c.nb, cb1 - cb);
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_expect_tx(&full[stage], n * box_bytes + (c.vrows ? n * c.vrows * 128 : 0));
      for (int j = 0; j < n; ++j)
        tma_load_2d(smem + stage * stage_bytes + j * box_bytes, &map, &full[stage], (cb + j) * c.box_cols,
                    m * c.box_rows);
      if (c.vrows)
        for (int j = 0; j < n; ++j)
          tma_load_2d(smem + c.stages * stage_bytes + 2048 + j * 8192, &mapv, &full[stage], (cb + j) * 64, 0);
      if (++stage == c.stages) stage = 0, phase ^= 1;
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long acc = 0;
    const uint32_t id = idesc_bf16(128, c.mma_n ? c.mma_n : 16, false, false);
    const uint32_t tm = *tmem_slot;
    const uint32_t vb = smem_u32(smem + c.stages * stage_bytes + 2048);   // B operand (V boxes land here)
    for (int cb = cb0; cb < cb1; cb += c.nb) {
      mbar_wait(&full[stage], phase);
      if (c.mma_n) {
        tc_fence_after();
        const uint32_t st0 = smem_u32(smem + stage * stage_bytes);
        for (int j = 0; j < c.nb; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16(tm, sdesc_sw128(st0 + j * box_bytes + k * 32, 16, 1024), sdesc_sw128(vb + k * 32, 16, 1024), id,
                     (cb != cb0 || j || k) ? 1u : 0u);
        mma_commit(&empty[stage]);
      } else {
        acc += *reinterpret_cast<volatile uint32_t*>(smem + stage * stage_bytes);
        mbar_arrive(&empty[stage]);
      }
      if (++stage == c.stages) stage = 0, phase ^= 1;
    }
    if (acc == 0x123456789ull) *sink = acc;
    mbar_arrive(done);
  } else if (threadIdx.x >= 128 && c.spin) {   // rowproj-like epilogue warps waiting
    mbar_wait(done, 0);
  }
  __syncthreads();
  if (threadIdx.x >= 64 && threadIdx.x < 96) tmem_dealloc<128>(*tmem_slot);
}

// LDG producer: 256 threads; each warp reads `seg` contiguous bytes of a row per step
template <int UNROLL>
__global__ void __launch_bounds__(256) k_ldg(const uint4* __restrict__ Z, int T, int K, int nsplit, int seg,
                                             unsigned long long* sink) {
  const int m = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  const int rowv = K / 8;                         // uint4 per row
  const int per = rowv / nsplit;
  const int v0 = split * per;
  const int lanes_per_row = seg / 16;             // 32 -> one row per warp step
  const int rows_per_warp_step = 32 / lanes_per_row;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (int cv = 0; cv < per; cv += lanes_per_row) {
    // 8 warps x rows_per_warp_step rows per pass, 128 rows
    uint4 v[UNROLL];
    for (int r0 = warp * rows_per_warp_step; r0 < 128; r0 += 8 * rows_per_warp_step * UNROLL) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int r = r0 + u * 8 * rows_per_warp_step + lane / lanes_per_row;
        const int row = m * 128 + r;
        v[u] = (r < 128 && row < T) ? __ldcs(Z + (size_t)row * rowv + v0 + cv + lane % lanes_per_row)
                                    : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_fill_random(uint32_t* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0x3fff3fffu) | 0x3c003c00u;   // two bf16 in [1, 4) with random mantissas
  }
}

// plain linear read (the copy-roofline reference)
__global__ void __launch_bounds__(256) k_linear(const uint4* __restrict__ Z, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(Z + i), b = __ldcs(Z + i + stride), c = __ldcs(Z + i + 2 * stride), d = __ldcs(Z + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldcs(Z + i).x;
  if (acc == 0x12345678u) *sink = acc;
}

static void make_map(CUtensorMap* map, void* ptr, int K, int T, int bc, int br, int swz) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)T};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d (box %d x %d)\n", (int)r, bc, br); exit(1); }
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int T = 16384;
  const int Ks[2] = {4096, 11008};
  void* Z;
  CK(cudaMalloc(&Z, (size_t)T * 11008 * 2));
  CK(cudaMemset(Z, 1, (size_t)T * 11008 * 2));
  void* V;
  CK(cudaMalloc(&V, (size_t)64 * 11008 * 2));
  CK(cudaMemset(V, 0, (size_t)64 * 11008 * 2));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  auto timeit = [&](auto launch, double bytes, const char* name) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-72s %8.1f us  %7.0f GB/s\n", name, 1e3 * ms / reps, bytes * reps / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
  for (int rnd = 0; rnd < 2; ++rnd) {
  if (rnd) { k_fill_random<<<1184, 256>>>((uint32_t*)Z, (size_t)T * 11008 / 2); CK(cudaDeviceSynchronize()); printf("--- random data\n"); }
  for (int K : Ks) {
    const double bytes = (double)T * K * 2;
    char name[256];
    snprintf(name, sizeof name, "K=%d linear LDG.128 (copy-read reference)", K);
    timeit([&] { k_linear<<<148 * 8, 256>>>((const uint4*)Z, (size_t)T * K / 8, sink); }, bytes, name);
    for (int seg : {512})
      for (int nsplit : {4}) {
        snprintf(name, sizeof name, "K=%d LDG tile 128 rows, %d B/row/step, nsplit %d", K, seg, nsplit);
        timeit([&] { k_ldg<4><<<(T / 128) * nsplit, 256>>>((const uint4*)Z, T, K, nsplit, seg, sink); }, bytes, name);
      }
    std::vector<Cfg> cfgs;
    cfgs.push_back({128, 64, 1, 2, 5, 1, 0, 0, 0, 16, 16});
    cfgs.push_back({128, 64, 1, 2, 5, 1, 0, 0, 0, 0, 0});
    for (const Cfg& c : cfgs) {
      CUtensorMap map, mapv;
      make_map(&map, Z, K, T, c.box_cols, c.box_rows, c.swz);
      make_map(&mapv, V, K, 64, 64, c.vrows ? c.vrows : 16, 1);
      const int ntiles = T / c.box_rows;
      const int smem = c.stages * c.nb * c.box_rows * c.box_cols * 2 + 1024 + 2048 + 16384 + c.pad_kb * 1024;
      if (smem > 227 * 1024) continue;
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma, 256, smem));
      snprintf(name, sizeof name, "K=%d TMA box %dx%dB%s nb %d st %d nsplit %d %s%s mma_n %d vrows %d (%d CTA/SM, grid %d)", K,
               c.box_rows, c.box_cols * 2, c.swz ? " sw128" : "", c.nb, c.stages, c.nsplit,
               c.mfast ? "m-fast" : "split-fast", c.spin ? " +4 spin warps" : "", c.mma_n, c.vrows, occ, ntiles * c.nsplit);
      timeit([&] { k_tma<<<ntiles * c.nsplit, 256, smem>>>(map, mapv, T, K, c, ntiles, sink); }, bytes, name);
    }
  }
  }
  CK(cudaGetLastError());
  return 0;
}
