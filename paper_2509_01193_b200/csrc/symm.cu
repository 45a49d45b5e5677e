// Own TP all-reduce over peer memory (Megatron row-parallel forward Y and
// column-parallel backward dX all-reduces), replacing NCCL for the TP group.
//
// Every rank of a TP group allocates one symmetric buffer [flags | data] and maps its peers'
// buffers with CUDA IPC (NVLink / NVSwitch peer access inside a node: plain loads and stores
// to peer memory).  The all-reduce of n elements is two-shot and deterministic:
//   barrier A (every partial is in its owner's data area)
//   reduce-scatter: rank r sums chunk r of all P partials in rank order 0..P-1 (fp32),
//                   writes the rounded sum in place into its own chunk r
//   barrier B (every chunk reduced)
//   all-gather:     every rank copies chunk c from rank c into its output
//   barrier C (peers finished reading before the next call overwrites the data area)
// so every rank gets bitwise the same result.  Barriers are epoch flags written into the
// peers' flag areas with st.release.sys and polled with ld.acquire.sys; epochs only grow,
// so flags are never reset.  The projection GEMMs can write their partial straight into
// the data area (lobra_symm_data), which turns "GEMM -> all-reduce" into GEMM -> peer
// reduction with no staging copy.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.h"
#include "lora_internal.h"

namespace lobra {
int64_t count_launch(int kind, cudaStream_t st, bool begin);   // lora_host.cu
}

struct lobra_symm_s {
  int rank = 0, world = 1;
  size_t bytes = 0;          // data bytes per rank
  uint8_t* base = nullptr;   // own allocation: [kHdr flags | data]
  std::vector<uint8_t*> peer;          // peer bases (own base at [rank])
  uint8_t** d_peer = nullptr;          // device copy of peer bases
  uint64_t epoch = 0;
  bool opened = false;
};

namespace lobra {
namespace {

constexpr size_t kHdr = 4096;   // 3 barrier kinds x 64 ranks x 8 bytes, padded
constexpr int kMaxRanks = 64;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One CTA: signal `epoch` into every peer's flag slot [kind][rank], then wait for all peers.
__global__ void k_symm_barrier(uint8_t* const* __restrict__ peer, int rank, int world, int kind, uint64_t epoch) {
  __threadfence_system();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < world && t != rank)
    st_release_sys(reinterpret_cast<uint64_t*>(peer[t]) + kind * kMaxRanks + rank, epoch);
  if (t < world && t != rank) {
    const uint64_t* f = reinterpret_cast<const uint64_t*>(peer[rank]) + kind * kMaxRanks + t;
    // a peer that never arrives (a crashed rank, a broken mapping) must not hang the GPU:
    // after 300 s (far beyond any start-up skew between ranks) the kernel traps and the
    // error surfaces at the caller's next sync
    uint64_t t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (uint32_t spin = 0; ld_acquire_sys(f) < epoch; ++spin) {
      if ((spin & 0xFFFF) == 0xFFFF) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        if (t1 - t0 > 300000000000ull) __trap();
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void add(float* acc, const uint4& u) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] += f.x, acc[2 * i + 1] += f.y;
    }
  }
  static __device__ __forceinline__ uint4 pack(const float* a) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
    return u;
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void add(float* acc, const uint4& u) {
    const float* f = reinterpret_cast<const float*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += f[i];
  }
  static __device__ __forceinline__ uint4 pack(const float* a) {
    uint4 u;
    float* f = reinterpret_cast<float*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = a[i];
    return u;
  }
};

// chunk c = vectors [c * cv, min(nv, (c + 1) * cv))
template <typename T>
__global__ void k_symm_reduce_scatter(uint8_t* const* __restrict__ peer, int rank, int world, long long nv,
                                      long long cv) {
  const long long v0 = rank * cv, v1 = min(nv, v0 + cv);
  for (long long v = v0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; v < v1;
       v += (long long)gridDim.x * blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < world; ++p)   // fixed rank order: every rank computes the same bits
      Vec<T>::add(acc, reinterpret_cast<const uint4*>(peer[p] + kHdr)[v]);
    reinterpret_cast<uint4*>(peer[rank] + kHdr)[v] = Vec<T>::pack(acc);
  }
}

template <typename T>
__global__ void k_symm_all_gather(uint8_t* const* __restrict__ peer, int world, long long nv, long long cv,
                                  uint4* __restrict__ dst) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(v / cv);
    dst[v] = reinterpret_cast<const uint4*>(peer[c] + kHdr)[v];
  }
}

// Fused path, after the GEMM stored row r of its partial into rank (r / chunk)'s slot
// [this rank]: the owner sums its chunk over the slots in rank order (local memory only) into
// its own slot, in place.
__global__ void k_tp_reduce_rows(uint8_t* const* __restrict__ peer, int rank, int world, long long chunk_rows,
                                 long long rows_here, int nv_row /* uint4 per row */) {
  uint8_t* base = peer[rank] + kHdr;
  const long long slot_v = chunk_rows * nv_row;
  const long long total = rows_here * nv_row;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
       v += (long long)gridDim.x * blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < world; ++p)
      Vec<__nv_bfloat16>::add(acc, reinterpret_cast<const uint4*>(base)[p * slot_v + v]);
    reinterpret_cast<uint4*>(base)[rank * slot_v + v] = Vec<__nv_bfloat16>::pack(acc);
  }
}

// dst row r <- owner (r / chunk)'s reduced slot
__global__ void k_tp_gather_rows(uint8_t* const* __restrict__ peer, long long chunk_rows, long long T, int nv_row,
                                 uint4* __restrict__ dst) {
  const long long total = T * nv_row;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
       v += (long long)gridDim.x * blockDim.x) {
    const long long row = v / nv_row;
    const int c = (int)(row / chunk_rows);
    const long long local = v - c * chunk_rows * nv_row;
    dst[v] = reinterpret_cast<const uint4*>(peer[c] + kHdr)[c * chunk_rows * nv_row + local];
  }
}

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

// count elements of type T, src and dst local device buffers (either may be the data area)
template <typename T>
lobra_status symm_allreduce(lobra_symm s, const void* src, void* dst, size_t count, cudaStream_t st) {
  if (!s || !s->opened) return fail(LOBRA_ERR_INPUT, "symmetric buffer not opened");
  const size_t bytes = count * sizeof(T);
  if (bytes > s->bytes) return fail(LOBRA_ERR_INPUT, "all-reduce of %zu bytes exceeds the symmetric buffer (%zu)", bytes, s->bytes);
  if (bytes % 16) return fail(LOBRA_ERR_INPUT, "all-reduce size must be a multiple of 16 bytes");
  if (count == 0) return LOBRA_OK;
  uint8_t* data = s->base + kHdr;
  if (src != data && cudaMemcpyAsync(data, src, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "symm: staging copy failed");
  const long long nv = (long long)(bytes / 16);
  const long long cv = (nv + s->world - 1) / s->world;
  const uint64_t e = ++s->epoch;
  const int grid = 4 * sms();
  auto counted = [&](auto&& launch) {
    count_launch(LOBRA_K_COMM, st, true);
    launch();
    count_launch(LOBRA_K_COMM, st, false);
  };
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 0, e); });
  counted([&] { k_symm_reduce_scatter<T><<<grid, 256, 0, st>>>(s->d_peer, s->rank, s->world, nv, cv); });
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 1, e); });
  counted([&] { k_symm_all_gather<T><<<grid, 256, 0, st>>>(s->d_peer, s->world, nv, cv, static_cast<uint4*>(dst)); });
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 2, e); });
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(LOBRA_ERR_CUDA, "symm all-reduce: %s", cudaGetErrorString(err));
  return LOBRA_OK;
}
template lobra_status symm_allreduce<__nv_bfloat16>(lobra_symm, const void*, void*, size_t, cudaStream_t);
template lobra_status symm_allreduce<float>(lobra_symm, const void*, void*, size_t, cudaStream_t);

// Target of the fused GEMM -> reduce-scatter for a [T, N] bf16 result (nullptr-peer target
// when the buffer cannot hold world x ceil(T / world) rows of N).
bool symm_scatter_target(lobra_symm s, long long T, long long N, TpScatter* out) {
  if (!s || !s->opened || T <= 0) return false;
  const long long chunk = (T + s->world - 1) / s->world;
  if ((size_t)(s->world * chunk * N * 2) > s->bytes) return false;
  out->peer = s->d_peer;
  out->data_off = (long long)kHdr;
  out->rank = s->rank;
  out->chunk_rows = (int)chunk;
  return true;
}

// After the fused GEMM: barrier, owner-local reduction of its row chunk, barrier, gather of
// every chunk into dst [T, N], barrier.  Same rank-order fp32 sums as symm_allreduce.
lobra_status symm_scatter_finish(lobra_symm s, long long T, long long N, void* dst, cudaStream_t st) {
  const long long chunk = (T + s->world - 1) / s->world;
  const long long r0 = s->rank * chunk, rows_here = std::max(0LL, std::min(T, r0 + chunk) - r0);
  const int nv_row = (int)(N / 8);
  const uint64_t e = ++s->epoch;
  const int grid = 4 * sms();
  auto counted = [&](auto&& launch) {
    count_launch(LOBRA_K_COMM, st, true);
    launch();
    count_launch(LOBRA_K_COMM, st, false);
  };
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 0, e); });
  if (rows_here > 0)
    counted([&] { k_tp_reduce_rows<<<grid, 256, 0, st>>>(s->d_peer, s->rank, s->world, chunk, rows_here, nv_row); });
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 1, e); });
  counted([&] { k_tp_gather_rows<<<grid, 256, 0, st>>>(s->d_peer, chunk, T, nv_row, static_cast<uint4*>(dst)); });
  counted([&] { k_symm_barrier<<<1, 64, 0, st>>>(s->d_peer, s->rank, s->world, 2, e); });
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(LOBRA_ERR_CUDA, "fused TP reduce-scatter: %s", cudaGetErrorString(err));
  return LOBRA_OK;
}

void* symm_data(lobra_symm s) { return s ? s->base + kHdr : nullptr; }
size_t symm_capacity(lobra_symm s) { return s ? s->bytes : 0; }
int symm_world(lobra_symm s) { return s ? s->world : 0; }
int symm_rank(lobra_symm s) { return s ? s->rank : 0; }

}  // namespace lobra

using namespace lobra;

extern "C" lobra_status lobra_symm_create(int32_t rank, int32_t world, size_t bytes, lobra_symm* out,
                                          void* ipc_handle_out) {
  clear_error();
  if (!out || !ipc_handle_out || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || bytes % 16)
    return fail(LOBRA_ERR_INPUT, "symm_create: need 1 <= world <= %d, 0 <= rank < world, bytes %% 16 == 0", kMaxRanks);
  lobra_symm s = new lobra_symm_s();
  s->rank = rank, s->world = world, s->bytes = bytes;
  if (cudaMalloc(&s->base, kHdr + bytes) != cudaSuccess) {
    delete s;
    return fail(LOBRA_ERR_CUDA, "symm_create: cudaMalloc(%zu) failed", kHdr + bytes);
  }
  cudaMemset(s->base, 0, kHdr);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, s->base) != cudaSuccess) {
    cudaFree(s->base);
    delete s;
    return fail(LOBRA_ERR_CUDA, "symm_create: cudaIpcGetMemHandle failed");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  memcpy(ipc_handle_out, &h, 64);
  cudaDeviceSynchronize();   // the zeroed flags are visible before any peer opens the buffer
  *out = s;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_symm_open(lobra_symm s, const void* handles) {
  clear_error();
  if (!s || !handles) return fail(LOBRA_ERR_INPUT, "symm_open: null argument");
  if (s->opened) return fail(LOBRA_ERR_INPUT, "symm_open: already opened");
  s->peer.assign(s->world, nullptr);
  for (int p = 0; p < s->world; ++p) {
    if (p == s->rank) {
      s->peer[p] = s->base;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * p, 64);
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "symm_open: peer %d: %s", p, cudaGetErrorString(e));
    s->peer[p] = static_cast<uint8_t*>(ptr);
  }
  if (cudaMalloc(&s->d_peer, sizeof(uint8_t*) * s->world) != cudaSuccess ||
      cudaMemcpy(s->d_peer, s->peer.data(), sizeof(uint8_t*) * s->world, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "symm_open: peer table upload failed");
  s->opened = true;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_symm_destroy(lobra_symm s) {
  clear_error();
  if (!s) return LOBRA_OK;
  cudaDeviceSynchronize();
  for (int p = 0; p < (int)s->peer.size(); ++p)
    if (p != s->rank && s->peer[p]) cudaIpcCloseMemHandle(s->peer[p]);
  if (s->d_peer) cudaFree(s->d_peer);
  if (s->base) cudaFree(s->base);
  delete s;
  return LOBRA_OK;
}

extern "C" void* lobra_symm_data(lobra_symm s) { return symm_data(s); }

extern "C" lobra_status lobra_symm_allreduce(lobra_symm s, int32_t dtype, const void* src, void* dst, size_t count,
                                             lobra_stream_t stream) {
  clear_error();
  if (!src || !dst) return fail(LOBRA_ERR_INPUT, "symm_allreduce: null buffer");
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return fail(LOBRA_ERR_INPUT, "symm_allreduce: buffers must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == LOBRA_BF16) return symm_allreduce<__nv_bfloat16>(s, src, dst, count, st);
  if (dtype == LOBRA_FP32) return symm_allreduce<float>(s, src, dst, count, st);
  return fail(LOBRA_ERR_INPUT, "symm_allreduce: unknown dtype %d", dtype);
}
