// Decoder-layer elementwise operations around the LoRA projections:
// RMSNorm (+ fused residual add / residual-gradient add), rotary embeddings restarted per
// packed sequence, SwiGLU.  All HBM-bound: 16-byte vector accesses, fp32 arithmetic, one
// bf16 rounding per output; the definitions are in include/lobra.h (reading Q27).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "common.h"

namespace lobra {
int64_t count_launch(int kind, cudaStream_t st, bool begin);   // lora_host.cu

namespace {

constexpr int kMaxVec = 8;   // uint4 (8 bf16) per thread per row: h <= 8 * threads * 8

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x, f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < nw ? red[l] : 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// One CTA per row; the row stays in registers between the reduction and the output.
// VPT = 16-byte vectors per thread (h = 8 * VPT * blockDim): a small VPT keeps the
// register file (and so the rows in flight per SM) large.
template <int VPT>
__global__ void __launch_bounds__(1024) k_rmsnorm_fwd(int h, const __nv_bfloat16* __restrict__ X,
                                                      const __nv_bfloat16* __restrict__ R,
                                                      __nv_bfloat16* __restrict__ S_out,
                                                      const __nv_bfloat16* __restrict__ g, float eps,
                                                      __nv_bfloat16* __restrict__ Y, float* __restrict__ rstd) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const int nv = h / 8;
  float s[VPT][8];
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (c < nv) {
      unpack8(__ldg(reinterpret_cast<const uint4*>(X + row * h) + c), s[k]);
      if (R) {
        float r[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(R + row * h) + c), r);
#pragma unroll
        for (int e = 0; e < 8; ++e) s[k][e] = __bfloat162float(__float2bfloat16_rn(s[k][e] + r[e]));
        reinterpret_cast<uint4*>(S_out + row * h)[c] = pack8(s[k]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += s[k][e] * s[k][e];
    }
  }
  const float rs = rsqrtf(block_sum(ss, red) / (float)h + eps);
  if (threadIdx.x == 0) rstd[row] = rs;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (c < nv) {
      float gg[8], y[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(g) + c), gg);
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = s[k][e] * rs * gg[e];
      reinterpret_cast<uint4*>(Y + row * h)[c] = pack8(y);
    }
  }
}

template <int VPT>
__global__ void __launch_bounds__(1024) k_rmsnorm_bwd(int h, const __nv_bfloat16* __restrict__ dY,
                                                      const __nv_bfloat16* __restrict__ S,
                                                      const __nv_bfloat16* __restrict__ g,
                                                      const float* __restrict__ rstd,
                                                      const __nv_bfloat16* __restrict__ dRes,
                                                      __nv_bfloat16* __restrict__ dS) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const int nv = h / 8;
  float u[VPT][8], x[VPT][8];
  float dot = 0.0f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (c < nv) {
      float gg[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(dY + row * h) + c), u[k]);
      unpack8(__ldg(reinterpret_cast<const uint4*>(S + row * h) + c), x[k]);
      unpack8(__ldg(reinterpret_cast<const uint4*>(g) + c), gg);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        u[k][e] *= gg[e];
        dot += u[k][e] * x[k][e];
      }
    }
  }
  const float r = rstd[row];
  const float coef = block_sum(dot, red) * r * r * r / (float)h;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (c < nv) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r * u[k][e] - x[k][e] * coef;
      if (dRes) {
        float d[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(dRes + row * h) + c), d);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] += d[e];
      }
      reinterpret_cast<uint4*>(dS + row * h)[c] = pack8(o);
    }
  }
}

// One thread per (token, 8 consecutive pair indices j, group of kRopeHG heads): the 8
// (cos, sin) pairs are computed once and applied to the group's heads of Q and K; the loads
// of 4 heads are issued before their stores so the read-modify-writes overlap.
constexpr int kRopeHG = 8;
__global__ void k_rope(int num_seqs, const int32_t* __restrict__ cu, long long T, int nh, int D, float log2theta,
                       __nv_bfloat16* __restrict__ Q, long long ldq, __nv_bfloat16* __restrict__ K, long long ldk,
                       float sign) {
  const int half = D / 2, per_tok = half / 8, ngrp = (nh + kRopeHG - 1) / kRopeHG;
  const long long total = T * per_tok * ngrp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int jv = (int)(i % per_tok);
    const int hg = (int)((i / per_tok) % ngrp);
    const long long tok = i / ((long long)per_tok * ngrp);
    int lo = 0, hi = num_seqs - 1;   // last sequence with cu[s] <= tok
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cu[mid] <= tok) lo = mid; else hi = mid - 1;
    }
    const float pos = (float)(tok - cu[lo]);
    float c[8], s[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = jv * 8 + e;
      const float inv = exp2f(-(2.0f * j / (float)D) * log2theta);
      sincosf(pos * inv, &s[e], &c[e]);
      s[e] *= sign;
    }
    const int h0 = hg * kRopeHG, h1 = min(nh, h0 + kRopeHG);
    for (int which = 0; which < 2; ++which) {
      __nv_bfloat16* base = which == 0 ? Q + tok * ldq : (K ? K + tok * ldk : nullptr);
      if (!base) continue;
      for (int hb = h0; hb < h1; hb += 4) {
        uint4 ua[4], ub[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (hb + u < h1) {
            ua[u] = reinterpret_cast<const uint4*>(base + (hb + u) * D)[jv];
            ub[u] = reinterpret_cast<const uint4*>(base + (hb + u) * D + half)[jv];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (hb + u < h1) {
            float a[8], b[8], oa[8], ob[8];
            unpack8(ua[u], a);
            unpack8(ub[u], b);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              oa[e] = a[e] * c[e] - b[e] * s[e];
              ob[e] = b[e] * c[e] + a[e] * s[e];
            }
            reinterpret_cast<uint4*>(base + (hb + u) * D)[jv] = pack8(oa);
            reinterpret_cast<uint4*>(base + (hb + u) * D + half)[jv] = pack8(ob);
          }
      }
    }
  }
}

__global__ void k_swiglu_fwd(long long nv, const __nv_bfloat16* __restrict__ gate, const __nv_bfloat16* __restrict__ up,
                             __nv_bfloat16* __restrict__ act) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float g[8], u[8], o[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(gate) + i), g);
    unpack8(__ldg(reinterpret_cast<const uint4*>(up) + i), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = g[e] / (1.0f + __expf(-g[e])) * u[e];
    reinterpret_cast<uint4*>(act)[i] = pack8(o);
  }
}

__global__ void k_swiglu_bwd(long long nv, const __nv_bfloat16* __restrict__ d, const __nv_bfloat16* __restrict__ gate,
                             const __nv_bfloat16* __restrict__ up, __nv_bfloat16* __restrict__ dg,
                             __nv_bfloat16* __restrict__ du) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float dd[8], g[8], u[8], og[8], ou[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(d) + i), dd);
    unpack8(__ldg(reinterpret_cast<const uint4*>(gate) + i), g);
    unpack8(__ldg(reinterpret_cast<const uint4*>(up) + i), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float sg = 1.0f / (1.0f + __expf(-g[e]));
      og[e] = dd[e] * u[e] * sg * (1.0f + g[e] * (1.0f - sg));
      ou[e] = dd[e] * g[e] * sg;
    }
    reinterpret_cast<uint4*>(dg)[i] = pack8(og);
    reinterpret_cast<uint4*>(du)[i] = pack8(ou);
  }
}

__global__ void k_add(long long nv, const __nv_bfloat16* A, const __nv_bfloat16* B, __nv_bfloat16* C) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float a[8], b[8];
    unpack8(reinterpret_cast<const uint4*>(A)[i], a);
    unpack8(reinterpret_cast<const uint4*>(B)[i], b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    reinterpret_cast<uint4*>(C)[i] = pack8(a);
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

lobra_status done(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return LOBRA_OK;
}

// Row kernels: VPT vectors per thread with blockDim = ceil(h / 8 / VPT) rounded to 32,
// VPT the smallest of {1, 2, 4, 8} keeping blockDim <= 256.
int row_vpt(int64_t h) {
  const int64_t nv = h / 8;
  for (int v : {1, 2, 4, 8})
    if ((nv + v - 1) / v <= 256) return v;
  return kMaxVec;
}
int row_threads(int64_t h, int vpt) {
  const int t = (int)(((h / 8 + vpt - 1) / vpt + 31) / 32 * 32);
  return t < 32 ? 32 : t;
}

template <typename F>
void dispatch_vpt(int vpt, F&& f) {
  switch (vpt) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    default: f(std::integral_constant<int, 8>{}); break;
  }
}

}  // namespace
}  // namespace lobra

using namespace lobra;

extern "C" lobra_status lobra_rmsnorm_fwd(int64_t T, int64_t h, const void* X, const void* R, void* S_out,
                                          const void* g, float eps, void* Y, float* rstd, lobra_stream_t stream) {
  clear_error();
  if (T < 0 || h < 8 || h % 8 || h > 16384) return fail(LOBRA_ERR_INPUT, "rmsnorm: need T >= 0, h % 8 == 0, 8 <= h <= 16384");
  if (!X || !g || !Y || !rstd || (R && !S_out)) return fail(LOBRA_ERR_INPUT, "rmsnorm: null pointer");
  if (!al16(X) || !al16(g) || !al16(Y) || (R && (!al16(R) || !al16(S_out))))
    return fail(LOBRA_ERR_INPUT, "rmsnorm: pointers must be 16-byte aligned");
  if (!(eps >= 0.0f)) return fail(LOBRA_ERR_INPUT, "rmsnorm: eps must be >= 0");
  if (T == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  const int vpt = row_vpt(h);
  dispatch_vpt(vpt, [&](auto V) {
    k_rmsnorm_fwd<decltype(V)::value><<<(unsigned)T, row_threads(h, vpt), 0, st>>>(
        (int)h, static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(R),
        static_cast<__nv_bfloat16*>(S_out), static_cast<const __nv_bfloat16*>(g), eps,
        static_cast<__nv_bfloat16*>(Y), rstd);
  });
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_rmsnorm_fwd");
}

extern "C" lobra_status lobra_rmsnorm_bwd(int64_t T, int64_t h, const void* dY, const void* S, const void* g,
                                          const float* rstd, const void* dRes, void* dS, lobra_stream_t stream) {
  clear_error();
  if (T < 0 || h < 8 || h % 8 || h > 16384) return fail(LOBRA_ERR_INPUT, "rmsnorm: need T >= 0, h % 8 == 0, 8 <= h <= 16384");
  if (!dY || !S || !g || !rstd || !dS) return fail(LOBRA_ERR_INPUT, "rmsnorm_bwd: null pointer");
  if (!al16(dY) || !al16(S) || !al16(g) || !al16(dS) || (dRes && !al16(dRes)))
    return fail(LOBRA_ERR_INPUT, "rmsnorm_bwd: pointers must be 16-byte aligned");
  if (T == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  const int vpt = row_vpt(h);
  dispatch_vpt(vpt, [&](auto V) {
    k_rmsnorm_bwd<decltype(V)::value><<<(unsigned)T, row_threads(h, vpt), 0, st>>>(
        (int)h, static_cast<const __nv_bfloat16*>(dY), static_cast<const __nv_bfloat16*>(S),
        static_cast<const __nv_bfloat16*>(g), rstd, static_cast<const __nv_bfloat16*>(dRes),
        static_cast<__nv_bfloat16*>(dS));
  });
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_rmsnorm_bwd");
}

extern "C" lobra_status lobra_rope(int32_t num_seqs, const int32_t* cu_seqlens, int64_t T, int32_t n_heads,
                                   int32_t head_dim, float theta, void* Q, int64_t ldq, void* K, int64_t ldk,
                                   int inverse, lobra_stream_t stream) {
  clear_error();
  if (num_seqs < 1 || !cu_seqlens || T < 0 || n_heads < 1 || head_dim < 16 || head_dim % 16 || !(theta > 1.0f))
    return fail(LOBRA_ERR_INPUT, "rope: need num_seqs >= 1, head_dim % 16 == 0, theta > 1");
  if (!Q || ldq < (int64_t)n_heads * head_dim || (K && ldk < (int64_t)n_heads * head_dim) || ldq % 8 || (K && ldk % 8))
    return fail(LOBRA_ERR_INPUT, "rope: bad Q/K pointer or row stride");
  if (!al16(Q) || (K && !al16(K))) return fail(LOBRA_ERR_INPUT, "rope: pointers must be 16-byte aligned");
  if (T == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  const long long total = T * (head_dim / 16) * ((n_heads + 7) / 8);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 16LL * sm_count());
  k_rope<<<blocks, 256, 0, st>>>(num_seqs, cu_seqlens, T, n_heads, head_dim, std::log2(theta),
                                 static_cast<__nv_bfloat16*>(Q), ldq, static_cast<__nv_bfloat16*>(K), ldk,
                                 inverse ? -1.0f : 1.0f);
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_rope");
}

extern "C" lobra_status lobra_swiglu_fwd(int64_t n, const void* gate, const void* up, void* act,
                                         lobra_stream_t stream) {
  clear_error();
  if (n < 0 || n % 8 || !gate || !up || !act) return fail(LOBRA_ERR_INPUT, "swiglu: n % 8 == 0 and non-null pointers");
  if (!al16(gate) || !al16(up) || !al16(act)) return fail(LOBRA_ERR_INPUT, "swiglu: pointers must be 16-byte aligned");
  if (n == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  k_swiglu_fwd<<<4 * sm_count(), 256, 0, st>>>(n / 8, static_cast<const __nv_bfloat16*>(gate),
                                                static_cast<const __nv_bfloat16*>(up), static_cast<__nv_bfloat16*>(act));
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_swiglu_fwd");
}

extern "C" lobra_status lobra_swiglu_bwd(int64_t n, const void* d, const void* gate, const void* up, void* d_gate,
                                         void* d_up, lobra_stream_t stream) {
  clear_error();
  if (n < 0 || n % 8 || !d || !gate || !up || !d_gate || !d_up)
    return fail(LOBRA_ERR_INPUT, "swiglu_bwd: n % 8 == 0 and non-null pointers");
  if (!al16(d) || !al16(gate) || !al16(up) || !al16(d_gate) || !al16(d_up))
    return fail(LOBRA_ERR_INPUT, "swiglu_bwd: pointers must be 16-byte aligned");
  if (n == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  k_swiglu_bwd<<<4 * sm_count(), 256, 0, st>>>(n / 8, static_cast<const __nv_bfloat16*>(d),
                                                static_cast<const __nv_bfloat16*>(gate),
                                                static_cast<const __nv_bfloat16*>(up),
                                                static_cast<__nv_bfloat16*>(d_gate), static_cast<__nv_bfloat16*>(d_up));
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_swiglu_bwd");
}

extern "C" lobra_status lobra_add(int64_t n, const void* A, const void* B, void* C, lobra_stream_t stream) {
  clear_error();
  if (n < 0 || n % 8 || !A || !B || !C) return fail(LOBRA_ERR_INPUT, "add: n % 8 == 0 and non-null pointers");
  if (!al16(A) || !al16(B) || !al16(C)) return fail(LOBRA_ERR_INPUT, "add: pointers must be 16-byte aligned");
  if (n == 0) return LOBRA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_LAYER, st, true);
  k_add<<<4 * sm_count(), 256, 0, st>>>(n / 8, static_cast<const __nv_bfloat16*>(A),
                                         static_cast<const __nv_bfloat16*>(B), static_cast<__nv_bfloat16*>(C));
  count_launch(LOBRA_K_LAYER, st, false);
  return done("lobra_add");
}
