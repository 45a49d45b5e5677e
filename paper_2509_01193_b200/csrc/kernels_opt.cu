// Multi-tenant AdamW over the flat adapter parameter buffer.
// HBM-bound elementwise kernel: per element reads p, g, m, v (+ group id) and writes
// p, m, v (+ the bf16 operand copy); 16-byte vector accesses, grid = 4 x #SMs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "common.h"

namespace lobra {
// lora_host.cu
int64_t count_launch(int kind, cudaStream_t st, bool begin);

namespace {

constexpr int kMaxGroups = 64;

struct AdamArgs {
  float lr[kMaxGroups], b1[kMaxGroups], b2[kMaxGroups], eps[kMaxGroups], wd[kMaxGroups];
  float c1[kMaxGroups], c2[kMaxGroups];   // 1 / (1 - b^step)
  float grad_scale;
  int num_groups;
};

__device__ __forceinline__ float adam_one(float p, float g, float& m, float& v, int k,
                                          const AdamArgs& a) {
  if (k >= a.num_groups) return p;   // not an adapter element of any group: untouched
  g *= a.grad_scale;
  m = a.b1[k] * m + (1.0f - a.b1[k]) * g;
  v = a.b2[k] * v + (1.0f - a.b2[k]) * g * g;
  const float mh = m * a.c1[k];
  const float vh = v * a.c2[k];
  return p - a.lr[k] * (mh / (sqrtf(vh) + a.eps[k]) + a.wd[k] * p);
}

__global__ void k_adamw(float* __restrict__ p, __nv_bfloat16* __restrict__ pb,
                        const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                        const uint8_t* __restrict__ grp, long long n, const AdamArgs a) {
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 P = reinterpret_cast<const float4*>(p)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float4 M = reinterpret_cast<const float4*>(m)[i];
    float4 V = reinterpret_cast<const float4*>(v)[i];
    int k0 = 0, k1 = 0, k2 = 0, k3 = 0;
    if (grp) {
      const uchar4 q = reinterpret_cast<const uchar4*>(grp)[i];
      k0 = q.x, k1 = q.y, k2 = q.z, k3 = q.w;
    }
    P.x = adam_one(P.x, G.x, M.x, V.x, k0, a);
    P.y = adam_one(P.y, G.y, M.y, V.y, k1, a);
    P.z = adam_one(P.z, G.z, M.z, V.z, k2, a);
    P.w = adam_one(P.w, G.w, M.w, V.w, k3, a);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = M;
    reinterpret_cast<float4*>(v)[i] = V;
    if (pb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pb)[i] = o;
    }
  }
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int k = grp ? grp[i] : 0;
    float M = m[i], V = v[i];
    const float P = adam_one(p[i], g[i], M, V, k, a);
    p[i] = P, m[i] = M, v[i] = V;
    if (pb) pb[i] = __float2bfloat16_rn(P);
  }
}

bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

}  // namespace
}  // namespace lobra

using namespace lobra;

extern "C" lobra_status lobra_adamw_step(float* params, void* params_bf16, const float* grads,
                                         float* m, float* v, const uint8_t* group, size_t count,
                                         const lobra_adamw_hparams* hp, int32_t num_groups,
                                         int64_t step, float grad_scale, lobra_stream_t stream) {
  clear_error();
  if (!params || !grads || !m || !v || !hp) return fail(LOBRA_ERR_INPUT, "null argument");
  if (num_groups < 1 || num_groups > kMaxGroups)
    return fail(LOBRA_ERR_INPUT, "num_groups must be in [1, %d]", kMaxGroups);
  if (step < 1) return fail(LOBRA_ERR_INPUT, "step must be >= 1");
  if (!al16(params) || !al16(grads) || !al16(m) || !al16(v) || (params_bf16 && !al16(params_bf16)) ||
      (group && (reinterpret_cast<uintptr_t>(group) & 3)))
    return fail(LOBRA_ERR_INPUT, "device pointers must be 16-byte aligned (group 4-byte)");
  AdamArgs a;
  memset(&a, 0, sizeof(a));
  for (int k = 0; k < num_groups; ++k) {
    const lobra_adamw_hparams& h = hp[k];
    if (!(h.beta1 >= 0 && h.beta1 < 1 && h.beta2 >= 0 && h.beta2 < 1 && h.eps > 0))
      return fail(LOBRA_ERR_INPUT, "group %d: need 0 <= beta < 1 and eps > 0", k);
    a.lr[k] = h.lr, a.b1[k] = h.beta1, a.b2[k] = h.beta2, a.eps[k] = h.eps, a.wd[k] = h.weight_decay;
    const int64_t t = h.step > 0 ? h.step : step;
    if (h.step < 0) return fail(LOBRA_ERR_INPUT, "group %d: step must be >= 0", k);
    a.c1[k] = (float)(1.0 / (1.0 - std::pow((double)h.beta1, (double)t)));
    a.c2[k] = (float)(1.0 / (1.0 - std::pow((double)h.beta2, (double)t)));
  }
  a.grad_scale = grad_scale;
  a.num_groups = num_groups;
  if (count == 0) return LOBRA_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  count_launch(LOBRA_K_OPT, st, true);
  k_adamw<<<4 * sms, 256, 0, st>>>(params, static_cast<__nv_bfloat16*>(params_bf16), grads, m, v,
                                   group, (long long)count, a);
  count_launch(LOBRA_K_OPT, st, false);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "lobra_adamw_step: %s", cudaGetErrorString(e));
  return LOBRA_OK;
}
