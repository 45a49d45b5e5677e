// Probe: NVLS multicast objects on this box (one process, one GPU).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_nvls tools/probe_nvls.cu -lcuda
// Creates a multicast object with one device, binds local physical memory, maps the
// multicast and unicast views and runs multimem.ld_reduce / multimem.st over it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    CUresult r_ = (x);                                                     \
    if (r_ != CUDA_SUCCESS) {                                              \
      const char* s_ = nullptr;                                            \
      cuGetErrorString(r_, &s_);                                           \
      printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");            \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void k_nvls(float* mc, float* uc, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + i) : "memory");
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(a * 2), "f"(b * 2),
               "f"(c * 2), "f"(d * 2) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mcs = -1, fab = -1;
  CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handle_supported=%d\n", mcs, fab);
  cudaSetDevice(0);
  cudaFree(0);
  const size_t n = 1 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, gran_rec = 0;
  mp.size = n * 4;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&gran_rec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("granularity min=%zu recommended=%zu\n", gran, gran_rec);
  const size_t bytes = ((n * 4 + gran_rec - 1) / gran_rec) * gran_rec;
  mp.size = bytes;
  for (int nd = 1; nd <= 2; ++nd)
    for (int ht = 0; ht < 3; ++ht)
      for (int big = 0; big < 2; ++big) {
        CUmulticastObjectProp q = {};
        q.numDevices = nd;
        q.handleTypes = ht == 0 ? (CUmemAllocationHandleType)0
                        : ht == 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_FABRIC;
        q.size = big ? bytes : gran;
        CUmemGenericAllocationHandle t;
        CUresult r = cuMulticastCreate(&t, &q);
        printf("create nd=%d ht=%d size=%zu -> %d\n", nd, ht, q.size, (int)r);
        if (r == CUDA_SUCCESS) cuMemRelease(t);
      }
  const size_t sz = ((n * 4 + gran - 1) / gran) * gran;
  mp.size = sz;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  CK(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("alloc granularity=%zu bytes=%zu\n", agran, sz);
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, sz, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, sz, 0));
  CUdeviceptr uc = 0, mva = 0;
  CK(cuMemAddressReserve(&uc, sz, gran, 0, 0));
  CK(cuMemMap(uc, sz, 0, phys, 0));
  CK(cuMemAddressReserve(&mva, sz, gran, 0, 0));
  CK(cuMemMap(mva, sz, 0, mc, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, sz, &acc, 1));
  CK(cuMemSetAccess(mva, sz, &acc, 1));
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
  cudaMemcpy((void*)uc, h.data(), n * 4, cudaMemcpyHostToDevice);
  k_nvls<<<(n / 4 + 255) / 256, 256>>>((float*)mva, (float*)uc, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> g(n);
  cudaMemcpy(g.data(), (void*)uc, n * 4, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += g[i] != h[i] * 2;
  printf("mismatches=%zu (of %zu)\n", bad, n);
  int fd = -1;
  CUresult ex = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  printf("export mc fd: rc=%d fd=%d\n", (int)ex, fd);
  printf("%s\n", bad == 0 && e == cudaSuccess ? "NVLS_OK" : "NVLS_FAIL");
  return 0;
}
