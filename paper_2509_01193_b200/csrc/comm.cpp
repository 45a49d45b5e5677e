// NCCL plumbing: world communicator + per-replica TP sub-communicator
// (ncclCommSplit(color = replica id)), the TP all-reduces of Megatron tensor parallelism
// and the per-step adapter-gradient all-reduce across FT replicas (P:170,
// P:306).  NCCL is resolved at run time with dlopen so that the process uses the single
// libnccl.so.2 that torch already loaded (NCCL 2.28 in this image).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.h"
#include "nccl.h"

namespace lobra {
namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

Nccl g_nccl;
std::once_flag g_once;

void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
#define LOAD(f, name)                                                  \
  g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, name));     \
  if (!g_nccl.f) return;
  LOAD(GetUniqueId, "ncclGetUniqueId");
  LOAD(CommInitRank, "ncclCommInitRank");
  LOAD(CommSplit, "ncclCommSplit");
  LOAD(CommDestroy, "ncclCommDestroy");
  LOAD(CommCount, "ncclCommCount");
  LOAD(CommUserRank, "ncclCommUserRank");
  LOAD(AllReduce, "ncclAllReduce");
  LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
  g_nccl.ok = true;
}

// LOBRA_FORCE_COLLECTIVES=1 issues the NCCL calls even on 1-rank groups (tests exercise
// the collective path on a single GPU).
bool force_collectives() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_FORCE_COLLECTIVES");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

lobra_status need_nccl() {
  std::call_once(g_once, load_nccl);
  if (!g_nccl.ok) return fail(LOBRA_ERR_NCCL, "libnccl.so.2 could not be loaded (import torch first)");
  return LOBRA_OK;
}

lobra_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return LOBRA_OK;
  return fail(LOBRA_ERR_NCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
}

}  // namespace
}  // namespace lobra

struct lobra_comm_s {
  ncclComm_t world = nullptr;
  ncclComm_t tp = nullptr;
  int world_size = 0, rank = 0, tp_size = 0, tp_rank = 0;
  lobra_symm symm = nullptr;   // own peer-memory TP collectives (symm.cu), not owned
};

namespace lobra {
// symm.cu
template <typename T>
lobra_status symm_allreduce(lobra_symm s, const void* src, void* dst, size_t count, cudaStream_t st);
int symm_world(lobra_symm s);
int symm_rank(lobra_symm s);

void* symm_data(lobra_symm s);
size_t symm_capacity(lobra_symm s);
lobra_status comm_tp_allreduce_bf16(lobra_comm c, void* buf, size_t count, cudaStream_t st);

lobra_symm comm_symm(lobra_comm c) { return c ? c->symm : nullptr; }

// The symmetric data area of the comm's TP group when it can hold `bytes` (the projection
// GEMMs then write their partial straight into peer-visible memory), else nullptr.
void* comm_tp_stage(lobra_comm c, size_t bytes) {
  if (!c || !c->symm || symm_capacity(c->symm) < bytes) return nullptr;
  return symm_data(c->symm);
}

// dst = sum over the TP group of src (src may be the stage area); bf16.
lobra_status comm_tp_allreduce_bf16_to(lobra_comm c, const void* src, void* dst, size_t count, cudaStream_t st) {
  if (c && c->symm) return symm_allreduce<__nv_bfloat16>(c->symm, src, dst, count, st);
  if (src != dst && cudaMemcpyAsync(dst, src, count * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "TP staging copy failed");
  return comm_tp_allreduce_bf16(c, dst, count, st);
}

lobra_status comm_tp_allreduce_bf16(lobra_comm c, void* buf, size_t count, cudaStream_t st) {
  if (c && c->symm) return symm_allreduce<__nv_bfloat16>(c->symm, buf, buf, count, st);
  lobra_status s = need_nccl();
  if (s != LOBRA_OK) return s;
  if (!c || !c->tp) return fail(LOBRA_ERR_INPUT, "comm has no TP communicator");
  if (c->tp_size == 1 && !force_collectives()) return LOBRA_OK;
  return nccl_check(g_nccl.AllReduce(buf, buf, count, ncclBfloat16, ncclSum, c->tp, st),
                    "TP all-reduce");
}
lobra_status comm_tp_allreduce_f32(lobra_comm c, float* buf, size_t count, cudaStream_t st) {
  if (c && c->symm) return symm_allreduce<float>(c->symm, buf, buf, count, st);
  lobra_status s = need_nccl();
  if (s != LOBRA_OK) return s;
  if (!c || !c->tp) return fail(LOBRA_ERR_INPUT, "comm has no TP communicator");
  if (c->tp_size == 1 && !force_collectives()) return LOBRA_OK;
  return nccl_check(g_nccl.AllReduce(buf, buf, count, ncclFloat32, ncclSum, c->tp, st),
                    "TP all-reduce");
}
}  // namespace lobra

using namespace lobra;

extern "C" lobra_status lobra_nccl_unique_id(void* out128) {
  clear_error();
  if (!out128) return fail(LOBRA_ERR_INPUT, "null output");
  lobra_status s = need_nccl();
  if (s != LOBRA_OK) return s;
  ncclUniqueId id;
  if ((s = nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId")) != LOBRA_OK) return s;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return LOBRA_OK;
}

extern "C" lobra_status lobra_comm_init(const void* id128, int32_t world, int32_t rank,
                                        int32_t replica_id, lobra_comm* out) {
  clear_error();
  if (!id128 || !out || world < 1 || rank < 0 || rank >= world || replica_id < 0)
    return fail(LOBRA_ERR_INPUT, "bad comm_init arguments");
  lobra_status s = need_nccl();
  if (s != LOBRA_OK) return s;
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  lobra_comm c = new lobra_comm_s();
  c->world_size = world;
  c->rank = rank;
  if ((s = nccl_check(g_nccl.CommInitRank(&c->world, world, id, rank), "ncclCommInitRank")) != LOBRA_OK) {
    delete c;
    return s;
  }
  if ((s = nccl_check(g_nccl.CommSplit(c->world, replica_id, rank, &c->tp, nullptr), "ncclCommSplit")) !=
      LOBRA_OK) {
    g_nccl.CommDestroy(c->world);
    delete c;
    return s;
  }
  g_nccl.CommCount(c->tp, &c->tp_size);
  g_nccl.CommUserRank(c->tp, &c->tp_rank);
  *out = c;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_comm_from_symm(lobra_symm s, lobra_comm* out) {
  clear_error();
  if (!s || !out) return fail(LOBRA_ERR_INPUT, "null argument");
  lobra_comm c = new lobra_comm_s();
  c->symm = s;
  c->world_size = c->tp_size = symm_world(s);
  c->rank = c->tp_rank = symm_rank(s);
  *out = c;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_comm_attach_symm(lobra_comm c, lobra_symm s) {
  clear_error();
  if (!c) return fail(LOBRA_ERR_INPUT, "null comm");
  if (s && symm_world(s) != c->tp_size)
    return fail(LOBRA_ERR_INPUT, "symmetric group size %d != TP size %d", symm_world(s), c->tp_size);
  c->symm = s;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_comm_destroy(lobra_comm c) {
  clear_error();
  if (!c) return LOBRA_OK;
  if (g_nccl.ok) {
    if (c->tp) g_nccl.CommDestroy(c->tp);
    if (c->world) g_nccl.CommDestroy(c->world);
  }
  delete c;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_comm_tp_info(lobra_comm c, int32_t* tp_size, int32_t* tp_rank) {
  clear_error();
  if (!c || !tp_size || !tp_rank) return fail(LOBRA_ERR_INPUT, "null argument");
  *tp_size = c->tp_size;
  *tp_rank = c->tp_rank;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_adapter_allreduce(lobra_comm c, float* flat, size_t count,
                                                lobra_stream_t stream) {
  clear_error();
  if (c && !c->world && c->symm) {   // symmetric-group comm: the group is the world
    if (!flat && count) return fail(LOBRA_ERR_INPUT, "null buffer");
    if (c->world_size == 1 || count == 0) return LOBRA_OK;
    return symm_allreduce<float>(c->symm, flat, flat, count, reinterpret_cast<cudaStream_t>(stream));
  }
  if (!c || !c->world) return fail(LOBRA_ERR_INPUT, "null comm");
  if (!flat && count) return fail(LOBRA_ERR_INPUT, "null buffer");
  lobra_status s = need_nccl();
  if (s != LOBRA_OK) return s;
  if ((c->world_size == 1 && !force_collectives()) || count == 0) return LOBRA_OK;
  return nccl_check(g_nccl.AllReduce(flat, flat, count, ncclFloat32, ncclSum, c->world,
                                     reinterpret_cast<cudaStream_t>(stream)),
                    "adapter all-reduce");
}
