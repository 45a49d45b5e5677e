// Host side of lobra_lora_fwd / lobra_lora_bwd: argument validation, batch metadata
// (segments, per-tile adapter slots, reduction units), workspace layout, TMA tensor maps,
// and the launch sequence.  See include/lobra.h for the contract.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "lora_internal.h"

namespace lobra {

// ------------------------------------------------------------------ errors / version
static thread_local std::string g_err;
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
void clear_error() { g_err.clear(); }

// comm.cpp
lobra_status comm_tp_allreduce_bf16(lobra_comm c, void* buf, size_t count, cudaStream_t st);
lobra_status comm_tp_allreduce_f32(lobra_comm c, float* buf, size_t count, cudaStream_t st);
void* comm_tp_stage(lobra_comm c, size_t bytes);
lobra_symm comm_symm(lobra_comm c);
bool symm_scatter_target(lobra_symm s, long long T, long long N, TpScatter* out);
lobra_status symm_scatter_finish(lobra_symm s, long long T, long long N, void* dst, cudaStream_t st);

// LOBRA_TP_FUSED=0: row-parallel GEMM writes its partial locally and the own all-reduce
// follows (A/B of the fused reduce-scatter epilogue)
bool tp_fused() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_TP_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
lobra_status comm_tp_allreduce_bf16_to(lobra_comm c, const void* src, void* dst, size_t count, cudaStream_t st);

// ------------------------------------------------------------------ tracing
namespace {
std::atomic<int64_t> g_launches{0};
std::mutex g_prof_mu;
bool g_prof_on = false;
struct ProfRec {
  int kind;
  cudaEvent_t e0, e1;
};
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;
int64_t g_prof_count[LOBRA_K_NUM] = {0};
double g_prof_ms[LOBRA_K_NUM] = {0};

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one kernel launch: counts it and, while tracing is enabled, records events
// on the launching stream around it.
struct Prof {
  int kind;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  Prof(int k, cudaStream_t s) : kind(k), st(s) {
    // launches are counted where they happen (note_launch: launch_k and the fp32 launchers),
    // so a launcher that enqueues two kernels (dY pass + G finalize) counts two
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (g_prof_on) {
      e0 = prof_event();
      cudaEventRecord(e0, st);
    }
  }
  ~Prof() {
    if (!e0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e1 = prof_event();
    cudaEventRecord(e1, st);
    g_prof_recs.push_back({kind, e0, e1});
  }
};
}  // namespace

// One kernel launch of the library (called by every launcher right after it enqueues).
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Launch accounting for kernels outside this file (begin/end bracket one launch).
int64_t count_launch(int kind, cudaStream_t st, bool begin) {
  static thread_local cudaEvent_t e0 = nullptr;
  if (begin) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    e0 = nullptr;
    if (g_prof_on) {
      e0 = prof_event();
      cudaEventRecord(e0, st);
    }
  } else if (e0) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e1 = prof_event();
    cudaEventRecord(e1, st);
    g_prof_recs.push_back({kind, e0, e1});
    e0 = nullptr;
  }
  return g_launches.load();
}

// ------------------------------------------------------------------ per-device context
namespace {

constexpr int kRing = 64;   // metadata uploads in flight before a slot is reused (a host wait)

struct DevCtx {
  int dev = -1, num_sms = 0, cc_major = 0, cc_minor = 0;
  std::vector<uint8_t*> pinned;
  std::vector<size_t> pinned_bytes;
  std::vector<cudaEvent_t> ev;
  int next = 0;
  std::mutex mu;
};

std::mutex g_ctx_mu;
std::vector<DevCtx*> g_ctx;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

lobra_status get_ctx(DevCtx** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(LOBRA_ERR_CUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
  if (!g_ctx[dev]) {
    DevCtx* c = new DevCtx();
    c->dev = dev;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    c->pinned.assign(kRing, nullptr);
    c->pinned_bytes.assign(kRing, 0);
    c->ev.assign(kRing, nullptr);
    for (int i = 0; i < kRing; ++i)
      if (cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(LOBRA_ERR_CUDA, "cudaEventCreate failed");
    g_ctx[dev] = c;
  }
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(LOBRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  *out = g_ctx[dev];
  if (g_ctx[dev]->cc_major != 10 || g_ctx[dev]->cc_minor != 0)
    return fail(LOBRA_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                dev, g_ctx[dev]->cc_major, g_ctx[dev]->cc_minor);
  return LOBRA_OK;
}

// The metadata reaches the device through a KERNEL that reads the pinned staging buffer over
// PCIe (UVA: cudaMallocHost memory is mapped), not through cudaMemcpyAsync: a copy-engine
// transfer queues behind whatever else the copy engines carry, so while a caller streams the
// next micro-batch's activations host -> device (bench.py's e2e leg: 8.6 GB per C3 step) each
// call's few-KB metadata copy waited for them and the compute serialised with the copies.
__global__ void k_meta_copy(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int n4) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int n16 = n4 >> 2;   // 16-byte words, then the 4-byte tail
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  const int t = (n16 << 2) + blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n4) dst[t] = src[t];
}

// Copies `bytes` of host data to device `dst` on `st` through a pinned staging ring.
lobra_status upload(DevCtx* c, const void* src, size_t bytes, void* dst, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(c->mu);
  const int k = c->next;
  c->next = (k + 1) % kRing;
  if (cudaEventSynchronize(c->ev[k]) != cudaSuccess) return fail(LOBRA_ERR_CUDA, "event sync");
  if (c->pinned_bytes[k] < bytes) {
    if (c->pinned[k]) cudaFreeHost(c->pinned[k]);
    size_t sz = std::max<size_t>(bytes, 1 << 16);
    if (cudaMallocHost(reinterpret_cast<void**>(&c->pinned[k]), sz) != cudaSuccess)
      return fail(LOBRA_ERR_CUDA, "cudaMallocHost(%zu) failed", sz);
    c->pinned_bytes[k] = sz;
  }
  std::memcpy(c->pinned[k], src, bytes);
  static const bool memcpy_path = getenv("LOBRA_META_MEMCPY") != nullptr;   // A/B switch
  if (!memcpy_path && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && bytes % 4 == 0) {   // read over PCIe
    const int n4 = (int)(bytes / 4);
    const int grid = std::max(1, std::min(64, (n4 / 4 + 255) / 256));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_meta_copy, static_cast<const uint32_t*>(static_cast<const void*>(c->pinned[k])),
                           static_cast<uint32_t*>(dst), n4) != cudaSuccess)
      return fail(LOBRA_ERR_CUDA, "metadata copy kernel launch failed");
    note_launch();
  } else if (cudaMemcpyAsync(dst, c->pinned[k], bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    return fail(LOBRA_ERR_CUDA, "cudaMemcpyAsync H2D failed");
  }
  if (cudaEventRecord(c->ev[k], st) != cudaSuccess) return fail(LOBRA_ERR_CUDA, "event record");
  return LOBRA_OK;
}

// Metadata upload with an optional cache (LOBRA_META_CACHE=1, probe builds only): skip the
// H2D copy when this device address already holds byte-identical metadata.  Not in the
// product library: the cache keys on the address, so a reused workspace could go stale.
bool meta_cache_on() {
#ifdef LOBRA_PROBES
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_META_CACHE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
#else
  return false;
#endif
}
std::mutex g_meta_mu;
std::vector<std::pair<const void*, uint64_t>> g_meta_cache;

lobra_status upload_meta(DevCtx* c, const std::vector<int32_t>& buf, void* dst, cudaStream_t st) {
  if (meta_cache_on()) {
    uint64_t h = 1469598103934665603ULL;
    for (int32_t v : buf) h = (h ^ (uint32_t)v) * 1099511628211ULL;
    h ^= buf.size();
    std::lock_guard<std::mutex> lk(g_meta_mu);
    for (auto& e : g_meta_cache)
      if (e.first == dst) {
        if (e.second == h) return LOBRA_OK;
        e.second = h;
        return upload(c, buf.data(), buf.size() * 4, dst, st);
      }
    g_meta_cache.emplace_back(dst, h);
  }
  return upload(c, buf.data(), buf.size() * 4, dst, st);
}

// ------------------------------------------------------------------ batch plan
struct Plan {
  int T = 0, ntasks = 0, rsum = 0;
  std::vector<int32_t> buf;  // serialized int32 metadata (floats bit-cast)
  // offsets (in int32 words) of each array inside buf
  int o_seg_off, o_seg_task, o_tile_slot_off, o_slot_task, o_slot_tile, o_task_slot_off,
      o_task_slots, o_unit_task, o_unit_s0, o_unit_s1, o_task_unit_off, o_ranks, o_roff, o_boff,
      
      o_scales, o_ranks_g, o_roff_g;
  int np = 1;       // projections sharing the slots (projection group)
  int ld8 = 0;      // row stride of the B operand the kernels read (rsum if direct)
  bool bdirect = true;
  int nseg = 0, ntiles = 0, nslots = 0, nunits = 0, max_slots = 0, qp = 16, ndyunits = 0;
  // fused dY pass schedules, one per distinct output width (a projection group's k/v can be
  // narrower than q): CTAs of the static schedule, 512-column chunks, segment arrays
  struct DySet {
    int width = 0, ncta = 1, nch = 1, nseg = 0;
    int o_task = 0, o_s0 = 0, o_s1 = 0, o_off = 0, o_chunk = 0, o_cta = 0;
  };
  std::vector<DySet> dy;
  std::vector<DySet> sr;   // k_segred schedules (128-column chunks), per reduction width
  int nsrseg = 0;          // max segments over sr
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

lobra_status validate(const lobra_problem* prob, const lobra_batch* b, const lobra_adapters* ad) {
  if (!prob || !b || !ad) return fail(LOBRA_ERR_INPUT, "null problem/batch/adapters");
  if (prob->dtype != LOBRA_BF16 && prob->dtype != LOBRA_FP32)
    return fail(LOBRA_ERR_INPUT, "unknown dtype %d", (int)prob->dtype);
  if (prob->in < 1 || prob->out < 1) return fail(LOBRA_ERR_INPUT, "in/out must be positive");
  if (prob->dtype == LOBRA_BF16 && (prob->in % 64 || prob->out % 64))
    return fail(LOBRA_ERR_INPUT, "bf16 path needs in and out multiples of 64 (got %lld, %lld)",
                (long long)prob->in, (long long)prob->out);
  if (prob->in > (1 << 30) || prob->out > (1 << 30)) return fail(LOBRA_ERR_INPUT, "in/out too large");
  if (prob->tp_kind != LOBRA_TP_NONE && prob->tp_kind != LOBRA_TP_COLUMN &&
      prob->tp_kind != LOBRA_TP_ROW)
    return fail(LOBRA_ERR_INPUT, "unknown tp_kind");
  if (prob->dA_ld != 0 && prob->dA_ld < prob->in) return fail(LOBRA_ERR_INPUT, "dA_ld < in");
  if (b->num_seqs < 1 || !b->seq_lens || !b->seq_task)
    return fail(LOBRA_ERR_INPUT, "batch needs num_seqs >= 1 and host seq_lens/seq_task");
  if (ad->num_tasks < 1 || !ad->ranks || !ad->scales)
    return fail(LOBRA_ERR_INPUT, "adapters need num_tasks >= 1 and host ranks/scales");
  if (!ad->A || !ad->B) return fail(LOBRA_ERR_INPUT, "adapter A/B device pointers missing");
  for (int t = 0; t < ad->num_tasks; ++t)
    if (ad->ranks[t] < 1 || ad->ranks[t] > 64)
      return fail(LOBRA_ERR_INPUT, "task %d rank %d outside [1, 64]", t, ad->ranks[t]);
  long long T = 0;
  for (int k = 0; k < b->num_seqs; ++k) {
    if (b->seq_lens[k] < 0) return fail(LOBRA_ERR_INPUT, "sequence %d has negative length", k);
    if (b->seq_task[k] < 0 || b->seq_task[k] >= ad->num_tasks)
      return fail(LOBRA_ERR_INPUT, "sequence %d task id %d out of range [0, %d)", k,
                  b->seq_task[k], ad->num_tasks);
    T += b->seq_lens[k];
  }
  if (T > (1LL << 30)) return fail(LOBRA_ERR_INPUT, "too many tokens");
  return LOBRA_OK;
}

void build_plan(const lobra_batch* b, const lobra_adapters* ad, int width_hint, int dy_width,
                int num_sms, Plan& P, int np = 1, const std::vector<int>& dy_widths = {},
                const std::vector<int>& sr_widths = {}) {
  const int n = b->num_seqs, G = ad->num_tasks;
  P.ntasks = G;
  P.np = np;
  std::vector<int> seg_off{0}, seg_task;
  int T = 0;
  for (int k = 0; k < n; ++k) {
    const int L = b->seq_lens[k], t = b->seq_task[k];
    if (L == 0) continue;
    if (!seg_task.empty() && seg_task.back() == t) {
      seg_off.back() += L;
    } else {
      seg_task.push_back(t);
      seg_off.push_back(seg_off.back() + L);
    }
    T += L;
  }
  P.T = T;
  P.nseg = (int)seg_task.size();
  P.ntiles = (T + kTileM - 1) / kTileM;
  // slots: per tile, tasks in order of first appearance
  std::vector<int> tile_slot_off{0}, slot_task, slot_tile;
  int sg = 0;
  for (int m = 0; m < P.ntiles; ++m) {
    const int r0 = m * kTileM, r1 = std::min(T, r0 + kTileM);
    while (seg_off[sg + 1] <= r0) ++sg;
    std::vector<int> seen;
    for (int s = sg; s < P.nseg && seg_off[s] < r1; ++s)
      if (std::find(seen.begin(), seen.end(), seg_task[s]) == seen.end()) seen.push_back(seg_task[s]);
    for (int t : seen) slot_task.push_back(t), slot_tile.push_back(m);
    tile_slot_off.push_back((int)slot_task.size());
    P.max_slots = std::max(P.max_slots, (int)seen.size());
  }
  P.nslots = (int)slot_task.size();
  std::vector<int> task_slot_off(G + 1, 0), task_slots;
  for (int t = 0; t < G; ++t) {
    for (int s = 0; s < P.nslots; ++s)
      if (slot_task[s] == t) task_slots.push_back(s);
    task_slot_off[t + 1] = (int)task_slots.size();
  }
  // reduction units: each task's slot list split into near-equal contiguous ranges so
  // that units x chunks ~ 4 items per SM of equal cost (balanced persistent schedule)
  const int nchunks = std::max(1, (width_hint + 127) / 128);
  const double target = 4.0 * std::max(num_sms, 1);
  const double per = std::max(1.0, (double)P.nslots * nchunks / target);
  std::vector<int> unit_task, unit_s0, unit_s1, task_unit_off(G + 1, 0);
  for (int t = 0; t < G; ++t) {
    const int n_t = task_slot_off[t + 1] - task_slot_off[t];
    const int nu = n_t ? std::max(1, (int)std::lround(n_t / per)) : 0;
    for (int u = 0; u < nu; ++u) {
      unit_task.push_back(t);
      unit_s0.push_back(task_slot_off[t] + (int)((long long)n_t * u / nu));
      unit_s1.push_back(task_slot_off[t] + (int)((long long)n_t * (u + 1) / nu));
    }
    task_unit_off[t + 1] = (int)unit_task.size();
  }
  P.nunits = (int)unit_task.size();
  // segments of the fused dY pass: the (task, 512-column chunk, slot) entries in that order
  // are cut into one contiguous range of equal length per CTA (a static balanced schedule:
  // every entry streams one 128 x 512 dY block), and each range into segments of equal
  // (task, chunk) -- a segment accumulates its dB chunk over its slots in TMEM and writes one
  // partial; the segments of one (task, chunk) are consecutive (k_finalize_multi sums them in order).
  // The schedule depends only on (batch, width), so a projection group reduces in exactly the
  // order of the single-projection calls.
  struct DyVecs {
    std::vector<int> task, s0, s1, chunk, off, cta_off{0};
    int ncta = 1, nch = 1;
  };
  // weighted = true (the dY pass): an entry's weight is its measured cost, 5 per 128-column
  // dY sub-block + 10 fixed (the H ring load and the 128-row G partial written per entry) +
  // 7 for a task of rank > 32 (wider B_t / H boxes, G and dB partials).  Least-squares fit of
  // per-CTA times against each CTA's entries (LOBRA_TRACE_DY, tools/trace_dy.py, C3): full
  // entries 3.0 us, rank > 32 3.65, the 256-column last chunk of width 11008 2.0 / 2.7, plus
  // 1.5 per segment (each (task, chunk) run is charged one).  With equal entry counts per CTA the CTA times spread 179-343 us
  // (11008) and 89-123 us (4096).
  auto build_dy = [&](int width, int chunk_cols, bool weighted) {
    DyVecs v;
    const int nch = std::max(1, (width + chunk_cols - 1) / chunk_cols);
    const int n128 = (width + 127) / 128;
    auto weight = [&](int t, int c) -> long long {
      if (!weighted) return 1;
      const int nb = std::max(0, std::min(chunk_cols / 128, n128 - c * (chunk_cols / 128)));
      return 5LL * nb + 10 + (ad->ranks[t] > 32 ? 7 : 0);
    };
    // each (task, chunk) run also costs one segment (a dB drain: ~1.5 us, weight 15)
    const long long seg_w = weighted ? 15 : 0;
    long long W = 0, nent = 0;
    for (int t = 0; t < G; ++t)
      for (int c = 0; c < nch; ++c) {
        const long long n_t = task_slot_off[t + 1] - task_slot_off[t];
        W += n_t * weight(t, c) + (n_t ? seg_w : 0);
        nent += n_t;
      }
    const int ncta = (int)std::max<long long>(1, std::min<long long>(std::max(num_sms, 1), nent));
    v.off.assign((size_t)G * nch + 1, 0);
    long long e = 0;   // cumulative weight of the entries in (task, chunk, slot) order
    int cta = 0;
    auto cta_end = [&](int c) { return (long long)W * (c + 1) / ncta; };
    for (int t = 0; t < G; ++t) {
      const int k0 = task_slot_off[t], k1 = task_slot_off[t + 1];
      for (int c = 0; c < nch; ++c) {
        const long long w = std::max<long long>(1, weight(t, c));
        if (k1 > k0) e += seg_w;
        int k = k0;
        while (k < k1) {
          while (cta < ncta - 1 && e >= cta_end(cta)) {
            v.cta_off.push_back((int)v.task.size());
            ++cta;
          }
          const long long room = cta == ncta - 1 ? (long long)(k1 - k) * w : cta_end(cta) - e;
          const int take = (int)std::min<long long>(k1 - k, std::max<long long>(1, (room + w - 1) / w));
          v.task.push_back(t), v.chunk.push_back(c);
          v.s0.push_back(k), v.s1.push_back(k + take);
          k += take, e += take * w;
        }
        v.off[(size_t)t * nch + c + 1] = (int)v.task.size();
      }
    }
    while ((int)v.cta_off.size() < ncta + 1) v.cta_off.push_back((int)v.task.size());
    v.ncta = ncta;
    v.nch = nch;
    return v;
  };
  // the same static balanced schedule for the token reduction k_segred (128-column chunks),
  // for the dA width and (unfused dY pass) the dB width
  std::vector<DyVecs> srv;
  P.sr.clear();
  P.nsrseg = 0;
  for (int wdt : sr_widths.empty() ? std::vector<int>{width_hint, dy_width} : sr_widths) {
    bool seen = false;
    for (const auto& d : P.sr) seen = seen || d.width == wdt;
    if (seen || wdt <= 0) continue;
    srv.push_back(build_dy(wdt, 128, false));
    Plan::DySet ds;
    ds.width = wdt;
    ds.ncta = srv.back().ncta;
    ds.nch = srv.back().nch;
    ds.nseg = (int)srv.back().task.size();
    P.nsrseg = std::max(P.nsrseg, ds.nseg);
    P.sr.push_back(ds);
  }
  std::vector<int> widths = dy_widths;
  if (widths.empty()) widths.push_back(dy_width);
  std::vector<DyVecs> dyv;
  P.dy.clear();
  P.ndyunits = 0;
  for (int wdt : widths) {
    bool seen = false;
    for (const auto& d : P.dy) seen = seen || d.width == wdt;
    if (seen) continue;
    dyv.push_back(build_dy(wdt, 512, true));
    Plan::DySet ds;
    ds.width = wdt;
    ds.ncta = dyv.back().ncta;
    ds.nch = dyv.back().nch;
    ds.nseg = (int)dyv.back().task.size();
    P.ndyunits = std::max(P.ndyunits, ds.nseg);
    P.dy.push_back(ds);
  }
  std::vector<int> roff(G + 1, 0);
  for (int t = 0; t < G; ++t) roff[t + 1] = roff[t] + ad->ranks[t];
  P.rsum = roff[G];
  P.qp = 16;
  for (int t = 0; t < G; ++t) P.qp = std::max(P.qp, (ad->ranks[t] + 15) & ~15);
  // serialize
  P.buf.clear();
  auto put = [&](const std::vector<int>& v) {
    const int o = (int)P.buf.size();
    P.buf.insert(P.buf.end(), v.begin(), v.end());
    while (P.buf.size() % 4) P.buf.push_back(0);   // 16-byte alignment of every array
    return o;
  };
  P.o_seg_off = put(seg_off);
  P.o_seg_task = put(seg_task);
  P.o_tile_slot_off = put(tile_slot_off);
  P.o_slot_task = put(slot_task);
  P.o_slot_tile = put(slot_tile);
  P.o_task_slot_off = put(task_slot_off);
  P.o_task_slots = put(task_slots);
  P.o_unit_task = put(unit_task);
  P.o_unit_s0 = put(unit_s0);
  P.o_unit_s1 = put(unit_s1);
  P.o_task_unit_off = put(task_unit_off);
  for (size_t i = 0; i < P.sr.size(); ++i) {
    P.sr[i].o_task = put(srv[i].task);
    P.sr[i].o_s0 = put(srv[i].s0);
    P.sr[i].o_s1 = put(srv[i].s1);
    P.sr[i].o_off = put(srv[i].off);
    P.sr[i].o_chunk = put(srv[i].chunk);
    P.sr[i].o_cta = put(srv[i].cta_off);
  }
  for (size_t i = 0; i < P.dy.size(); ++i) {
    P.dy[i].o_task = put(dyv[i].task);
    P.dy[i].o_s0 = put(dyv[i].s0);
    P.dy[i].o_s1 = put(dyv[i].s1);
    P.dy[i].o_off = put(dyv[i].off);
    P.dy[i].o_chunk = put(dyv[i].chunk);
    P.dy[i].o_cta = put(dyv[i].cta_off);
  }
  P.o_ranks = put(std::vector<int>(ad->ranks, ad->ranks + G));
  P.o_roff = put(roff);
  std::vector<int> boff(G + 1, 0);
  P.bdirect = true;
  for (int t = 0; t < G; ++t) P.bdirect &= (ad->ranks[t] % 8) == 0;
  for (int t = 0; t < G; ++t) boff[t + 1] = boff[t] + (P.bdirect ? ad->ranks[t] : (ad->ranks[t] + 7) & ~7);
  P.ld8 = boff[G];
  P.o_boff = put(boff);
  std::vector<int> sc(G);
  std::memcpy(sc.data(), ad->scales, sizeof(float) * G);
  P.o_scales = put(sc);
  // projection group: the packed A_grp holds np bands of qp rows per task
  std::vector<int> rg(G, np * P.qp), rog(G + 1, 0);
  for (int t = 0; t < G; ++t) rog[t + 1] = rog[t] + np * P.qp;
  P.o_ranks_g = put(rg);
  P.o_roff_g = put(rog);
}

// point the fused dY pass fields of `m` at the schedule built for output width `width`
void set_dy(Meta& m, const Plan& P, const void* dev_base, int width) {
  const int32_t* d = reinterpret_cast<const int32_t*>(dev_base);
  const Plan::DySet* ds = P.dy.empty() ? nullptr : &P.dy[0];
  for (const auto& x : P.dy)
    if (x.width == width) ds = &x;
  if (!ds) {
    m.ndycta = 0, m.dy_nch = 1, m.ndyunits = 0;
    return;
  }
  m.ndyunits = ds->nseg;
  m.ndycta = ds->ncta;
  m.dy_nch = ds->nch;
  m.dy_unit_task = d + ds->o_task;
  m.dy_unit_s0 = d + ds->o_s0;
  m.dy_unit_s1 = d + ds->o_s1;
  m.dy_task_unit_off = d + ds->o_off;
  m.dy_unit_chunk = d + ds->o_chunk;
  m.dy_cta_off = d + ds->o_cta;
}

// point the token-reduction (k_segred) schedule fields of `m` at the one built for `width`
void set_sr(Meta& m, const Plan& P, const void* dev_base, int width) {
  const int32_t* d = reinterpret_cast<const int32_t*>(dev_base);
  const Plan::DySet* ds = nullptr;
  for (const auto& x : P.sr)
    if (x.width == width) ds = &x;
  if (!ds) {
    m.nsrcta = 0, m.sr_nch = 1, m.nsrseg = 0;
    return;
  }
  m.nsrseg = ds->nseg;
  m.nsrcta = ds->ncta;
  m.sr_nch = ds->nch;
  m.sr_task = d + ds->o_task;
  m.sr_s0 = d + ds->o_s0;
  m.sr_s1 = d + ds->o_s1;
  m.sr_tc_off = d + ds->o_off;
  m.sr_chunk = d + ds->o_chunk;
  m.sr_cta_off = d + ds->o_cta;
}

Meta device_meta(const Plan& P, const void* dev_base) {
  const int32_t* d = reinterpret_cast<const int32_t*>(dev_base);
  Meta m;
  m.T = P.T;
  m.nseg = P.nseg;
  m.ntiles = P.ntiles;
  m.nslots = P.nslots;
  m.ntasks = P.ntasks;
  m.nunits = P.nunits;
  m.rsum = P.rsum;
  m.max_slots_per_tile = P.max_slots;
  m.qp = P.qp;
  m.seg_off = d + P.o_seg_off;
  m.seg_task = d + P.o_seg_task;
  m.tile_slot_off = d + P.o_tile_slot_off;
  m.slot_task = d + P.o_slot_task;
  m.slot_tile = d + P.o_slot_tile;
  m.task_slot_off = d + P.o_task_slot_off;
  m.task_slots = d + P.o_task_slots;
  m.unit_task = d + P.o_unit_task;
  m.unit_s0 = d + P.o_unit_s0;
  m.unit_s1 = d + P.o_unit_s1;
  m.task_unit_off = d + P.o_task_unit_off;
  m.ndyunits = P.ndyunits;
  m.use_dy_units = 0;
  set_dy(m, P, dev_base, P.dy.empty() ? 0 : P.dy[0].width);
  set_sr(m, P, dev_base, P.sr.empty() ? 0 : P.sr[0].width);
  m.ranks = d + P.o_ranks;
  m.roff = d + P.o_roff;
  m.boff = d + P.o_boff;
  m.scales = reinterpret_cast<const float*>(d + P.o_scales);
  m.band = 0;
  return m;
}

// The shrink / dA view of a projection group: every task has np * qp "rows" (the bands) at
// roff_g in the packed A_grp, partial stride np * qp.
Meta group_meta(const Plan& P, const void* dev_base) {
  Meta m = device_meta(P, dev_base);
  const int32_t* d = reinterpret_cast<const int32_t*>(dev_base);
  m.ranks = d + P.o_ranks_g;
  m.roff = d + P.o_roff_g;
  m.rsum = P.ntasks * P.np * P.qp;
  m.qp = P.np * P.qp;
  return m;
}

// Workspace layout (bytes from ws base); both directions share it.
struct Layout {
  size_t meta = 0, bpad = 0, bt = 0, gslots = 0, rpart = 0, counters = 0, partA = 0, partB = 0,
         gpart = 0, total = 0;
  size_t saved = 0;
  size_t partB_stride = 0;   // floats between a group's per-projection dB partial regions
  int ld8 = 0;   // row stride (elements) of the B operand the kernels read
};

Layout layout(const lobra_problem* prob, const Plan& P) {
  Layout L;
  const size_t in = prob->in, out = prob->out;
  size_t off = 0;
  L.meta = off;
  off += align256(P.buf.size() * 4);
  if (prob->dtype == LOBRA_BF16) {
    const size_t es = 2;
    L.ld8 = P.ld8;
    L.bpad = off;
    if (!P.bdirect) off += align256(out * L.ld8 * es);
    L.bt = off;       // B^T [rsum, out]: only the opt-in LDGSTS projection (LOBRA_RP_LD=1) reads it
    if (rowproj_uses_ld()) off += align256((size_t)P.rsum * out * es);
    L.gslots = off;   // + one all-zero slot (index nslots)
    off += align256((size_t)(P.nslots + 1) * kTileM * kSlotW * es);
    const int sp = std::max(rowproj_splits(P.ntiles, (int)in), rowproj_splits(P.ntiles, (int)out));
    L.rpart = off;
    if (sp > 1) off += align256((size_t)sp * P.nslots * kTileM * 64 * 4);
    L.counters = off;
    off += align256((size_t)P.ntiles * 4);
    const size_t chA = (in + 127) / 128, chB = (out + 127) / 128;
    L.partA = off;
    off += align256(std::max((size_t)P.nunits * chA, (size_t)P.nsrseg) * P.qp * 128 * 4);
    L.partB = off;
    // unfused: [nunits][chB][qp][128]; fused dY pass: [ndyunits (segments)][4][qp][128]
    off += align256(std::max({(size_t)P.nunits * chB, (size_t)P.ndyunits * 4, (size_t)P.nsrseg}) * P.qp * 128 * 4);
    L.gpart = off;    // fused dY pass: G partials [nslots][ceil(out/512)][128][qp]
    off += align256((size_t)P.nslots * ((out + 511) / 512) * kTileM * P.qp * 4);
    L.saved = (size_t)(P.nslots + 1) * kTileM * kSlotW * es;
  } else {
    L.gslots = off;
    off += align256((size_t)P.T * kSlotW * 4);
    L.saved = (size_t)P.T * kSlotW * 4;
  }
  L.total = off;
  return L;
}

lobra_status make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                      uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 128, bool f32 = false) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  static int promo = -1;   // LOBRA_L2PROMO: 0 none, 1 64B, 2 128B, 3 256B (default)
  if (promo < 0) {
    const char* e = getenv("LOBRA_L2PROMO");
    promo = e ? atoi(e) : 3;
    if (promo < 0 || promo > 3) promo = 3;
  }
  const CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  CUresult r = g_encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                        : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        pr[promo], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(LOBRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) dims=%llu x %llu box=%u x %u",
                (int)r, (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer);
  return LOBRA_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

lobra_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LOBRA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return LOBRA_OK;
}

bool dy_fused() {   // LOBRA_DY_UNFUSED=1: separate G projection + dB reduction (two dY reads)
  const char* e = getenv("LOBRA_DY_UNFUSED");
  return !(e && e[0] == '1');
}

int sms_hint() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
    return n;
  cudaGetLastError();
  return 148;   // B200
}

// Width the token-reduction units are balanced for: with the fused dY pass they only serve
// the dA reduction (over `in`); the two-pass backward also reduces dB (over `out`) with them.
int unit_width(const lobra_problem* prob) {
  if (!prob) return 1;
  return (int)(dy_fused() ? prob->in : std::min(prob->in, prob->out));
}

lobra_status prepare(const lobra_problem* prob, const lobra_batch* b, const lobra_adapters* ad,
                     int width_hint, int num_sms, Plan& P, Layout& L) {
  lobra_status st = validate(prob, b, ad);
  if (st != LOBRA_OK) return st;
  build_plan(b, ad, width_hint, (int)prob->out, num_sms, P, 1, {}, {(int)prob->in, (int)prob->out});
  L = layout(prob, P);
  return LOBRA_OK;
}

}  // namespace
}  // namespace lobra

using namespace lobra;

namespace lobra {
// TMA map for other translation units (attn.cu): bf16 2D [outer, inner] row-major, 128-byte
// swizzle; initialises the driver entry point on first use.
lobra_status upload_host_meta(const void* src, size_t bytes, void* dst, cudaStream_t st) {
  DevCtx* ctx = nullptr;
  lobra_status s = get_ctx(&ctx);
  if (s != LOBRA_OK) return s;
  return upload(ctx, src, bytes, dst, st);
}
lobra_status make_tensor_map_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                                uint32_t box_inner, uint32_t box_outer) {
  DevCtx* ctx = nullptr;
  lobra_status s = get_ctx(&ctx);
  if (s != LOBRA_OK) return s;
  return make_map(map, ptr, inner, outer, box_inner, box_outer);
}
}  // namespace lobra

extern "C" const char* lobra_last_error(void) { return lobra::g_err.c_str(); }
extern "C" const char* lobra_version(void) { return "lobra-b200 0.1 (sm_100a, tcgen05/TMEM/TMA)"; }

extern "C" size_t lobra_lora_workspace_bytes(const lobra_problem* prob, const lobra_batch* batch,
                                             const lobra_adapters* ad) {
  clear_error();
  Plan P;
  Layout L;
  // the reduction-unit split depends on the SM count of the current device
  if (prepare(prob, batch, ad, unit_width(prob),
              sms_hint(), P, L) != LOBRA_OK)
    return 0;
  return L.total;
}

extern "C" size_t lobra_lora_saved_bytes(const lobra_problem* prob, const lobra_batch* batch,
                                         const lobra_adapters* ad) {
  clear_error();
  Plan P;
  Layout L;
  if (prepare(prob, batch, ad, 128, 1 << 20, P, L) != LOBRA_OK) return 0;
  return std::max<size_t>(L.saved, 256);
}

namespace lobra {
namespace {
// skip_shrink: Hs already holds this projection's H_s slots (a wide projection group computed
// every projection's H_s in one pass over X, lobra_lora_group_fwd)
lobra_status lora_fwd_impl(const lobra_problem* prob, const lobra_batch* batch,
                           const lobra_adapters* ad, const void* X, const void* W, void* Y, void* Hs,
                           void* ws, size_t ws_bytes, lobra_stream_t stream_, bool skip_shrink);
}  // namespace
}  // namespace lobra

extern "C" lobra_status lobra_lora_fwd(const lobra_problem* prob, const lobra_batch* batch,
                                       const lobra_adapters* ad, const void* X, const void* W,
                                       void* Y, void* Hs, void* ws, size_t ws_bytes,
                                       lobra_stream_t stream_) {
  clear_error();
  return lora_fwd_impl(prob, batch, ad, X, W, Y, Hs, ws, ws_bytes, stream_, false);
}

namespace lobra {
namespace {
lobra_status lora_fwd_impl(const lobra_problem* prob, const lobra_batch* batch,
                           const lobra_adapters* ad, const void* X, const void* W, void* Y, void* Hs,
                           void* ws, size_t ws_bytes, lobra_stream_t stream_, bool skip_shrink) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  DevCtx* ctx = nullptr;
  Plan P;
  Layout L;
  lobra_status s = validate(prob, batch, ad);
  if (s != LOBRA_OK) return s;
  s = prepare(prob, batch, ad, unit_width(prob), sms_hint(), P, L);
  if (s != LOBRA_OK) return s;
  if ((s = get_ctx(&ctx)) != LOBRA_OK) return s;
  if (!X || !W || !Y || !Hs || !ws) return fail(LOBRA_ERR_INPUT, "null device pointer");
  if (ws_bytes < L.total) return fail(LOBRA_ERR_INPUT, "workspace too small: %zu < %zu", ws_bytes, L.total);
  if ((reinterpret_cast<uintptr_t>(ws) & 255) || !aligned16(X) || !aligned16(W) || !aligned16(Y) ||
      !aligned16(Hs) || !aligned16(ad->A) || !aligned16(ad->B))
    return fail(LOBRA_ERR_INPUT, "device pointers must be 16-byte aligned (ws 256-byte)");
  if (prob->tp_kind == LOBRA_TP_ROW && prob->tp == nullptr)
    return fail(LOBRA_ERR_INPUT, "row-parallel problem without a comm");
  uint8_t* w = static_cast<uint8_t*>(ws);
  if (P.T == 0) return LOBRA_OK;
  // the unit split only matters for the backward; metadata identical otherwise
  if ((s = upload_meta(ctx, P.buf, w + L.meta, st)) != LOBRA_OK) return s;
  const Meta meta = device_meta(P, w + L.meta);
  const int in = (int)prob->in, out = (int)prob->out;
  if (prob->dtype == LOBRA_FP32) {
    { Prof p_(LOBRA_K_FP32, st); launch_f32_rowproj(0, static_cast<const float*>(X), static_cast<const float*>(ad->A),
                       static_cast<const float*>(ad->B), in, out, meta, static_cast<float*>(Hs), st); }
    { Prof p_(LOBRA_K_FP32, st); launch_f32_gemm(0, static_cast<const float*>(X), static_cast<const float*>(W),
                    static_cast<const float*>(ad->A), static_cast<const float*>(ad->B),
                    static_cast<const float*>(Hs), in, out, meta, static_cast<float*>(Y), 0, st); }
  } else {
    const __nv_bfloat16* Bop = static_cast<const __nv_bfloat16*>(ad->B);
    if (!P.bdirect) {
      auto* Bp = reinterpret_cast<__nv_bfloat16*>(w + L.bpad);
      { Prof p_(LOBRA_K_PAD, st); launch_pad_cols(Bop, Bp, out, L.ld8, meta, st); }
      Bop = Bp;
    }
    CUtensorMap mX, mA, mW, mSlot, mB;
    if ((s = make_map(&mX, X, in, P.T, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mA, ad->A, in, (uint64_t)P.rsum, 64, 64)) != LOBRA_OK) return s;
    const uint32_t bn = 128;   // the 2-CTA GEMM: each CTA loads half of the 256 W rows
    if ((s = make_map(&mW, W, in, out, 64, bn)) != LOBRA_OK) return s;
    if ((s = make_map(&mSlot, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mB, Bop, L.ld8, out, 64, bn)) != LOBRA_OK) return s;
    if (skip_shrink) {
      // H_s computed by the caller (wide projection group)
    } else if (shrink_applies(P.ntiles, ctx->num_sms)) {
      CUtensorMap mAk;
      if ((s = make_map(&mAk, ad->A, in, (uint64_t)P.rsum, 64, P.qp)) != LOBRA_OK) return s;
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_shrink(mX, mAk, in, meta, static_cast<__nv_bfloat16*>(Hs), ctx->num_sms, st);
    } else if (rowproj_uses_ld()) {
      CUtensorMap mAk;
      if ((s = make_map(&mAk, ad->A, in, (uint64_t)P.rsum, 64, P.qp)) != LOBRA_OK) return s;
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_rowproj_ld(static_cast<const __nv_bfloat16*>(X), in, mAk, P.qp, meta,
                        static_cast<__nv_bfloat16*>(Hs), reinterpret_cast<float*>(w + L.rpart),
                        reinterpret_cast<int*>(w + L.counters), st);
    } else {
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_rowproj(false, mX, mA, in, meta, static_cast<__nv_bfloat16*>(Hs),
                     reinterpret_cast<float*>(w + L.rpart), reinterpret_cast<int*>(w + L.counters), st);
    }
    // row-parallel with a symmetric TP group: FUSED GEMM -> reduce-scatter (each output row is
    // stored into its owner rank's buffer over NVLink from the GEMM epilogue), then the owner
    // reduces locally and every rank gathers Y; else the GEMM writes its partial into the
    // peer-visible stage area and the own all-reduce follows (no staging copy either way)
    TpScatter tps;
    if (prob->tp_kind == LOBRA_TP_ROW && tp_fused() &&
        symm_scatter_target(comm_symm(prob->tp), P.T, out, &tps)) {
      { Prof p_(LOBRA_K_GEMM_FWD, st); launch_gemm(false, mX, mW, mSlot, mB, P.T, out, in,
                                                     static_cast<__nv_bfloat16*>(Y), 0, meta, ctx->num_sms, st,
                                                     &tps); }
      if ((s = check_launch("lobra_lora_fwd")) != LOBRA_OK) return s;
      return symm_scatter_finish(comm_symm(prob->tp), P.T, out, Y, st);
    }
    void* stage = prob->tp_kind == LOBRA_TP_ROW ? comm_tp_stage(prob->tp, (size_t)P.T * out * 2) : nullptr;
    { Prof p_(LOBRA_K_GEMM_FWD, st); launch_gemm(false, mX, mW, mSlot, mB, P.T, out, in,
                                                   static_cast<__nv_bfloat16*>(stage ? stage : Y), 0, meta,
                                                   ctx->num_sms, st); }
    if ((s = check_launch("lobra_lora_fwd")) != LOBRA_OK) return s;
    if (prob->tp_kind == LOBRA_TP_ROW) return comm_tp_allreduce_bf16_to(prob->tp, stage ? stage : Y, Y, (size_t)P.T * out, st);
    return LOBRA_OK;
  }
  if ((s = check_launch("lobra_lora_fwd")) != LOBRA_OK) return s;
  if (prob->tp_kind == LOBRA_TP_ROW)
    return comm_tp_allreduce_f32(prob->tp, static_cast<float*>(Y), (size_t)P.T * out, st);
  return LOBRA_OK;
}

}  // namespace
}  // namespace lobra

extern "C" lobra_status lobra_lora_bwd(const lobra_problem* prob, const lobra_batch* batch,
                                       const lobra_adapters* ad, const void* X, const void* W,
                                       const void* Hs, const void* dY, void* dX, int accumulate_dx,
                                       float* dA, float* dB, int accumulate_dadb, void* ws,
                                       size_t ws_bytes, lobra_stream_t stream_) {
  clear_error();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  DevCtx* ctx = nullptr;
  lobra_status s = validate(prob, batch, ad);
  if (s != LOBRA_OK) return s;
  if ((s = get_ctx(&ctx)) != LOBRA_OK) return s;
  Plan P;
  Layout L;
  // units sized for the wider of the two reductions (dA over `in`, dB over `out`)
  if ((s = prepare(prob, batch, ad, unit_width(prob), ctx->num_sms, P, L)) != LOBRA_OK)
    return s;
  if (!X || !W || !Hs || !dY || !dX || !dA || !dB || !ws)
    return fail(LOBRA_ERR_INPUT, "null device pointer");
  if (ws_bytes < L.total)
    return fail(LOBRA_ERR_INPUT, "workspace too small: %zu < %zu", ws_bytes, L.total);
  if ((reinterpret_cast<uintptr_t>(ws) & 255) || !aligned16(X) || !aligned16(W) || !aligned16(Hs) ||
      !aligned16(dY) || !aligned16(dX) || !aligned16(ad->A) || !aligned16(ad->B) || !aligned16(dA) ||
      !aligned16(dB))
    return fail(LOBRA_ERR_INPUT, "device pointers must be 16-byte aligned (ws 256-byte)");
  if (prob->tp_kind == LOBRA_TP_COLUMN && prob->tp == nullptr)
    return fail(LOBRA_ERR_INPUT, "column-parallel problem without a comm");
  const int in = (int)prob->in, out = (int)prob->out;
  const long long ldA = prob->dA_ld ? prob->dA_ld : prob->in;
  uint8_t* w = static_cast<uint8_t*>(ws);
  if (P.T == 0) {
    // no tokens: dX untouched (nothing to write), gradients zero unless accumulating
    if (!accumulate_dadb) {
      for (int r = 0; r < P.rsum; ++r) cudaMemsetAsync(dA + (size_t)r * ldA, 0, sizeof(float) * in, st);
      cudaMemsetAsync(dB, 0, sizeof(float) * (size_t)out * P.rsum, st);
    }
    return check_launch("lobra_lora_bwd(empty)");
  }
  if ((s = upload_meta(ctx, P.buf, w + L.meta, st)) != LOBRA_OK) return s;
  const Meta meta = device_meta(P, w + L.meta);
  if (prob->dtype == LOBRA_FP32) {
    float* G = reinterpret_cast<float*>(w + L.gslots);
    const float* Af = static_cast<const float*>(ad->A);
    const float* Bf = static_cast<const float*>(ad->B);
    { Prof p_(LOBRA_K_FP32, st); launch_f32_rowproj(1, static_cast<const float*>(dY), Af, Bf, in, out, meta, G, st); }
    { Prof p_(LOBRA_K_FP32, st); launch_f32_gemm(1, static_cast<const float*>(dY), static_cast<const float*>(W), Af, Bf, G, in,
                    out, meta, static_cast<float*>(dX), accumulate_dx, st); }
    { Prof p_(LOBRA_K_FP32, st); launch_f32_segred(0, static_cast<const float*>(X), G, in, meta, dA, ldA, accumulate_dadb, st); }
    { Prof p_(LOBRA_K_FP32, st); launch_f32_segred(1, static_cast<const float*>(dY), static_cast<const float*>(Hs), out, meta,
                      dB, 0, accumulate_dadb, st); }
  } else {
    auto* Gs = reinterpret_cast<__nv_bfloat16*>(w + L.gslots);
    float* partA = reinterpret_cast<float*>(w + L.partA);
    float* partB = reinterpret_cast<float*>(w + L.partB);
    const __nv_bfloat16* Bop = static_cast<const __nv_bfloat16*>(ad->B);
    if (!P.bdirect) {
      auto* Bp = reinterpret_cast<__nv_bfloat16*>(w + L.bpad);
      { Prof p_(LOBRA_K_PAD, st); launch_pad_cols(Bop, Bp, out, L.ld8, meta, st); }
      Bop = Bp;
    }
    CUtensorMap mdY, mBt, mWmn, mG, mAt, mX, mHs;
    if ((s = make_map(&mdY, dY, out, P.T, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mBt, Bop, L.ld8, out, 64, 64)) != LOBRA_OK) return s;
    if ((s = make_map(&mWmn, W, in, out, 64, 64)) != LOBRA_OK) return s;
    if ((s = make_map(&mG, Gs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mAt, ad->A, in, (uint64_t)P.rsum, 64, 64)) != LOBRA_OK) return s;
    if ((s = make_map(&mX, X, in, P.T, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mHs, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
    const bool fused_dy = dy_fused();
    Meta meta_b = meta;
    if (fused_dy) {
      // G_s and the dB partials in ONE read of dY; B read in place
      // (MN-major operand, box 64 q x 64 o rows: the same map as the two-pass projection)
      const int sp = dypass_span(P.qp);
      CUtensorMap mHd, mBd;
      if ((s = make_map(&mHd, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, sp / 2, 128, sp)) != LOBRA_OK) return s;
      if ((s = make_map(&mBd, Bop, L.ld8, out, sp / 2, 64, sp)) != LOBRA_OK) return s;
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_dypass(mdY, mHd, mBd, out, P.qp, meta, reinterpret_cast<float*>(w + L.gpart), partB, Gs,
                    ctx->num_sms, st);
      meta_b.use_dy_units = 1;
    } else if (rowproj_uses_ld()) {   // workspace has L.bt only in this mode
      auto* Bt = reinterpret_cast<__nv_bfloat16*>(w + L.bt);
      {
        Prof p_(LOBRA_K_PAD, st);
        launch_transpose_b(static_cast<const __nv_bfloat16*>(ad->B), Bt, out, P.rsum, st);
      }
      CUtensorMap mBk;
      if ((s = make_map(&mBk, Bt, out, (uint64_t)P.rsum, 64, P.qp)) != LOBRA_OK) return s;
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_rowproj_ld(static_cast<const __nv_bfloat16*>(dY), out, mBk, P.qp, meta, Gs,
                        reinterpret_cast<float*>(w + L.rpart), reinterpret_cast<int*>(w + L.counters),
                        st);
    } else {
      Prof p_(LOBRA_K_ROWPROJ, st);
      launch_rowproj(true, mdY, mBt, out, meta, Gs, reinterpret_cast<float*>(w + L.rpart),
                     reinterpret_cast<int*>(w + L.counters), st);
    }
    // column-parallel with a symmetric TP group: FUSED GEMM -> reduce-scatter (the epilogue adds
    // the local partial in dX when accumulating and stores each row into its owner's buffer)
    TpScatter tps;
    const bool fused_tp = prob->tp_kind == LOBRA_TP_COLUMN && tp_fused() &&
                          symm_scatter_target(comm_symm(prob->tp), P.T, in, &tps);
    { Prof p_(LOBRA_K_GEMM_BWD, st); launch_gemm(true, mdY, mWmn, mG, mAt, P.T, in, out, static_cast<__nv_bfloat16*>(dX),
                accumulate_dx, meta, ctx->num_sms, st, fused_tp ? &tps : nullptr); }
    Meta meta_a = meta;
    set_sr(meta_a, P, w + L.meta, in);
    if (meta.nunits) { Prof p_(LOBRA_K_SEGRED, st); launch_segred(mX, mG, in, meta_a, partA, ctx->num_sms, st); }
    Meta meta_s = meta;
    set_sr(meta_s, P, w + L.meta, out);
    if (!fused_dy && meta.nunits) { Prof p_(LOBRA_K_SEGRED, st); launch_segred(mdY, mHs, out, meta_s, partB, ctx->num_sms, st); }
    {
      // dA and dB in one launch (segment partials: k_segred [seg][qp][128], dY pass [seg][4][qp][128])
      const FinJob jobs[2] = {
          {partA, dA, ldA, meta_a.sr_tc_off, 0, in, (in + 127) / 128, 0, meta.qp, 1, meta_a.sr_nch, accumulate_dadb, 1},
          {partB, dB, 0, fused_dy ? meta_b.dy_task_unit_off : meta_s.sr_tc_off, 1, out, (out + 127) / 128, 0,
           meta.qp, 1, fused_dy ? meta_b.dy_nch : meta_s.sr_nch, accumulate_dadb, fused_dy ? 4 : 1}};
      Prof p_(LOBRA_K_FINALIZE, st);
      launch_finalize_multi(jobs, 2, meta, st);
    }
  }
  if ((s = check_launch("lobra_lora_bwd")) != LOBRA_OK) return s;
  if (prob->dtype == LOBRA_BF16 && prob->tp_kind == LOBRA_TP_COLUMN && tp_fused()) {
    TpScatter tps;
    if (symm_scatter_target(comm_symm(prob->tp), P.T, in, &tps))   // the GEMM already scattered
      return symm_scatter_finish(comm_symm(prob->tp), P.T, in, dX, st);
  }
  if (prob->tp_kind == LOBRA_TP_COLUMN) {
    const size_t cnt = (size_t)P.T * in;
    return prob->dtype == LOBRA_BF16 ? comm_tp_allreduce_bf16(prob->tp, dX, cnt, st)
                                     : comm_tp_allreduce_f32(prob->tp, static_cast<float*>(dX), cnt, st);
  }
  return LOBRA_OK;
}

// ======================================================================================
// Projection groups (include/lobra.h): projections sharing X read it once for the shrink
// and once for the dA reduction; H_s / G_s slots hold one qp-wide band per projection.
// ======================================================================================
namespace lobra {
namespace {

lobra_status validate_group(const lobra_group_problem* g, const lobra_batch* b,
                            const lobra_group_adapters* ga) {
  if (!g || !b || !ga) return fail(LOBRA_ERR_INPUT, "null problem/batch/adapters");
  if (g->num_proj < 1 || g->num_proj > 4 || !g->out)
    return fail(LOBRA_ERR_INPUT, "num_proj must be 1..4 with an out[] array");
  if (!ga->A || !ga->B) return fail(LOBRA_ERR_INPUT, "A[] / B[] pointer arrays missing");
  for (int p = 0; p < g->num_proj; ++p) {
    lobra_problem sp{g->dtype, g->in, g->out[p], g->tp_kind, g->tp, g->dA_ld};
    lobra_adapters sa{ga->num_tasks, ga->ranks, ga->scales, ga->A[p], ga->B[p]};
    lobra_status s = validate(&sp, b, &sa);
    if (s != LOBRA_OK) return s;
  }
  return LOBRA_OK;
}

lobra_problem single_problem(const lobra_group_problem* g, int p, lobra_tp_kind kind) {
  return lobra_problem{g->dtype, g->in, g->out[p], kind, g->tp, g->dA_ld};
}
lobra_adapters single_adapters(const lobra_group_adapters* ga, int p) {
  return lobra_adapters{ga->num_tasks, ga->ranks, ga->scales, ga->A[p], ga->B[p]};
}

int64_t max_out(const lobra_group_problem* g) {
  int64_t m = 0;
  for (int p = 0; p < g->num_proj; ++p) m = std::max<int64_t>(m, g->out[p]);
  return m;
}

// Banded path applies: bf16, the bands fit the 64-wide slot, default backward kernels.
bool group_fused(const lobra_group_problem* g, const lobra_group_adapters* ga) {
  if (g->dtype != LOBRA_BF16 || !dy_fused() || rowproj_uses_ld()) return false;
  int qp = 16;
  for (int t = 0; t < ga->num_tasks; ++t) qp = std::max(qp, (ga->ranks[t] + 15) & ~15);
  return g->num_proj * qp <= kSlotW;
}

struct GroupLayout {
  size_t meta = 0, bpad = 0, agrp = 0, gslots = 0, rpart = 0, counters = 0, partA = 0, partB = 0,
         gpart = 0, total = 0, saved = 0;
  size_t partB_stride = 0;   // floats between the per-projection dB partial regions
};

GroupLayout group_layout(const lobra_group_problem* g, const Plan& P) {
  GroupLayout L;
  const size_t in = g->in, omax = max_out(g), qg = (size_t)P.np * P.qp;
  size_t off = 0;
  L.meta = off;
  off += align256(P.buf.size() * 4);
  L.bpad = off;
  if (!P.bdirect) off += align256(omax * P.ld8 * 2);
  L.agrp = off;
  off += align256((size_t)P.ntasks * qg * in * 2);
  L.gslots = off;
  off += align256((size_t)(P.nslots + 1) * kTileM * kSlotW * 2);
  const int sp = rowproj_splits(P.ntiles, (int)in);
  L.rpart = off;
  if (sp > 1) off += align256((size_t)sp * P.nslots * kTileM * 64 * 4);
  L.counters = off;
  off += align256((size_t)P.ntiles * 4);
  L.partA = off;
  off += align256(std::max((size_t)P.nunits * ((in + 127) / 128), (size_t)P.nsrseg) * qg * 128 * 4);
  L.partB = off;
  // per projection [segments][4][qp][128] (the dB finalize of the whole group runs after the loop)
  L.partB_stride = (size_t)P.ndyunits * 4 * P.qp * 128;
  off += align256(L.partB_stride * 4 * P.np);
  L.gpart = off;
  off += align256((size_t)P.nslots * ((omax + 511) / 512) * kTileM * P.qp * 4);
  L.saved = (size_t)(P.nslots + 1) * kTileM * kSlotW * 2;
  L.total = off;
  return L;
}

void group_plan(const lobra_group_problem* g, const lobra_batch* b, const lobra_group_adapters* ga,
                int num_sms, Plan& P) {
  lobra_adapters a0 = single_adapters(ga, 0);
  std::vector<int> outs;
  for (int p = 0; p < g->num_proj; ++p) outs.push_back((int)g->out[p]);
  // units: dA over in; one fused-dY schedule per distinct output width
  build_plan(b, &a0, (int)g->in, (int)max_out(g), num_sms, P, g->num_proj, outs, {(int)g->in});
}

// Wide group (bands exceed the 64-wide slot, np * qp in (64, 256], e.g. q/k/v at rank 64): the
// per-projection sequence, except that ONE k_shrink pass over X computes every projection's
// H_s into its own slot buffer (planes), so X is read once for the shrinks instead of np times.
bool wide_planes(const lobra_group_problem* g, const lobra_batch* b, const lobra_group_adapters* ga) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LOBRA_WIDE_GROUP");   // 0: plain per-projection sequence (A/B)
    v = e ? atoi(e) : 1;
  }
  if (!v || g->dtype != LOBRA_BF16 || !dy_fused() || rowproj_uses_ld() ||
      g->tp_kind == LOBRA_TP_ROW || g->num_proj < 2)
    return false;
  int qp = 16;
  for (int t = 0; t < ga->num_tasks; ++t) qp = std::max(qp, (ga->ranks[t] + 15) & ~15);
  if (g->num_proj * qp <= kSlotW || g->num_proj * qp > 256) return false;
  long long T = 0;
  for (int k = 0; k < b->num_seqs; ++k) T += b->seq_lens[k];
  return shrink_applies((int)((T + kTileM - 1) / kTileM), sms_hint());
}
// workspace of the wide-group shrink: group metadata + the packed group A
size_t planes_ws(const lobra_group_problem* g, const Plan& P) {
  return align256(P.buf.size() * 4) + align256((size_t)P.ntasks * P.np * P.qp * g->in * 2);
}

// workspace / saved sizes of the fallback (per-projection sequences)
size_t fallback_ws(const lobra_group_problem* g, const lobra_batch* b, const lobra_group_adapters* ga) {
  size_t m = 0;
  for (int p = 0; p < g->num_proj; ++p) {
    lobra_problem sp = single_problem(g, p, g->tp_kind);
    lobra_adapters sa = single_adapters(ga, p);
    m = std::max(m, lobra_lora_workspace_bytes(&sp, b, &sa));
  }
  if (wide_planes(g, b, ga)) {
    Plan P;
    group_plan(g, b, ga, sms_hint(), P);
    m = std::max(m, planes_ws(g, P));
  }
  return m;
}
size_t fallback_saved_each(const lobra_group_problem* g, const lobra_batch* b,
                           const lobra_group_adapters* ga) {
  size_t m = 0;
  for (int p = 0; p < g->num_proj; ++p) {
    lobra_problem sp = single_problem(g, p, g->tp_kind);
    lobra_adapters sa = single_adapters(ga, p);
    m = std::max(m, lobra_lora_saved_bytes(&sp, b, &sa));
  }
  return (m + 255) & ~size_t(255);
}

}  // namespace
}  // namespace lobra

extern "C" size_t lobra_lora_group_workspace_bytes(const lobra_group_problem* g, const lobra_batch* b,
                                                   const lobra_group_adapters* ga) {
  clear_error();
  if (validate_group(g, b, ga) != LOBRA_OK) return 0;
  if (!group_fused(g, ga)) return fallback_ws(g, b, ga);
  Plan P;
  group_plan(g, b, ga, sms_hint(), P);
  return group_layout(g, P).total;
}

extern "C" size_t lobra_lora_group_saved_bytes(const lobra_group_problem* g, const lobra_batch* b,
                                               const lobra_group_adapters* ga) {
  clear_error();
  if (validate_group(g, b, ga) != LOBRA_OK) return 0;
  if (!group_fused(g, ga)) return fallback_saved_each(g, b, ga) * g->num_proj;
  Plan P;
  group_plan(g, b, ga, 1 << 20, P);
  return std::max<size_t>(group_layout(g, P).saved, 256);
}

extern "C" lobra_status lobra_lora_group_fwd(const lobra_group_problem* g, const lobra_batch* batch,
                                             const lobra_group_adapters* ga, const void* X,
                                             const void* const* W, void* const* Y, void* Hs, void* ws,
                                             size_t ws_bytes, lobra_stream_t stream_) {
  clear_error();
  lobra_status s = validate_group(g, batch, ga);
  if (s != LOBRA_OK) return s;
  if (!W || !Y) return fail(LOBRA_ERR_INPUT, "W[] / Y[] pointer arrays missing");
  const int np = g->num_proj;
  if (!group_fused(g, ga)) {
    // fallback: np single-projection forwards, each with its own band of Hs; a wide group
    // computes every projection's H_s first in one pass over X
    const size_t each = fallback_saved_each(g, batch, ga);
    const bool planes = wide_planes(g, batch, ga);
    if (planes) {
      cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
      DevCtx* ctx = nullptr;
      if ((s = get_ctx(&ctx)) != LOBRA_OK) return s;
      Plan P;
      group_plan(g, batch, ga, sms_hint(), P);
      if (!X || !Hs || !ws) return fail(LOBRA_ERR_INPUT, "null device pointer");
      if (ws_bytes < planes_ws(g, P)) return fail(LOBRA_ERR_INPUT, "workspace too small: %zu < %zu", ws_bytes,
                                                  planes_ws(g, P));
      if (P.T > 0) {
        uint8_t* w = static_cast<uint8_t*>(ws);
        if ((s = upload_meta(ctx, P.buf, w, st)) != LOBRA_OK) return s;
        const Meta meta = device_meta(P, w);
        const Meta meta_g = group_meta(P, w);
        const int in = (int)g->in;
        auto* Ag = reinterpret_cast<__nv_bfloat16*>(w + align256(P.buf.size() * 4));
        {
          const __nv_bfloat16* As[4];
          for (int p = 0; p < np; ++p) As[p] = static_cast<const __nv_bfloat16*>(ga->A[p]);
          Prof p_(LOBRA_K_PAD, st);
          launch_pack_a_group(As, np, P.qp, in, meta, Ag, st);
        }
        CUtensorMap mX, mAgk;
        if ((s = make_map(&mX, X, in, P.T, 64, 128)) != LOBRA_OK) return s;
        if ((s = make_map(&mAgk, Ag, in, (uint64_t)P.ntasks * np * P.qp, 64, np * P.qp)) != LOBRA_OK) return s;
        const ShrinkPlanes pl{np, P.qp, (long long)(each / 2), meta.ranks, meta.scales};
        Prof p_(LOBRA_K_ROWPROJ, st);
        launch_shrink(mX, mAgk, in, meta_g, static_cast<__nv_bfloat16*>(Hs), ctx->num_sms, st, &pl);
      }
    }
    for (int p = 0; p < np; ++p) {
      lobra_problem sp = single_problem(g, p, g->tp_kind);
      lobra_adapters sa = single_adapters(ga, p);
      if ((s = lora_fwd_impl(&sp, batch, &sa, X, W[p], Y[p], static_cast<uint8_t*>(Hs) + p * each, ws,
                             ws_bytes, stream_, planes)) != LOBRA_OK)
        return s;
    }
    return LOBRA_OK;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  DevCtx* ctx = nullptr;
  if ((s = get_ctx(&ctx)) != LOBRA_OK) return s;
  Plan P;
  group_plan(g, batch, ga, sms_hint(), P);
  const GroupLayout L = group_layout(g, P);
  if (!X || !Hs || !ws) return fail(LOBRA_ERR_INPUT, "null device pointer");
  if (ws_bytes < L.total) return fail(LOBRA_ERR_INPUT, "workspace too small: %zu < %zu", ws_bytes, L.total);
  bool al = (reinterpret_cast<uintptr_t>(ws) & 255) == 0 && aligned16(X) && aligned16(Hs);
  for (int p = 0; p < np; ++p)
    al = al && W[p] && Y[p] && aligned16(W[p]) && aligned16(Y[p]) && aligned16(ga->A[p]) && aligned16(ga->B[p]);
  if (!al) return fail(LOBRA_ERR_INPUT, "device pointers must be non-null and 16-byte aligned (ws 256-byte)");
  if (g->tp_kind == LOBRA_TP_ROW && g->tp == nullptr)
    return fail(LOBRA_ERR_INPUT, "row-parallel problem without a comm");
  if (P.T == 0) return LOBRA_OK;
  uint8_t* w = static_cast<uint8_t*>(ws);
  if ((s = upload_meta(ctx, P.buf, w + L.meta, st)) != LOBRA_OK) return s;
  const Meta meta = device_meta(P, w + L.meta);
  const Meta meta_g = group_meta(P, w + L.meta);
  const int in = (int)g->in;
  auto* Ag = reinterpret_cast<__nv_bfloat16*>(w + L.agrp);
  {
    const __nv_bfloat16* As[4];
    for (int p = 0; p < np; ++p) As[p] = static_cast<const __nv_bfloat16*>(ga->A[p]);
    Prof p_(LOBRA_K_PAD, st);
    launch_pack_a_group(As, np, P.qp, in, meta, Ag, st);
  }
  CUtensorMap mX, mAg, mSlot;
  if ((s = make_map(&mX, X, in, P.T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_map(&mAg, Ag, in, (uint64_t)P.ntasks * np * P.qp, 64, 64)) != LOBRA_OK) return s;
  if ((s = make_map(&mSlot, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
  if (shrink_applies(P.ntiles, ctx->num_sms)) {
    // a1: every projection's H_s from ONE pass over X (band p = columns [p qp, (p+1) qp))
    CUtensorMap mAgk;
    if ((s = make_map(&mAgk, Ag, in, (uint64_t)P.ntasks * np * P.qp, 64, np * P.qp)) != LOBRA_OK) return s;
    Prof p_(LOBRA_K_ROWPROJ, st);
    launch_shrink(mX, mAgk, in, meta_g, static_cast<__nv_bfloat16*>(Hs), ctx->num_sms, st);
  } else {
    Prof p_(LOBRA_K_ROWPROJ, st);
    launch_rowproj(false, mX, mAg, in, meta_g, static_cast<__nv_bfloat16*>(Hs),
                   reinterpret_cast<float*>(w + L.rpart), reinterpret_cast<int*>(w + L.counters), st);
  }
  for (int p = 0; p < np; ++p) {
    const int out = (int)g->out[p];
    const __nv_bfloat16* Bop = static_cast<const __nv_bfloat16*>(ga->B[p]);
    if (!P.bdirect) {
      auto* Bp = reinterpret_cast<__nv_bfloat16*>(w + L.bpad);
      { Prof p_(LOBRA_K_PAD, st); launch_pad_cols(Bop, Bp, out, P.ld8, meta, st); }
      Bop = Bp;
    }
    CUtensorMap mW, mB;
    if ((s = make_map(&mW, W[p], in, out, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mB, Bop, P.ld8, out, 64, 128)) != LOBRA_OK) return s;
    Meta mp = meta;
    mp.band = p * P.qp;
    void* stage = g->tp_kind == LOBRA_TP_ROW ? comm_tp_stage(g->tp, (size_t)P.T * out * 2) : nullptr;
    { Prof p_(LOBRA_K_GEMM_FWD, st); launch_gemm(false, mX, mW, mSlot, mB, P.T, out, in,
                                                   static_cast<__nv_bfloat16*>(stage ? stage : Y[p]), 0, mp,
                                                   ctx->num_sms, st); }
    if ((s = check_launch("lobra_lora_group_fwd")) != LOBRA_OK) return s;
    if (g->tp_kind == LOBRA_TP_ROW)
      if ((s = comm_tp_allreduce_bf16_to(g->tp, stage ? stage : Y[p], Y[p], (size_t)P.T * out, st)) != LOBRA_OK)
        return s;
  }
  return LOBRA_OK;
}

extern "C" lobra_status lobra_lora_group_bwd(const lobra_group_problem* g, const lobra_batch* batch,
                                             const lobra_group_adapters* ga, const void* X,
                                             const void* const* W, const void* Hs,
                                             const void* const* dY, void* dX, int accumulate_dx,
                                             float* const* dA, float* const* dB, int accumulate_dadb,
                                             void* ws, size_t ws_bytes, lobra_stream_t stream_) {
  clear_error();
  lobra_status s = validate_group(g, batch, ga);
  if (s != LOBRA_OK) return s;
  if (!W || !dY || !dA || !dB) return fail(LOBRA_ERR_INPUT, "W[] / dY[] / dA[] / dB[] pointer arrays missing");
  const int np = g->num_proj;
  if (!group_fused(g, ga)) {
    const size_t each = fallback_saved_each(g, batch, ga);
    for (int p = 0; p < np; ++p) {
      // dX accumulates across the group; a column-parallel group all-reduces once, last
      lobra_problem sp = single_problem(g, p, p == np - 1 || g->tp_kind != LOBRA_TP_COLUMN
                                                  ? g->tp_kind : LOBRA_TP_NONE);
      lobra_adapters sa = single_adapters(ga, p);
      if ((s = lobra_lora_bwd(&sp, batch, &sa, X, W[p], static_cast<const uint8_t*>(Hs) + p * each, dY[p], dX,
                              p > 0 ? 1 : accumulate_dx, dA[p], dB[p], accumulate_dadb, ws, ws_bytes,
                              stream_)) != LOBRA_OK)
        return s;
    }
    return LOBRA_OK;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  DevCtx* ctx = nullptr;
  if ((s = get_ctx(&ctx)) != LOBRA_OK) return s;
  Plan P;
  group_plan(g, batch, ga, ctx->num_sms, P);
  const GroupLayout L = group_layout(g, P);
  if (!X || !Hs || !dX || !ws) return fail(LOBRA_ERR_INPUT, "null device pointer");
  if (ws_bytes < L.total) return fail(LOBRA_ERR_INPUT, "workspace too small: %zu < %zu", ws_bytes, L.total);
  bool al = (reinterpret_cast<uintptr_t>(ws) & 255) == 0 && aligned16(X) && aligned16(Hs) && aligned16(dX);
  for (int p = 0; p < np; ++p)
    al = al && W[p] && dY[p] && dA[p] && dB[p] && aligned16(W[p]) && aligned16(dY[p]) && aligned16(dA[p]) &&
         aligned16(dB[p]) && aligned16(ga->A[p]) && aligned16(ga->B[p]);
  if (!al) return fail(LOBRA_ERR_INPUT, "device pointers must be non-null and 16-byte aligned (ws 256-byte)");
  if (g->tp_kind == LOBRA_TP_COLUMN && g->tp == nullptr)
    return fail(LOBRA_ERR_INPUT, "column-parallel problem without a comm");
  const int in = (int)g->in;
  const long long ldA = g->dA_ld ? g->dA_ld : g->in;
  if (P.T == 0) {
    if (!accumulate_dadb)
      for (int p = 0; p < np; ++p) {
        for (int r = 0; r < P.rsum; ++r) cudaMemsetAsync(dA[p] + (size_t)r * ldA, 0, sizeof(float) * in, st);
        cudaMemsetAsync(dB[p], 0, sizeof(float) * (size_t)g->out[p] * P.rsum, st);
      }
    return check_launch("lobra_lora_group_bwd(empty)");
  }
  uint8_t* w = static_cast<uint8_t*>(ws);
  if ((s = upload_meta(ctx, P.buf, w + L.meta, st)) != LOBRA_OK) return s;
  const Meta meta = device_meta(P, w + L.meta);
  const Meta meta_g = group_meta(P, w + L.meta);
  auto* Gs = reinterpret_cast<__nv_bfloat16*>(w + L.gslots);
  float* partA = reinterpret_cast<float*>(w + L.partA);
  float* partB = reinterpret_cast<float*>(w + L.partB);
  CUtensorMap mX, mG, mHs;
  if ((s = make_map(&mX, X, in, P.T, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_map(&mG, Gs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
  if ((s = make_map(&mHs, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, 64, 128)) != LOBRA_OK) return s;
  // column-parallel with a symmetric TP group: the group's dX GEMMs accumulate straight into
  // the peer-visible stage area, the own all-reduce then reduces it into dX
  TpScatter tps;
  const bool fused_tp = g->tp_kind == LOBRA_TP_COLUMN && tp_fused() &&
                        symm_scatter_target(comm_symm(g->tp), P.T, in, &tps);
  void* stage = g->tp_kind == LOBRA_TP_COLUMN && !fused_tp ? comm_tp_stage(g->tp, (size_t)P.T * in * 2) : nullptr;
  if (stage && accumulate_dx &&
      cudaMemcpyAsync(stage, dX, (size_t)P.T * in * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return fail(LOBRA_ERR_CUDA, "TP stage copy failed");
  auto* dXacc = static_cast<__nv_bfloat16*>(stage ? stage : dX);
  FinJob jobs[kMaxFinJobs];
  for (int p = 0; p < np; ++p) {
    const int out = (int)g->out[p];
    const __nv_bfloat16* Bop = static_cast<const __nv_bfloat16*>(ga->B[p]);
    if (!P.bdirect) {
      auto* Bp = reinterpret_cast<__nv_bfloat16*>(w + L.bpad);
      { Prof p_(LOBRA_K_PAD, st); launch_pad_cols(Bop, Bp, out, P.ld8, meta, st); }
      Bop = Bp;
    }
    CUtensorMap mdY, mBt, mWmn, mAt;
    if ((s = make_map(&mdY, dY[p], out, P.T, 64, 128)) != LOBRA_OK) return s;
    if ((s = make_map(&mBt, Bop, P.ld8, out, 64, 64)) != LOBRA_OK) return s;
    if ((s = make_map(&mWmn, W[p], in, out, 64, 64)) != LOBRA_OK) return s;
    if ((s = make_map(&mAt, ga->A[p], in, (uint64_t)P.rsum, 64, 64)) != LOBRA_OK) return s;
    Meta mp = meta;
    mp.band = p * P.qp;
    set_dy(mp, P, w + L.meta, out);
    const int sp = dypass_span(P.qp);
    CUtensorMap mHd, mBd;
    if ((s = make_map(&mHd, Hs, 64, (uint64_t)(P.nslots + 1) * kTileM, sp / 2, 128, sp)) != LOBRA_OK) return s;
    if ((s = make_map(&mBd, Bop, P.ld8, out, sp / 2, 64, sp)) != LOBRA_OK) return s;
    {
      // a3 for projection p: G_s into band p, dB partials against band p of H_s
      Prof p_(LOBRA_K_ROWPROJ, st);
      // dB partials of projection p in their own region (finalized after the loop)
      launch_dypass(mdY, mHd, mBd, out, P.qp, mp, reinterpret_cast<float*>(w + L.gpart),
                    partB + (size_t)p * L.partB_stride, Gs, ctx->num_sms, st);
    }
    // fused TP: projections 0..np-2 accumulate locally in dX, the last one scatters the rows
    { Prof p_(LOBRA_K_GEMM_BWD, st); launch_gemm(true, mdY, mWmn, mG, mAt, P.T, in, out, dXacc,
                                                   p > 0 ? 1 : accumulate_dx, mp, ctx->num_sms, st,
                                                   fused_tp && p == np - 1 ? &tps : nullptr); }
    jobs[np + p] = {partB + (size_t)p * L.partB_stride, dB[p], 0, mp.dy_task_unit_off, 1, out,
                    (out + 127) / 128, 0, P.qp, 1, mp.dy_nch, accumulate_dadb, 4};
  }
  // a5 for the whole group: ONE pass over X against all bands of G_s
  if (meta.nunits) { Prof p_(LOBRA_K_SEGRED, st); launch_segred(mX, mG, in, meta_g, partA, ctx->num_sms, st); }
  for (int p = 0; p < np; ++p)
    jobs[p] = {partA, dA[p], ldA, meta_g.sr_tc_off, 0, in, (in + 127) / 128, p * P.qp, np * P.qp, 1,
               meta_g.sr_nch, accumulate_dadb, 1};
  {
    // every projection's dA and dB in one launch
    Prof p_(LOBRA_K_FINALIZE, st);
    launch_finalize_multi(jobs, 2 * np, meta, st);
  }
  if ((s = check_launch("lobra_lora_group_bwd")) != LOBRA_OK) return s;
  if (fused_tp) return symm_scatter_finish(comm_symm(g->tp), P.T, in, dX, st);
  if (g->tp_kind == LOBRA_TP_COLUMN) return comm_tp_allreduce_bf16_to(g->tp, dXacc, dX, (size_t)P.T * in, st);
  return LOBRA_OK;
}

extern "C" lobra_status lobra_profile_enable(int on) {
  clear_error();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return LOBRA_OK;
}

extern "C" lobra_status lobra_profile_read(lobra_profile* out, int reset) {
  clear_error();
  if (!out) return fail(LOBRA_ERR_INPUT, "null output");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfRec& r : g_prof_recs) {
    if (cudaEventSynchronize(r.e1) != cudaSuccess) return fail(LOBRA_ERR_CUDA, "event sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    g_prof_ms[r.kind] += ms;
    g_prof_count[r.kind] += 1;
    g_prof_pool.push_back(r.e0);
    g_prof_pool.push_back(r.e1);
  }
  g_prof_recs.clear();
  for (int k = 0; k < LOBRA_K_NUM; ++k) out->count[k] = g_prof_count[k], out->ms[k] = g_prof_ms[k];
  if (reset)
    for (int k = 0; k < LOBRA_K_NUM; ++k) g_prof_count[k] = 0, g_prof_ms[k] = 0;
  return LOBRA_OK;
}

extern "C" int64_t lobra_launch_count(void) { return g_launches.load(); }

extern "C" lobra_status lobra_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  for (DevCtx* c : g_ctx) {
    if (!c) continue;
    for (int i = 0; i < kRing; ++i) {
      if (c->ev[i]) cudaEventSynchronize(c->ev[i]), cudaEventDestroy(c->ev[i]);
      if (c->pinned[i]) cudaFreeHost(c->pinned[i]);
    }
    delete c;
  }
  g_ctx.clear();
  return LOBRA_OK;
}
