// C-ABI of libhet (include/het.h): argument checks, allocation, per-call
// orchestration of the sm_100a kernels on the caller's stream, profiling.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/het.h"
#include "het_internal.cuh"
#include "het_mgpu.h"
#include "het_p2p.h"

// NVTX ranges over the public calls (header-only NVTX 3: a null check when no
// tool is attached), so nsys/ncu timelines show the protocol phases.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace het {
void dedup_set_attrs();
void cache_set_attrs();
size_t evbuf_struct_size();
void evbuf_init(void* evbuf, uint32_t* hist, uint32_t* khist, int32_t* victims, int32_t* cand,
                int32_t* sub, int32_t* flags, int64_t* vkeys, uint8_t* vdirty, int64_t* vsel);
}  // namespace het

using namespace het;

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};

struct het_cache;
// Loopback group (het_group_create): N workers of one process on one device,
// their inboxes shared by plain device pointers; every collective call is
// driven phase by phase across the members (no NCCL, no spinning wait).
struct het_group {
  std::vector<het_cache*> m;   // members in rank order
};

struct het_cache {
  Dev d{};
  uint64_t R = 0;
  uint32_t D = 0;
  int64_t C = 0;
  uint32_t n_max = 0;
  int pbits = 1;
  // per-call scratch
  Call call{};
  void* evbuf_host = nullptr;  // EvBuf struct (host copy, device pointers inside)
  int32_t* victims = nullptr;
  int64_t* victim_keys = nullptr;
  uint8_t* victim_dirty = nullptr;
  int64_t* victim_sel = nullptr;
  // staging for host pointers (allocated on first use)
  int64_t* stage_keys = nullptr;
  int64_t* stage_pref = nullptr;   // het_prefetch's host keys
  float* stage_rows = nullptr;
  float* stage_out = nullptr;
  // protocol state
  bool have_lookup = false;
  bool fused = false;          // the last lookup ran the fused kernels
  uint32_t last_n = 0;
  const int64_t* last_keys = nullptr;  // the lookup's keys as passed by the caller
  bool no_fused = false;       // env HET_NO_FUSED (read once at create)
  bool ev_pending = false;     // a fused update may have left listed victims (evicted by the next call's first kernel)
  bool ev_captured = false;    // a fused update was captured into a CUDA graph (replays leave victims listed)
  std::shared_ptr<het_group> group;    // loopback member (nullptr: one process per GPU)
  // het_prefetch (NEXT-1): the next lookup's dedup, run ahead into the
  // alternate sort/perm buffers
  uint64_t* sb_alt = nullptr;
  int32_t* perm_alt = nullptr;
  const int64_t* pref_keys = nullptr;  // as the caller passed them (nullptr: nothing prefetched)
  uint32_t pref_n = 0;
  int64_t overflow_bound = 0;  // worst-case residents above C since the last eviction
  uint64_t lookups = 0, keys = 0, updates = 0, launches = 0;
  // multi-GPU
  MgpuState* mg = nullptr;
  // segment reduce of large batches: heavy keys on a forked stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // host gradients: staged on a copy stream, so the H2D overlaps the lookup's
  // kernels and its D2H of the rows (full-duplex link); the events order it
  // after the previous update's reads of the staging buffer and before this one's
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_rows_free = nullptr, ev_rows_ready = nullptr;
  // host rows out of a lookup: the update that follows with host gradients
  // runs on `ustream`, after the lookup's kernels (ev_lk_done, recorded before
  // the D2H of the rows) instead of after the D2H, and the caller's stream
  // waits for it (ev_upd_done): the update's kernels overlap the copy.  Valid
  // only for the call right after the lookup (lk_done_valid).
  cudaStream_t ustream = nullptr;
  cudaEvent_t ev_lk_done = nullptr, ev_upd_done = nullptr;
  bool lk_done_valid = false;
  // profiling
  bool prof = false;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<std::string, std::pair<double, uint64_t>>> prof_acc;
  std::string last_error;
  std::vector<void*> allocs;
};

// ---------------------------------------------------------------- helpers
static het_status_t fail(het_cache* h, het_status_t st, const std::string& msg) {
  if (h) h->last_error = msg;
  return st;
}

#define CUDA_TRY(h, x)                                                           \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess)                                                       \
      return fail((h), HET_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
static cudaError_t dalloc(het_cache* h, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e == cudaSuccess) h->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return e;
}

// Pointer kind, remembered for the last few pointers (a training loop passes
// the same buffers every step; under UVA a device range stays device memory
// and a host range host memory, so a reused address keeps its kind).
static bool is_device_ptr(const void* p) {
  if (!p) return false;
  struct Kind { const void* p; bool dev; };
  thread_local Kind seen[8] = {};
  thread_local int next = 0;
  for (const Kind& k : seen)
    if (k.p == p) return k.dev;
  cudaPointerAttributes a;
  bool dev = false;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) cudaGetLastError();
  else dev = a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
  seen[next] = Kind{p, dev};
  next = (next + 1) & 7;
  return dev;
}

static cudaEvent_t ev_get(het_cache* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Prof {
  het_cache* h;
  cudaStream_t st;
  ProfRec r{};
  Prof(het_cache* h_, const char* name, cudaStream_t s) : h(h_), st(s) {
    if (h->prof) {
      r.name = name;
      r.a = ev_get(h);
      r.b = ev_get(h);
      cudaEventRecord(r.a, st);
    }
  }
  ~Prof() {
    if (h->prof) {
      cudaEventRecord(r.b, st);
      h->prof_pending.push_back(r);
    }
  }
};

static int bits_for(uint64_t x) {  // bits needed to represent values in [0, x]
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

// ---------------------------------------------------------------- utility kernels
__global__ void k_read_global(Dev s, const int64_t* keys, int n, float* rows, uint32_t* cg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)n * s.D;
  for (int64_t j = i; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = j / s.D;
    int64_t row = keys[r] / s.world;
    if (rows) rows[j] = s.W[row * s.D + (j - r * s.D)];
  }
  for (int64_t r = i; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (cg) cg[r] = s.cg[keys[r] / s.world];
}

// explicit Evict(key) at N = 1: push if dirty, delete, free
__global__ void k_evict_keys_local(Dev s, Call c) {
  __shared__ int dpop[LFU_CB_MAX];
  dpop_init(dpop);
  __syncthreads();
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (!ctl->abort && u < ctl->U) {
    int64_t key = c.uniq[u];
    int32_t e = warp_find(s, key, lane);
    if (e >= 0) {
      uint32_t ecs = s.cs[e], ecc = s.cc[e];
      bool dirty = ecc > ecs;
      if (dirty) {
        float* Wr = s.W + key * s.D;
        const float* pr = s.p + (int64_t)e * s.D;
        for (uint32_t d = lane; d < s.D; d += 32) Wr[d] = __fadd_rn(Wr[d], pr[d]);
        if (lane == 0) { uint32_t g = s.cg[key]; s.cg[key] = g > ecc ? g : ecc; }
      }
      warp_erase(s, key, lane);
      if (lane == 0) {
        if (s.policy == 0) lfu_move(s, key, s.eprim[e], EP_FREE, dpop);
        unpin_count(s, s.eprim[e]);
        s.eprim[e] = EP_FREE;
        s.ekey[e] = -1;
        s.fstack[atomicAdd(&ctl->ftop, 1)] = e;
        atomicAdd(&s.cnt[C_EVICTIONS], 1ull);
        if (dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], 1ull);
      }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
}

// het_sync at N = 1: every dirty entry pushes (distinct keys: order-free)
__global__ void k_flush_local(Dev s) {
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t e = w; e < s.Ecap; e += nw) {
    int64_t key = s.ekey[e];
    if (key < 0) continue;
    uint32_t ecs = s.cs[e], ecc = s.cc[e];
    if (ecc <= ecs) continue;
    float* Wr = s.W + key * s.D;
    const float* pr = s.p + e * s.D;
    for (uint32_t d = lane; d < s.D; d += 32) Wr[d] = __fadd_rn(Wr[d], pr[d]);
    if (lane == 0) { uint32_t g = s.cg[key]; s.cg[key] = g > ecc ? g : ecc; }
  }
}

__global__ void k_gather_entries(Dev s, const int32_t* idx, int m, float* v, float* p, uint32_t* cs,
                                 uint32_t* cc, uint32_t* prim) {
  int64_t total = (int64_t)m * s.D;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = j / s.D;
    int64_t e = idx[r];
    if (v) v[j] = s.v[e * s.D + (j - r * s.D)];
    if (p) p[j] = (s.cc[e] > s.cs[e]) ? s.p[e * s.D + (j - r * s.D)] : 0.0f;
  }
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = idx[r];
    if (cs) cs[r] = s.cs[e];
    if (cc) cc[r] = s.cc[e];
    if (prim) prim[r] = s.eprim[e];
  }
}

__global__ void k_scale(float* buf, uint64_t count, float f) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = __fmul_rn(buf[i], f);
}

// ---------------------------------------------------------------- C-ABI
extern "C" {

het_status_t het_get_unique_id(void* out128) {
  if (!out128) return HET_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return HET_ERR_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return HET_OK;
}

static constexpr uint64_t DENSE_DEFAULT = 1ull << 22;   // floats of dense all-reduce staging by default

// one worker; world > 1 with uid == nullptr: a loopback member (het_group_create)
static het_status_t create_impl(uint64_t rows, uint32_t D, double cache_frac, uint32_t s, het_policy_t policy,
                                int rank, int world, const void* uid, const het_opts_t* opt, cudaStream_t stream,
                                het_cache_t* out) {
  *out = nullptr;
  if (rows == 0 || rows > (1ull << 32) || D == 0 || (D % 4) != 0 || D > (1u << 16)) return HET_ERR_ARG;
  if (!(cache_frac >= 0.0 && cache_frac <= 1.0)) return HET_ERR_ARG;
  if (policy != HET_LFU && policy != HET_LRU && policy != HET_LIGHT_LFU) return HET_ERR_ARG;
  if (world < 1 || rank < 0 || rank >= world) return HET_ERR_ARG;
  het_cache* h = new het_cache();
  h->no_fused = std::getenv("HET_NO_FUSED") != nullptr;
  h->R = rows;
  h->D = D;
  h->C = (int64_t)std::floor(cache_frac * (double)rows);  // R10
  h->n_max = opt && opt->max_keys_per_call ? opt->max_keys_per_call : 65536;
  if (h->n_max > (1u << 24)) { delete h; return HET_ERR_ARG; }
  h->pbits = std::max(1, bits_for(h->n_max - 1));
  Dev& d = h->d;
  d.R = (int64_t)rows;
  d.D = D;
  d.C = h->C;
  d.s = s;
  d.policy = policy == HET_LRU ? 1 : 0;   // light-LFU is LFU plus pinning (R27)
  d.pin_thr = policy == HET_LIGHT_LFU ? ((opt && opt->pin_threshold) ? opt->pin_threshold : 64u) : 0u;
  d.pin_max = h->C / 2;
  d.lfu_persist = opt ? (opt->lfu_persist != 0) : 1;
  if (!opt) d.lfu_persist = 1;
  d.rank = rank;
  d.world = world;
  d.seed0 = (opt && opt->init_seed) ? opt->init_seed : 2112072210ull;
  d.kbits = std::max(1, bits_for(rows - 1));
  d.rows_local = ((int64_t)rows - rank + world - 1) / world;
  d.Ecap = h->C + 2 * (int64_t)h->n_max;
  int64_t S = 64;
  d.hbits = 6;
  while (S < 4 * d.Ecap) { S <<= 1; d.hbits++; }
  d.hmask = (uint64_t)S - 1;

  int prio_lo = 0, prio_hi = 0;   // heavy-key work on the side stream is scheduled first
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rows_free, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rows_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->ustream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_lk_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_upd_done, cudaEventDisableTiming) != cudaSuccess) {
    het_cache_destroy(h);
    return HET_ERR_CUDA;
  }
  het_status_t rc = HET_OK;
#define A(ptr, cnt)                                              \
  if (dalloc(h, &(ptr), (cnt)) != cudaSuccess) { rc = HET_ERR_OOM; goto oom; }
  A(d.W, (size_t)d.rows_local * D);
  A(d.cg, d.rows_local);
  A(d.ekey, d.Ecap);
  A(d.v, (size_t)d.Ecap * D);
  A(d.p, (size_t)d.Ecap * D);
  A(d.cs, d.Ecap);
  A(d.cc, d.Ecap);
  A(d.eprim, d.Ecap);
  A(d.estep, d.Ecap);
  A(d.fstack, d.Ecap);
  A(d.hslot, (size_t)S);
  A(d.count_by_key, d.lfu_persist ? rows : 1);
  d.bm_words = ((int64_t)rows + 31) / 32;
  d.nbk = ((int64_t)rows + (1 << LFU_BLK_SHIFT) - 1) >> LFU_BLK_SHIFT;
  d.nbk2 = (d.nbk + 63) >> 6;
  d.lfu_cb = 0;
  if (policy != HET_LRU) {  // count bitmaps, bounded to ~1 GB
    int cb = LFU_CB_MAX;
    while (cb > 2 && (double)cb * d.bm_words * 4 > 1.0e9) cb >>= 1;
    d.lfu_cb = cb;
    if (const char* env = std::getenv("HET_LFU_CB"))  // test knob: shrink the bitmap window
      d.lfu_cb = std::max(0, std::min(atoi(env), d.lfu_cb));
  }
  A(d.bm, d.lfu_cb ? (size_t)d.lfu_cb * d.bm_words : 1);
  A(d.bcnt, d.lfu_cb ? (size_t)d.lfu_cb * d.nbk : 1);
  A(d.bcnt2, d.lfu_cb ? (size_t)d.lfu_cb * d.nbk2 : 1);
  A(d.pop, LFU_CB_MAX);
  A(d.ctl, 1);
  A(d.cnt, C_NUM);
  A(d.pin_k, d.pin_thr ? h->n_max : 1);
  A(d.pin_e, d.pin_thr ? h->n_max : 1);
  {
    Call& c = h->call;
    uint32_t nm = h->n_max;
    A(c.uniq, nm);
    A(c.inverse, nm);
    A(c.perm, nm);
    A(c.seg_off, nm + 1);
    A(c.status, nm);
    A(c.uentry, nm);
    A(c.sortbuf0, nm);
    A(c.sortbuf1, nm);
    A(c.blockbuf, nm / 1024 + 2);
    A(c.hlist, nm);
    A(c.urec, nm);
    A(c.upos, nm);
    A(c.ucnt, nm);
    A(c.ucslot, nm);
    A(c.pref_bad, 1);
    A(h->sb_alt, nm);
    A(h->perm_alt, nm);
    A(c.ucword, nm);
    A(c.dbg_status, nm);
    A(c.dbg_inverse, nm);
    A(c.dbg_U, 1);
    c.pbits = h->pbits;
    A(c.hbuf, (size_t)nm * ((D + 15) / 16) * 16);
    c.hcap = (int)nm;
    uint32_t *hist, *khist;
    int32_t *cand, *sub, *flags;
    A(hist, 2048);
    A(khist, 2048);
    A(h->victims, 2 * (size_t)nm + 1);
    A(h->victim_keys, 2 * (size_t)nm + 1);
    A(h->victim_dirty, 2 * (size_t)nm + 1);
    A(h->victim_sel, 2 * (size_t)nm + 1);
    A(cand, d.Ecap);
    A(sub, d.Ecap);
    A(flags, 4);
    h->evbuf_host = std::malloc(evbuf_struct_size());
    evbuf_init(h->evbuf_host, hist, khist, h->victims, cand, sub, flags, h->victim_keys, h->victim_dirty,
               h->victim_sel);
    cudaMemsetAsync(hist, 0, 2048 * 4, stream);
    cudaMemsetAsync(khist, 0, 2048 * 4, stream);
    cudaMemsetAsync(flags, 0, 16, stream);
  }
#undef A
  dedup_set_attrs();
  cache_set_attrs();
  cudaMemsetAsync(d.ctl, 0, sizeof(Ctl), stream);
  cudaMemsetAsync(d.cnt, 0, C_NUM * 8, stream);
  cudaMemsetAsync(d.estep, 0, d.Ecap * 4, stream);
  if (d.lfu_persist) cudaMemsetAsync(d.count_by_key, 0, rows * 4, stream);
  cudaMemsetAsync(d.cs, 0, d.Ecap * 4, stream);
  cudaMemsetAsync(d.cc, 0, d.Ecap * 4, stream);
  launch_init_shard(d, stream);
  if (d.lfu_cb) {
    cudaMemsetAsync(d.bm, 0, (size_t)d.lfu_cb * d.bm_words * 4, stream);
    cudaMemsetAsync(d.bcnt, 0, (size_t)d.lfu_cb * d.nbk * 4, stream);
    cudaMemsetAsync(d.bcnt2, 0, (size_t)d.lfu_cb * d.nbk2 * 4, stream);
  }
  cudaMemsetAsync(d.pop, 0, LFU_CB_MAX * 4, stream);
  launch_reset_cache(d, stream);
  if (world > 1) {
    rc = mgpu_create(h->mg, d, h->n_max, uid, (opt && opt->dense_max) ? opt->dense_max : DENSE_DEFAULT, stream);
    if (rc != HET_OK) goto oom;
  }
  if (cudaStreamSynchronize(stream) != cudaSuccess) { rc = HET_ERR_CUDA; goto oom; }
  *out = h;
  return HET_OK;
oom:
  cudaGetLastError();
  for (void* q : h->allocs) cudaFree(q);
  if (h->mg) mgpu_destroy(h->mg);
  std::free(h->evbuf_host);
  delete h;
  return rc;
}

het_status_t het_cache_create(uint64_t rows, uint32_t D, double cache_frac, uint32_t s,
                              het_policy_t policy, const het_dist_t* dist, const het_opts_t* opt,
                              het_stream_t stream_, het_cache_t* out) {
  if (!out) return HET_ERR_ARG;
  *out = nullptr;
  int rank = 0, world = 1;
  const void* uid = nullptr;
  if (dist) {
    rank = dist->rank;
    world = dist->world;
    uid = dist->nccl_unique_id;
    if (world > 1 && !uid) return HET_ERR_ARG;
  }
  return create_impl(rows, D, cache_frac, s, policy, rank, world, uid, opt, (cudaStream_t)stream_, out);
}

het_status_t het_group_create(uint32_t N, uint64_t rows, uint32_t D, double cache_frac, uint32_t s,
                              het_policy_t policy, const het_opts_t* opt, het_stream_t stream_,
                              het_cache_t* out) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!out || N < 2 || N > 16) return HET_ERR_ARG;
  for (uint32_t r = 0; r < N; ++r) out[r] = nullptr;
  auto g = std::make_shared<het_group>();
  het_status_t rc = HET_OK;
  for (uint32_t r = 0; r < N && rc == HET_OK; ++r) {
    rc = create_impl(rows, D, cache_frac, s, policy, (int)r, (int)N, nullptr, opt, st, &out[r]);
    if (rc == HET_OK) g->m.push_back(out[r]);
  }
  if (rc == HET_OK) {
    std::vector<P2PState*> ps(N);
    for (uint32_t r = 0; r < N; ++r) ps[r] = mgpu_p2p(out[r]->mg);
    rc = p2p_loopback_connect(ps.data(), (int)N, st);
  }
  if (rc != HET_OK) {
    for (uint32_t r = 0; r < N; ++r) {
      if (out[r]) het_cache_destroy(out[r]);
      out[r] = nullptr;
    }
    return rc;
  }
  for (uint32_t r = 0; r < N; ++r) out[r]->group = g;
  return HET_OK;
}

static het_status_t stage_keys(het_cache* h, const int64_t*& keys, uint32_t n, cudaStream_t st) {
  if (n == 0 || is_device_ptr(keys)) return HET_OK;
  if (!h->stage_keys) CUDA_TRY(h, (dalloc(h, &h->stage_keys, h->n_max)));
  CUDA_TRY(h, cudaMemcpyAsync(h->stage_keys, keys, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  keys = h->stage_keys;
  return HET_OK;
}

// ---------------------------------------------------------------- members of a collective call
// One process per GPU: the call drives its own worker, every phase back to
// back (peers are other processes).  Loopback group: the call drives all N
// workers, phase k of every worker before phase k+1 of any.
struct Members {
  het_cache* const* hs;
  int n;
};
static P2PState* p2p_of(het_cache* h) { return mgpu_p2p(h->mg); }
static const void* p2p_view(het_cache* h) { return h->d.world > 1 ? (const void*)p2p_view_ptr(p2p_of(h)) : nullptr; }

// the overflow eviction the last fused update deferred (its victims are
// listed): run it before anything that reads or changes the cache
// (inspection calls -- het_stats, het_check, het_debug_* -- pass count =
// false: the launch counter reports the hot path's kernels)
static void flush_evict(het_cache* h, cudaStream_t st, bool count = true) {
  h->lk_done_valid = false;   // another call between the lookup and the update: the update stays on the stream
  // after a captured update, any graph replay may have listed victims: the
  // kernel tests the device flag (cheap when nothing is listed)
  if (!h->ev_pending && !h->ev_captured) return;
  const int l = launch_evict_pending(h->d, h->evbuf_host, p2p_view(h), st);
  if (count) h->launches += l;
  h->ev_pending = false;
}

static het_status_t check_members(het_cache* const* hs, uint32_t N) {
  if (!hs || N < 2 || !hs[0] || !hs[0]->group) return HET_ERR_ARG;
  const auto& m = hs[0]->group->m;
  if (m.size() != N) return HET_ERR_ARG;
  for (uint32_t i = 0; i < N; ++i)
    if (hs[i] != m[i]) return HET_ERR_ARG;   // every member, in rank order
  return HET_OK;
}

// a round of the peer-memory exchange carrying only the pending pushes
static void drain_round(Members g, cudaStream_t st) {
  for (int ph = 0; ph < RP_NUM; ++ph)
    for (int i = 0; i < g.n; ++i) {
      het_cache* h = g.hs[i];
      Prof p(h, "drain", st);
      h->launches += p2p_round_phase(p2p_of(h), h->d, h->call, 1, ph, st);
    }
}

// ---------------------------------------------------------------- lookup
struct LkCtx {
  float* out = nullptr;    // caller's
  float* dout = nullptr;   // device destination
  bool out_host = false;
};

// argument checks, staging, dedup (K1) and the per-call begin
static het_status_t lookup_pre(het_cache* h, const int64_t* keys, uint32_t n, uint64_t clock_t, float* out,
                               LkCtx& x, cudaStream_t st) {
  if (n > h->n_max) return fail(h, HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  if (n && (!keys || !out)) return fail(h, HET_ERR_ARG, "null keys/out");
  if (h->overflow_bound + (int64_t)n > 2 * (int64_t)h->n_max)
    return fail(h, HET_ERR_CAPACITY, "too many lookups without eviction");
  const int64_t* ukeys = keys;
  het_status_t rc = stage_keys(h, keys, n, st);
  if (rc) return rc;
  x.out = out;
  x.out_host = n && !is_device_ptr(out);
  x.dout = out;
  if (x.out_host) {
    if (!h->stage_out) CUDA_TRY(h, (dalloc(h, &h->stage_out, (size_t)h->n_max * h->D)));
    x.dout = h->stage_out;
  }
  Call& c = h->call;
  c.n = (int)n;
  c.t = clock_t;
  c.keys = keys;
  h->last_keys = ukeys;
  Dev& d = h->d;
  // fused path: N = 1 up to FUSED_LOOKUP_MAX keys (beyond, the large-batch
  // per-phase kernels with the sliced heavy-key segment reduce), N > 1 over
  // the peer-memory exchange for every n; the dedup kernel follows n
  h->fused = !h->no_fused && (d.world == 1 ? (int)n <= FUSED_LOOKUP_MAX : mgpu_p2p(h->mg) != nullptr);
  // after the fused dedups: per-key work indexed by sorted position (no compaction pass, R29)
  c.rmode = (h->fused && (int)n <= RMODE_MAX) ? 1 : 0;
  const bool pref = c.rmode && h->pref_keys && ukeys == h->pref_keys && n == h->pref_n;
  h->pref_keys = nullptr;   // consumed, or not the keys it was for
  if (c.rmode) {   // the dedup kernel also runs the deferred eviction
    // a captured graph replays after its own update: keep the eviction blocks
    // (they test the device flag and return when nothing is listed)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    const bool ev = h->ev_pending || cap == cudaStreamCaptureStatusActive;
    Prof p(h, "dedup", st);
    if (pref) {   // het_prefetch ran this dedup: take its buffers, begin + evict only
      std::swap(c.sortbuf0, h->sb_alt);
      std::swap(c.perm, h->perm_alt);
      h->launches += launch_begin_evict(d, c, (int)n, clock_t, st, h->evbuf_host, p2p_view(h), ev);
    } else if (fused_ok(d, (int)n))
      h->launches += launch_dd_fused(d, c, (int)n, h->pbits, clock_t, 1, st, h->evbuf_host, p2p_view(h), ev, 0);
    else
      h->launches += launch_dd_bucket(d, c, (int)n, h->pbits, clock_t, 1, st, h->evbuf_host, p2p_view(h), ev);
    h->ev_pending = false;
  } else {
    flush_evict(h, st);
    launch_begin(d, clock_t, (int)n, st);
    Prof p(h, "dedup", st);
    h->launches += 1 + launch_dedup(c, (int)n, d.R, h->pbits, d.ctl, st);
  }
  return HET_OK;
}

// one process per GPU: the rest of Alg. 2 (probe, CheckValid, sync/fetch, Get)
static het_status_t lookup_body(het_cache* h, LkCtx& x, cudaStream_t st) {
  Dev& d = h->d;
  Call& c = h->call;
  if (h->fused) {
    if (d.world == 1) {
      h->launches += launch_lookup_fused(d, c, x.dout, st, h);   // records its phases when profiling
    } else {
      Prof p(h, "exchange_fused", st);
      h->launches += p2p_round_fused(p2p_of(h), d, c, x.dout, st);
    }
    return HET_OK;
  }
  if (d.world == 1) {
    {
      Prof p(h, "probe", st);
      launch_probe(d, c, c.n, st);
    }
    {
      Prof p(h, "sync_fetch", st);
      launch_sync_fetch_install_local(d, c, c.n, st);
    }
    h->launches += 2;
  } else {
    het_status_t rc = mgpu_lookup(h->mg, d, c, h->prof ? (void*)h : nullptr, st);
    if (rc) return fail(h, rc, "multi-GPU lookup failed");
    h->launches += mgpu_take_launches(h->mg);
  }
  Prof p(h, "gather", st);
  launch_gather(d, c, x.dout, st);
  h->launches += 1;
  return HET_OK;
}

// loopback: phase `ph` of the exchange round of one member
static void lookup_phase(het_cache* h, LkCtx& x, int ph, cudaStream_t st) {
  Dev& d = h->d;
  Call& c = h->call;
  P2PState* p = p2p_of(h);
  if (h->fused) {
    Prof pr(h, "exchange_fused", st);
    h->launches += p2p_lookup_phase(p, d, c, x.dout, ph, st);
    return;
  }
  if (ph == RP_BUILD) {
    Prof pr(h, "probe", st);
    launch_probe(d, c, c.n, st);
    h->launches += 1;
  }
  {
    Prof pr(h, "exchange", st);
    h->launches += p2p_round_phase(p, d, c, 0, ph, st);
  }
  if (ph == RP_INSTALL) {
    Prof pr(h, "gather", st);
    launch_gather(d, c, x.dout, st);
    h->launches += 1;
  }
}

static het_status_t lookup_post(het_cache* h, LkCtx& x, cudaStream_t st) {
  Dev& d = h->d;
  const uint32_t n = (uint32_t)h->call.n;
  // light-LFU promotions of this lookup (the fused N = 1 lookup kernels apply them in their last block)
  if (d.pin_thr && !(h->fused && d.world == 1)) h->launches += launch_pin_apply(d, st);
  h->lk_done_valid = false;
  if (x.out_host) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (cap == cudaStreamCaptureStatusNone && h->fused && d.world == 1 && !h->group) {
      CUDA_TRY(h, cudaEventRecord(h->ev_lk_done, st));   // the lookup's kernels, before the rows' D2H
      h->lk_done_valid = true;
    }
    CUDA_TRY(h, cudaMemcpyAsync(x.out, x.dout, (size_t)n * h->D * 4, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(h, cudaGetLastError());
  h->have_lookup = true;
  h->last_n = n;
  h->overflow_bound += n;
  return HET_OK;
}

// NEXT-1 ("pre-fetch the next mini-batch of data in advance"): the
// dedup of the next lookup's keys, enqueued now (e.g. on a side stream while
// the dense backward and het_update run) into the alternate buffers; the next
// het_lookup with the same pointer and n skips its dedup.  The dedup is a
// function of the keys alone, so results are unchanged.
het_status_t het_prefetch(het_cache_t h, const int64_t* keys, uint32_t n, het_stream_t stream_) {
  NvtxRange nvtx_("het_prefetch");
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (n > h->n_max) return fail(h, HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  if (n && !keys) return fail(h, HET_ERR_ARG, "null keys");
  h->lk_done_valid = false;
  h->pref_keys = nullptr;
  if (h->no_fused || n == 0 || (int)n > RMODE_MAX) return HET_OK;   // nothing to run ahead on this path
  const int64_t* dkeys = keys;
  if (!is_device_ptr(keys)) {
    if (!h->stage_pref) CUDA_TRY(h, (dalloc(h, &h->stage_pref, h->n_max)));
    CUDA_TRY(h, cudaMemcpyAsync(h->stage_pref, keys, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    dkeys = h->stage_pref;
  }
  Call pc = h->call;   // the alternate buffers; nothing else of the call is written
  pc.keys = dkeys;
  pc.n = (int)n;
  pc.sortbuf0 = h->sb_alt;
  pc.perm = h->perm_alt;
  pc.rmode = 1;
  Dev& d = h->d;
  if (fused_ok(d, (int)n))
    h->launches += launch_dd_fused(d, pc, (int)n, h->pbits, 0, 2, st, h->evbuf_host, p2p_view(h), false, 0);
  else
    h->launches += launch_dd_bucket(d, pc, (int)n, h->pbits, 0, 2, st, h->evbuf_host, p2p_view(h), false);
  CUDA_TRY(h, cudaGetLastError());
  h->pref_keys = keys;
  h->pref_n = n;
  return HET_OK;
}

het_status_t het_lookup(het_cache_t h, const int64_t* keys, uint32_t n, uint64_t clock_t, float* out,
                        het_stream_t stream_) {
  NvtxRange nvtx_("het_lookup");
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (h->group) return fail(h, HET_ERR_PROTOCOL, "loopback workers are driven by het_group_lookup");
  LkCtx x;
  het_status_t rc = lookup_pre(h, keys, n, clock_t, out, x, st);
  if (rc == HET_OK) rc = lookup_body(h, x, st);
  if (rc == HET_OK) rc = lookup_post(h, x, st);
  return rc;
}

het_status_t het_group_lookup(const het_cache_t* hs, uint32_t N, const int64_t* const* keys, const uint32_t* n,
                              uint64_t clock_t, float* const* out, het_stream_t stream_) {
  NvtxRange nvtx_("het_group_lookup");
  cudaStream_t st = (cudaStream_t)stream_;
  if (check_members(hs, N) || !keys || !n || !out) return HET_ERR_ARG;
  std::vector<LkCtx> x(N);
  for (uint32_t i = 0; i < N; ++i)
    if (n[i] > hs[i]->n_max || hs[i]->overflow_bound + (int64_t)n[i] > 2 * (int64_t)hs[i]->n_max)
      return fail(hs[i], HET_ERR_CAPACITY, "n exceeds max_keys_per_call / too many lookups without eviction");
  for (uint32_t i = 0; i < N; ++i) {
    het_status_t rc = lookup_pre(hs[i], keys[i], n[i], clock_t, out[i], x[i], st);
    if (rc) return rc;
  }
  for (int ph = 0; ph < RP_NUM; ++ph)
    for (uint32_t i = 0; i < N; ++i) lookup_phase(hs[i], x[i], ph, st);
  for (uint32_t i = 0; i < N; ++i) {
    het_status_t rc = lookup_post(hs[i], x[i], st);
    if (rc) return rc;
  }
  return HET_OK;
}

// ---------------------------------------------------------------- update
static het_status_t evict_overflow(het_cache* h, cudaStream_t st) {
  Dev& d = h->d;
  if (d.world == 1) {
    {
      Prof p(h, "evict_select", st);
      h->launches += launch_evict_select(d, h->evbuf_host, st);
    }
    Prof p(h, "evict_apply", st);
    h->launches += launch_evict_apply_local(d, h->evbuf_host, st);
  } else {
    // select + PUSH records into the owners' inboxes (carried by the next round: no wait)
    het_status_t rc = mgpu_evict_overflow(h->mg, d, h->evbuf_host, h->prof ? (void*)h : nullptr, st);
    if (rc) return rc;
    h->launches += mgpu_take_launches(h->mg);
  }
  h->overflow_bound = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (cap == cudaStreamCaptureStatusActive || (++h->updates & 63) == 0) {
    launch_hash_rebuild(d, st);  // a captured graph re-checks every step
    h->launches += 2;
  }
  return HET_OK;
}

// Alg. 3 writes the keys Alg. 2 read: same n, and a buffer other
// than the lookup's is compared on the device, position by position, with the
// lookup's dedup (keys[pos] == unique[inverse[pos]]); a mismatch latches
// HET_ERR_PROTOCOL and aborts the update before it touches the cache.
__global__ void k_check_keys(const int64_t* __restrict__ keys, int n, Call c, Ctl* ctl) {
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bad |= keys[i] != (c.rmode ? (int64_t)(c.sortbuf0[c.inverse[i]] >> c.pbits) : c.uniq[c.inverse[i]]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) raise_err(ctl, 3 /*HET_ERR_PROTOCOL*/);
}

static het_status_t update_impl(het_cache* h, const int64_t* keys, uint32_t n, const float* grads, float lr,
                                cudaStream_t st) {
  if (!h->have_lookup || n != h->last_n) return fail(h, HET_ERR_PROTOCOL, "write without matching read");
  if (n && (!grads || !keys)) return fail(h, HET_ERR_ARG, "null keys/grads");
  Dev& d = h->d;
  if (n && keys != h->last_keys) {
    het_status_t rc = stage_keys(h, keys, n, st);
    if (rc) return rc;
    k_check_keys<<<std::min<int>(148, (n + 255) / 256), 256, 0, st>>>(keys, (int)n, h->call, d.ctl);
    h->launches += 1;
  }
  bool staged = false;
  // beside the lookup's D2H: host gradients, the lookup's own keys, no call in
  // between (the update then reads only the staged rows and library state)
  const bool beside = h->lk_done_valid && n && keys == h->last_keys && h->fused && !is_device_ptr(grads);
  h->lk_done_valid = false;
  cudaStream_t caller = st;
  if (n && !is_device_ptr(grads)) {
    if (!h->stage_rows) CUDA_TRY(h, (dalloc(h, &h->stage_rows, (size_t)h->n_max * h->D)));
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (cap == cudaStreamCaptureStatusNone) {   // H2D on the copy stream, beside the lookup's work
      CUDA_TRY(h, cudaStreamWaitEvent(h->copy, h->ev_rows_free, 0));
      CUDA_TRY(h, cudaMemcpyAsync(h->stage_rows, grads, (size_t)n * h->D * 4, cudaMemcpyHostToDevice, h->copy));
      CUDA_TRY(h, cudaEventRecord(h->ev_rows_ready, h->copy));
      if (beside) {
        st = h->ustream;
        CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_lk_done, 0));
      }
      CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_rows_ready, 0));
      staged = true;
    } else {
      CUDA_TRY(h, cudaMemcpyAsync(h->stage_rows, grads, (size_t)n * h->D * 4, cudaMemcpyHostToDevice, st));
    }
    grads = h->stage_rows;
  }
  if (h->fused) {
    h->launches += launch_update_fused(d, h->call, grads, lr, h->evbuf_host, st, p2p_view(h), h);
    h->overflow_bound = 0;
    h->ev_pending = true;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (cap == cudaStreamCaptureStatusActive) h->ev_captured = true;
  } else {
    {
      Prof p(h, "segreduce_apply", st);
      h->launches += launch_segreduce_apply(d, h->call, grads, lr, (int)n, st, h->side, h->ev_fork, h->ev_join);
    }
    het_status_t rc = evict_overflow(h, st);
    if (rc) return fail(h, rc, "evict failed");
  }
  if (staged) CUDA_TRY(h, cudaEventRecord(h->ev_rows_free, st));   // the staging buffer is read by now
  if (st != caller) {   // the caller's stream continues after this update
    CUDA_TRY(h, cudaEventRecord(h->ev_upd_done, st));
    CUDA_TRY(h, cudaStreamWaitEvent(caller, h->ev_upd_done, 0));
  }
  CUDA_TRY(h, cudaGetLastError());
  h->have_lookup = false;
  return HET_OK;
}

het_status_t het_update(het_cache_t h, const int64_t* keys, uint32_t n, const float* grads, float lr,
                        het_stream_t stream_) {
  NvtxRange nvtx_("het_update");
  if (!h) return HET_ERR_ARG;
  if (h->group) return fail(h, HET_ERR_PROTOCOL, "loopback workers are driven by het_group_update");
  return update_impl(h, keys, n, grads, lr, (cudaStream_t)stream_);
}

het_status_t het_group_update(const het_cache_t* hs, uint32_t N, const int64_t* const* keys, const uint32_t* n,
                              const float* const* grads, float lr, het_stream_t stream_) {
  NvtxRange nvtx_("het_group_update");
  if (check_members(hs, N) || !keys || !n || !grads) return HET_ERR_ARG;
  for (uint32_t i = 0; i < N; ++i)   // no partial group update on a synchronous error
    if (!hs[i]->have_lookup || n[i] != hs[i]->last_n)
      return fail(hs[i], HET_ERR_PROTOCOL, "write without matching read");
  for (uint32_t i = 0; i < N; ++i) {   // pushes go to the owners' inboxes: no cross-worker wait
    het_status_t rc = update_impl(hs[i], keys[i], n[i], grads[i], lr, (cudaStream_t)stream_);
    if (rc) return rc;
  }
  return HET_OK;
}

// ---------------------------------------------------------------- evict
static het_status_t evict_keys_pre(het_cache* h, const int64_t* keys, uint32_t n, cudaStream_t st) {
  h->lk_done_valid = false;
  if (n > h->n_max) return fail(h, HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  het_status_t rc = stage_keys(h, keys, n, st);
  if (rc) return rc;
  Call& c = h->call;
  c.n = (int)n;
  c.keys = keys;
  c.rmode = 0;
  cudaMemsetAsync(&h->d.ctl->abort, 0, 4, st);
  h->launches += launch_dedup(c, (int)n, h->d.R, h->pbits, h->d.ctl, st);
  return HET_OK;
}

// keys == nullptr: overflow Evict() (no cross-worker wait); else Cache.Evict(key)
static het_status_t evict_members(Members g, const int64_t* const* keys, const uint32_t* n, cudaStream_t st) {
  for (int i = 0; i < g.n; ++i) flush_evict(g.hs[i], st);
  if (!keys) {
    for (int i = 0; i < g.n; ++i) {
      het_status_t rc = evict_overflow(g.hs[i], st);
      if (rc) return fail(g.hs[i], rc, "evict failed");
    }
    return HET_OK;
  }
  het_cache* h0 = g.hs[0];
  if (h0->d.world == 1) {
    het_status_t rc = evict_keys_pre(h0, keys[0], n[0], st);
    if (rc) return rc;
    k_evict_keys_local<<<std::max(1, ((int)n[0] + 7) / 8), 256, 0, st>>>(h0->d, h0->call);
    h0->launches += 1;
  } else if (!p2p_of(h0)) {   // NCCL exchange (HET_P2P=0)
    het_status_t rc = evict_keys_pre(h0, keys[0], n[0], st);
    if (rc) return rc;
    rc = mgpu_evict_keys(h0->mg, h0->d, h0->call, st);
    if (rc) return fail(h0, rc, "multi-GPU evict failed");
    h0->launches += mgpu_take_launches(h0->mg);
  } else {
    drain_round(g, st);   // the pushes of the last update precede (U4 before this Evict)
    for (int i = 0; i < g.n; ++i) {
      het_status_t rc = evict_keys_pre(g.hs[i], keys[i], n[i], st);
      if (rc) return rc;
      g.hs[i]->launches += p2p_evict_keys(p2p_of(g.hs[i]), g.hs[i]->d, g.hs[i]->call, st);
    }
    drain_round(g, st);
  }
  for (int i = 0; i < g.n; ++i) {
    g.hs[i]->have_lookup = false;
    CUDA_TRY(g.hs[i], cudaGetLastError());
  }
  return HET_OK;
}

het_status_t het_evict(het_cache_t h, const int64_t* keys, uint32_t n, het_stream_t stream_) {
  NvtxRange nvtx_("het_evict");
  if (!h) return HET_ERR_ARG;
  if (h->group) return fail(h, HET_ERR_PROTOCOL, "loopback workers are driven by het_group_evict");
  het_cache* one[1] = {h};
  const int64_t* k1[1] = {keys};
  return evict_members(Members{one, 1}, keys ? k1 : nullptr, &n, (cudaStream_t)stream_);
}

het_status_t het_group_evict(const het_cache_t* hs, uint32_t N, const int64_t* const* keys, const uint32_t* n,
                             het_stream_t stream_) {
  NvtxRange nvtx_("het_group_evict");
  if (check_members(hs, N) || (keys && !n)) return HET_ERR_ARG;
  if (keys)
    for (uint32_t i = 0; i < N; ++i)
      if (n[i] > hs[i]->n_max) return fail(hs[i], HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  return evict_members(Members{hs, (int)N}, keys, n, (cudaStream_t)stream_);
}

// ---------------------------------------------------------------- sync (flush)
static het_status_t sticky(het_cache* h, cudaStream_t st) {
  Ctl ctl;
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (ctl.err) return fail(h, (het_status_t)ctl.err, "sticky device error");
  if (h->mg && mgpu_comm_error(h->mg)) return fail(h, HET_ERR_NCCL, "NCCL asynchronous error");
  return HET_OK;
}

// het_sync over the peer-memory exchange: dirty entries of key range [k0, k1)
// in rounds of whole key bins (a key's pushes from every worker meet at the
// owner in one round, applied in source-rank order, R1), each round at most
// CAPS records per source; a bin too large for one round is split again.
static het_status_t flush_range(Members g, int64_t k0, int64_t k1, cudaStream_t st) {
  std::vector<int32_t> bins(FBINS, 0), mine(FBINS);
  for (int i = 0; i < g.n; ++i) {
    het_cache* h = g.hs[i];
    het_status_t rc = mgpu_flush_hist(h->mg, h->d, k0, k1, mine.data(), st);
    if (rc) return fail(h, rc, "flush histogram failed");
    h->launches += mgpu_take_launches(h->mg);
    for (int b = 0; b < FBINS; ++b) bins[b] = std::max(bins[b], mine[b]);
  }
  if (g.n == 1) {   // one process per GPU: the max over the ranks
    het_status_t rc = mgpu_allreduce_max_host(g.hs[0]->mg, bins.data(), FBINS, st);
    if (rc) return fail(g.hs[0], rc, "flush histogram all-reduce failed");
  }
  const int64_t caps = p2p_caps(p2p_of(g.hs[0]));
  const int64_t W = k1 - k0;
  auto kb = [&](int b) { return k0 + ((int64_t)b * W + FBINS - 1) / FBINS; };   // first key of bin b
  int b0 = 0;
  while (b0 < FBINS) {
    if (bins[b0] > caps) {   // one bin over capacity: split it (its keys >= its dirty count per worker)
      het_status_t rc = flush_range(g, kb(b0), kb(b0 + 1), st);
      if (rc) return rc;
      ++b0;
      continue;
    }
    int64_t acc = 0;
    int b1 = b0;
    while (b1 < FBINS && bins[b1] <= caps && acc + bins[b1] <= caps) acc += bins[b1++];
    if (acc > 0) {
      for (int i = 0; i < g.n; ++i)
        g.hs[i]->launches += p2p_flush_build(p2p_of(g.hs[i]), g.hs[i]->d, kb(b0), kb(b1), st);
      drain_round(g, st);
    }
    b0 = b1;
  }
  return HET_OK;
}

static het_status_t sync_members(Members g, cudaStream_t st) {
  for (int i = 0; i < g.n; ++i) flush_evict(g.hs[i], st);
  het_cache* h0 = g.hs[0];
  if (h0->d.world == 1) {
    k_flush_local<<<148 * 4, 256, 0, st>>>(h0->d);
    h0->launches += 1;
  } else if (!p2p_of(h0)) {   // NCCL exchange (HET_P2P=0)
    het_status_t rc = mgpu_flush(h0->mg, h0->d, st);
    if (rc) return fail(h0, rc, "multi-GPU flush failed");
    h0->launches += mgpu_take_launches(h0->mg);
  } else {
    drain_round(g, st);   // U4 of the last update precedes the flush
    het_status_t rc = flush_range(g, 0, (int64_t)h0->R, st);
    if (rc) return rc;
  }
  het_status_t first = HET_OK;
  for (int i = 0; i < g.n; ++i) {
    het_cache* h = g.hs[i];
    Dev& d = h->d;
    launch_reset_cache(d, st);
    h->launches += 1;
    if (d.lfu_cb) {
      cudaMemsetAsync(d.bm, 0, (size_t)d.lfu_cb * d.bm_words * 4, st);
      cudaMemsetAsync(d.bcnt, 0, (size_t)d.lfu_cb * d.nbk * 4, st);
      cudaMemsetAsync(d.bcnt2, 0, (size_t)d.lfu_cb * d.nbk2 * 4, st);
    }
    cudaMemsetAsync(d.pop, 0, LFU_CB_MAX * 4, st);
    h->have_lookup = false;
    h->overflow_bound = 0;
    CUDA_TRY(h, cudaGetLastError());
    het_status_t rc = sticky(h, st);
    if (rc && !first) first = rc;
  }
  return first;
}

het_status_t het_sync(het_cache_t h, het_stream_t stream_) {
  NvtxRange nvtx_("het_sync");
  if (!h) return HET_ERR_ARG;
  if (h->group) return fail(h, HET_ERR_PROTOCOL, "loopback workers are driven by het_group_sync");
  h->lk_done_valid = false;
  het_cache* one[1] = {h};
  return sync_members(Members{one, 1}, (cudaStream_t)stream_);
}

het_status_t het_group_sync(const het_cache_t* hs, uint32_t N, het_stream_t stream_) {
  NvtxRange nvtx_("het_group_sync");
  if (check_members(hs, N)) return HET_ERR_ARG;
  return sync_members(Members{hs, (int)N}, (cudaStream_t)stream_);
}

het_status_t het_check(het_cache_t h) {
  if (!h) return HET_ERR_ARG;
  flush_evict(h, 0, false);
  return sticky(h, 0);
}

het_status_t het_stats(het_cache_t h, het_stats_t* out) {
  if (!h || !out) return HET_ERR_ARG;
  unsigned long long cnt[C_NUM];
  Ctl ctl;
  CUDA_TRY(h, cudaDeviceSynchronize());
  flush_evict(h, 0, false);
  CUDA_TRY(h, cudaDeviceSynchronize());
  CUDA_TRY(h, cudaMemcpy(cnt, h->d.cnt, sizeof(cnt), cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemcpy(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  std::memset(out, 0, sizeof(*out));
  out->lookups = cnt[C_LOOKUPS];
  out->keys = cnt[C_KEYS];
  out->unique = cnt[C_UNIQUE];
  out->hits = cnt[C_HITS];
  out->exp1 = cnt[C_EXP1];
  out->exp2 = cnt[C_EXP2];
  out->misses = cnt[C_MISSES];
  out->evictions = cnt[C_EVICTIONS];
  out->dirty_pushes = cnt[C_DIRTY_PUSHES];
  if (h->mg) mgpu_bytes(h->mg, &out->bytes_clock_tx, &out->bytes_clock_rx, &out->bytes_emb_tx, &out->bytes_emb_rx);
  out->bytes_clock_tx += cnt[C_BCLK_TX];   // device-counted (peer-memory exchange)
  out->bytes_clock_rx += cnt[C_BCLK_RX];
  out->bytes_emb_tx += cnt[C_BEMB_TX];
  out->bytes_emb_rx += cnt[C_BEMB_RX];
  out->launches = h->launches;
  out->resident = (uint32_t)(h->d.Ecap - ctl.ftop);
  out->capacity = (uint32_t)h->C;
  out->sticky_error = ctl.err ? ctl.err : (h->mg && mgpu_comm_error(h->mg) ? HET_ERR_NCCL : 0);
  out->pinned = (uint32_t)ctl.npinned;
  return HET_OK;
}

het_status_t het_read_global(het_cache_t h, const int64_t* keys, uint32_t n, float* rows, uint32_t* cg,
                             het_stream_t stream_) {
  NvtxRange nvtx_("het_read_global");
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (n == 0) return HET_OK;
  if (!keys) return HET_ERR_ARG;
  flush_evict(h, st, false);
  std::vector<int64_t> hk(n);
  if (is_device_ptr(keys)) {
    CUDA_TRY(h, cudaMemcpyAsync(hk.data(), keys, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
  } else {
    std::memcpy(hk.data(), keys, (size_t)n * 8);
  }
  for (uint32_t i = 0; i < n; ++i)
    if (hk[i] < 0 || (uint64_t)hk[i] >= h->R || hk[i] % h->d.world != h->d.rank)
      return fail(h, HET_ERR_ARG, "read_global key not owned by this rank");
  int64_t* dk;
  float* drows = nullptr;
  uint32_t* dcg = nullptr;
  CUDA_TRY(h, cudaMallocAsync((void**)&dk, (size_t)n * 8, st));
  if (rows) CUDA_TRY(h, cudaMallocAsync((void**)&drows, (size_t)n * h->D * 4, st));
  if (cg) CUDA_TRY(h, cudaMallocAsync((void**)&dcg, (size_t)n * 4, st));
  CUDA_TRY(h, cudaMemcpyAsync(dk, hk.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
  k_read_global<<<256, 256, 0, st>>>(h->d, dk, (int)n, drows, dcg);
  if (rows) CUDA_TRY(h, cudaMemcpyAsync(rows, drows, (size_t)n * h->D * 4, cudaMemcpyDefault, st));
  if (cg) CUDA_TRY(h, cudaMemcpyAsync(cg, dcg, (size_t)n * 4, cudaMemcpyDefault, st));
  cudaFreeAsync(dk, st);
  if (drows) cudaFreeAsync(drows, st);
  if (dcg) cudaFreeAsync(dcg, st);
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return HET_OK;
}

// ---------------------------------------------------------------- dense all-reduce (Eq. 2)
het_status_t het_dense_allreduce(het_cache_t h, float* buf, uint64_t count, het_stream_t stream_) {
  NvtxRange nvtx_("het_dense_allreduce");
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (h->group) return fail(h, HET_ERR_PROTOCOL, "loopback workers are driven by het_group_dense_allreduce");
  if (count == 0 || h->d.world == 1) return HET_OK;
  if (!buf || !is_device_ptr(buf)) return fail(h, HET_ERR_ARG, "dense buffer must be device memory");
  Prof p(h, "dense_allreduce", st);
  int l = 0;
  het_status_t rc = mgpu_dense_p2p(h->mg, h->d, buf, count, 0, st, &l);   // peer-memory one-shot mean
  if (rc == HET_OK) {
    h->launches += l;
    return HET_OK;
  }
  if (rc != HET_ERR_CAPACITY) return fail(h, rc, "peer all-reduce failed");
  rc = mgpu_allreduce_sum(h->mg, buf, count, st);   // count is collective: every rank falls back together
  if (rc) return fail(h, rc, "allreduce failed");
  k_scale<<<148 * 4, 256, 0, st>>>(buf, count, 1.0f / (float)h->d.world);
  h->launches += 1;
  return HET_OK;
}

het_status_t het_group_dense_allreduce(const het_cache_t* hs, uint32_t N, float* const* bufs, uint64_t count,
                                       het_stream_t stream_) {
  NvtxRange nvtx_("het_group_dense_allreduce");
  cudaStream_t st = (cudaStream_t)stream_;
  if (check_members(hs, N) || !bufs) return HET_ERR_ARG;
  if (count == 0) return HET_OK;
  for (uint32_t i = 0; i < N; ++i)
    if (!bufs[i] || !is_device_ptr(bufs[i])) return fail(hs[i], HET_ERR_ARG, "dense buffer must be device memory");
  for (int ph = 1; ph <= 2; ++ph)
    for (uint32_t i = 0; i < N; ++i) {
      int l = 0;
      Prof p(hs[i], "dense_allreduce", st);
      het_status_t rc = mgpu_dense_p2p(hs[i]->mg, hs[i]->d, bufs[i], count, ph, st, &l);
      if (rc) return fail(hs[i], rc, "loopback dense all-reduce: count exceeds the staging (opts.dense_max)");
      hs[i]->launches += l;
    }
  return HET_OK;
}

het_status_t het_debug_lookup_log(het_cache_t h, int64_t* uniq, int32_t* inverse, int32_t* perm,
                                  int32_t* seg_off, uint8_t* status, uint32_t* U, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !U) return HET_ERR_ARG;
  Ctl ctl;
  Call& c = h->call;
  if (c.rmode) launch_compact_log(h->d, c, st);   // the rmode lookup keeps no compact log: build it now
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  int32_t ur = 0;
  if (c.rmode) CUDA_TRY(h, cudaMemcpyAsync(&ur, c.dbg_U, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  uint32_t u = c.rmode ? (uint32_t)ur : (uint32_t)ctl.U;
  *U = u;
  size_t n = (size_t)h->call.n;
  if (uniq) CUDA_TRY(h, cudaMemcpyAsync(uniq, c.uniq, u * 8, cudaMemcpyDefault, st));
  if (inverse) CUDA_TRY(h, cudaMemcpyAsync(inverse, c.rmode ? c.dbg_inverse : c.inverse, n * 4, cudaMemcpyDefault, st));
  if (perm) CUDA_TRY(h, cudaMemcpyAsync(perm, c.perm, n * 4, cudaMemcpyDefault, st));
  if (seg_off) CUDA_TRY(h, cudaMemcpyAsync(seg_off, c.seg_off, (u + 1) * 4, cudaMemcpyDefault, st));
  if (status) CUDA_TRY(h, cudaMemcpyAsync(status, c.rmode ? c.dbg_status : c.status, u, cudaMemcpyDefault, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return HET_OK;
}

het_status_t het_debug_victims(het_cache_t h, int64_t* keys, uint8_t* dirty, uint32_t cap, uint32_t* e,
                               het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !e) return HET_ERR_ARG;
  flush_evict(h, st, false);
  Ctl ctl;
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  uint32_t nv = (ctl.abort || ctl.need <= 0) ? 0 : (uint32_t)ctl.nvict;
  *e = nv;
  if (nv > cap) return fail(h, HET_ERR_CAPACITY, "victim buffer too small");
  std::vector<int64_t> k(nv);
  std::vector<uint8_t> dt(nv);
  CUDA_TRY(h, cudaMemcpyAsync(k.data(), h->victim_keys, nv * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(dt.data(), h->victim_dirty, nv, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  std::vector<uint32_t> ord(nv);
  for (uint32_t i = 0; i < nv; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return k[a] < k[b]; });
  std::vector<int64_t> ks(nv);
  std::vector<uint8_t> ds(nv);
  for (uint32_t i = 0; i < nv; ++i) { ks[i] = k[ord[i]]; ds[i] = dt[ord[i]]; }
  if (keys) CUDA_TRY(h, cudaMemcpy(keys, ks.data(), nv * 8, cudaMemcpyDefault));
  if (dirty) CUDA_TRY(h, cudaMemcpy(dirty, ds.data(), nv, cudaMemcpyDefault));
  return HET_OK;
}

het_status_t het_debug_dump_cache(het_cache_t h, int64_t* keys, float* v, float* p, uint32_t* cs,
                                  uint32_t* cc, uint32_t* prim, uint32_t cap, uint32_t* m,
                                  het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !m) return HET_ERR_ARG;
  flush_evict(h, st, false);
  Dev& d = h->d;
  std::vector<int64_t> ek(d.Ecap);
  CUDA_TRY(h, cudaMemcpyAsync(ek.data(), d.ekey, d.Ecap * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  std::vector<int32_t> idx;
  for (int64_t e = 0; e < d.Ecap; ++e)
    if (ek[e] >= 0) idx.push_back((int32_t)e);
  std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return ek[a] < ek[b]; });
  *m = (uint32_t)idx.size();
  if (idx.size() > cap) return fail(h, HET_ERR_CAPACITY, "dump buffer too small");
  size_t mm = idx.size();
  if (keys) {
    std::vector<int64_t> ks(mm);
    for (size_t i = 0; i < mm; ++i) ks[i] = ek[idx[i]];
    CUDA_TRY(h, cudaMemcpy(keys, ks.data(), mm * 8, cudaMemcpyDefault));
  }
  if (mm == 0) return HET_OK;
  int32_t* didx;
  float *dv = nullptr, *dp = nullptr;
  uint32_t *dcs = nullptr, *dcc = nullptr, *dpr = nullptr;
  CUDA_TRY(h, cudaMalloc(&didx, mm * 4));
  CUDA_TRY(h, cudaMemcpy(didx, idx.data(), mm * 4, cudaMemcpyHostToDevice));
  if (v) CUDA_TRY(h, cudaMalloc(&dv, mm * d.D * 4));
  if (p) CUDA_TRY(h, cudaMalloc(&dp, mm * d.D * 4));
  if (cs) CUDA_TRY(h, cudaMalloc(&dcs, mm * 4));
  if (cc) CUDA_TRY(h, cudaMalloc(&dcc, mm * 4));
  if (prim) CUDA_TRY(h, cudaMalloc(&dpr, mm * 4));
  k_gather_entries<<<256, 256>>>(d, didx, (int)mm, dv, dp, dcs, dcc, dpr);
  CUDA_TRY(h, cudaDeviceSynchronize());
  if (v) CUDA_TRY(h, cudaMemcpy(v, dv, mm * d.D * 4, cudaMemcpyDefault));
  if (p) CUDA_TRY(h, cudaMemcpy(p, dp, mm * d.D * 4, cudaMemcpyDefault));
  if (cs) CUDA_TRY(h, cudaMemcpy(cs, dcs, mm * 4, cudaMemcpyDefault));
  if (cc) CUDA_TRY(h, cudaMemcpy(cc, dcc, mm * 4, cudaMemcpyDefault));
  if (prim) CUDA_TRY(h, cudaMemcpy(prim, dpr, mm * 4, cudaMemcpyDefault));
  cudaFree(didx);
  cudaFree(dv); cudaFree(dp); cudaFree(dcs); cudaFree(dcc); cudaFree(dpr);
  return HET_OK;
}

het_status_t het_debug_eviction_plan(het_cache_t h, int64_t* out8, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !out8) return HET_ERR_ARG;
  flush_evict(h, st, false);
  Ctl ctl;
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  const int64_t v[8] = {ctl.emode, ctl.need, ctl.nvict, ctl.T, ctl.Kstar, ctl.lowmask, 0, 0};
  std::memcpy(out8, v, sizeof(v));
  return HET_OK;
}

het_status_t het_profile_enable(het_cache_t h, int on) {
  if (!h) return HET_ERR_ARG;
  h->prof = on != 0;
  return HET_OK;
}

het_status_t het_profile_read(het_cache_t h, char (*names)[32], double* ms, uint64_t* launches,
                              uint32_t cap, uint32_t* k) {
  if (!h || !k) return HET_ERR_ARG;
  CUDA_TRY(h, cudaDeviceSynchronize());
  for (ProfRec& r : h->prof_pending) {
    float t = 0;
    cudaEventElapsedTime(&t, r.a, r.b);
    bool found = false;
    for (auto& a : h->prof_acc)
      if (a.first == r.name) { a.second.first += t; a.second.second += 1; found = true; break; }
    if (!found) h->prof_acc.push_back({r.name, {t, 1}});
    h->ev_pool.push_back(r.a);
    h->ev_pool.push_back(r.b);
  }
  h->prof_pending.clear();
  uint32_t i = 0;
  for (auto& a : h->prof_acc) {
    if (i >= cap) break;
    if (names) { std::strncpy(names[i], a.first.c_str(), 31); names[i][31] = 0; }
    if (ms) ms[i] = a.second.first;
    if (launches) launches[i] = a.second.second;
    ++i;
  }
  *k = i;
  h->prof_acc.clear();
  return HET_OK;
}

het_status_t het_cache_destroy(het_cache_t h) {
  if (!h) return HET_ERR_ARG;
  cudaDeviceSynchronize();
  if (h->mg) mgpu_destroy(h->mg);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->copy) cudaStreamDestroy(h->copy);
  if (h->ev_rows_free) cudaEventDestroy(h->ev_rows_free);
  if (h->ev_rows_ready) cudaEventDestroy(h->ev_rows_ready);
  if (h->ustream) cudaStreamDestroy(h->ustream);
  if (h->ev_lk_done) cudaEventDestroy(h->ev_lk_done);
  if (h->ev_upd_done) cudaEventDestroy(h->ev_upd_done);
  for (void* q : h->allocs) cudaFree(q);
  for (ProfRec& r : h->prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  std::free(h->evbuf_host);
  delete h;
  return HET_OK;
}

const char* het_last_error(het_cache_t h) { return h ? h->last_error.c_str() : "null handle"; }

}  // extern "C"

// profiling hook for the multi-GPU orchestration
namespace het {
void* prof_begin(void* hp, const char* name, cudaStream_t st) {
  if (!hp) return nullptr;
  het_cache* h = (het_cache*)hp;
  if (!h->prof) return nullptr;
  ProfRec* r = new ProfRec{name, ev_get(h), ev_get(h)};
  cudaEventRecord(r->a, st);
  return r;
}
void prof_end(void* hp, void* rec, cudaStream_t st) {
  if (!hp || !rec) return;
  het_cache* h = (het_cache*)hp;
  ProfRec* r = (ProfRec*)rec;
  cudaEventRecord(r->b, st);
  h->prof_pending.push_back(*r);
  delete r;
}
}  // namespace het
