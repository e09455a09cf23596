// C-ABI of libhet (include/het.h): argument checks, allocation, per-call
// orchestration of the sm_100a kernels on the caller's stream, profiling.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/het.h"
#include "het_internal.cuh"
#include "het_mgpu.h"
#include "het_p2p.h"

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
  float* stage_rows = nullptr;
  float* stage_out = nullptr;
  // protocol state
  bool have_lookup = false;
  bool fused = false;          // the last lookup ran the fused single-GPU kernels
  uint32_t last_n = 0;
  int64_t overflow_bound = 0;  // worst-case residents above C since the last eviction
  uint64_t lookups = 0, keys = 0, updates = 0, launches = 0;
  // multi-GPU
  MgpuState* mg = nullptr;
  // segment reduce of large batches: heavy keys on a forked stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
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

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
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

het_status_t het_cache_create(uint64_t rows, uint32_t D, double cache_frac, uint32_t s,
                              het_policy_t policy, const het_dist_t* dist, const het_opts_t* opt,
                              het_stream_t stream_, het_cache_t* out) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!out) return HET_ERR_ARG;
  *out = nullptr;
  if (rows == 0 || rows > (1ull << 32) || D == 0 || (D % 4) != 0 || D > (1u << 16)) return HET_ERR_ARG;
  if (!(cache_frac >= 0.0 && cache_frac <= 1.0)) return HET_ERR_ARG;
  if (policy != HET_LFU && policy != HET_LRU && policy != HET_LIGHT_LFU) return HET_ERR_ARG;
  int rank = 0, world = 1;
  if (dist) {
    rank = dist->rank;
    world = dist->world;
    if (world < 1 || rank < 0 || rank >= world) return HET_ERR_ARG;
    if (world > 1 && !dist->nccl_unique_id) return HET_ERR_ARG;
  }
  het_cache* h = new het_cache();
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
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
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
  A(d.hkey, (size_t)S);
  A(d.hval, (size_t)S);
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
    rc = mgpu_create(h->mg, d, h->n_max, dist->nccl_unique_id, stream);
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

static het_status_t stage_keys(het_cache* h, const int64_t*& keys, uint32_t n, cudaStream_t st) {
  if (n == 0 || is_device_ptr(keys)) return HET_OK;
  if (!h->stage_keys) CUDA_TRY(h, (dalloc(h, &h->stage_keys, h->n_max)));
  CUDA_TRY(h, cudaMemcpyAsync(h->stage_keys, keys, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  keys = h->stage_keys;
  return HET_OK;
}

het_status_t het_lookup(het_cache_t h, const int64_t* keys, uint32_t n, uint64_t clock_t, float* out,
                        het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (n > h->n_max) return fail(h, HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  if (n && (!keys || !out)) return fail(h, HET_ERR_ARG, "null keys/out");
  if (h->overflow_bound + (int64_t)n > 2 * (int64_t)h->n_max)
    return fail(h, HET_ERR_CAPACITY, "too many lookups without eviction");
  het_status_t rc = stage_keys(h, keys, n, st);
  if (rc) return rc;
  bool out_host = n && !is_device_ptr(out);
  float* dout = out;
  if (out_host) {
    if (!h->stage_out) CUDA_TRY(h, (dalloc(h, &h->stage_out, (size_t)h->n_max * h->D)));
    dout = h->stage_out;
  }
  Call& c = h->call;
  c.n = (int)n;
  c.t = clock_t;
  c.keys = keys;
  Dev& d = h->d;
  // fused path: N = 1 up to FUSED_LOOKUP_MAX keys (beyond, the large-batch
  // per-phase kernels with the sliced heavy-key segment reduce), N > 1 over
  // the peer-memory exchange for every n; the dedup kernel follows n
  h->fused = !getenv("HET_NO_FUSED") && (d.world == 1 ? (int)n <= FUSED_LOOKUP_MAX : mgpu_p2p(h->mg) != nullptr);
  if (h->fused) {
    if (fused_ok(d, (int)n)) {
      Prof p(h, "dedup", st);
      h->launches += launch_dd_fused(d, c, (int)n, h->pbits, clock_t, 1, st);
    } else {
      launch_begin(d, clock_t, (int)n, st);
      Prof p(h, "dedup", st);
      h->launches += 1 + launch_dedup(c, (int)n, d.R, h->pbits, d.ctl, st);
    }
    if (d.world == 1) {
      Prof p(h, "lookup_fused", st);
      h->launches += launch_lookup_fused(d, c, dout, st);
    } else {
      Prof p(h, "exchange_fused", st);
      h->launches += p2p_round_fused(mgpu_p2p(h->mg), d, c, dout, st);
    }
  } else {
    launch_begin(d, clock_t, (int)n, st);
    h->launches += 1;
    {
      Prof p(h, "dedup", st);
      h->launches += launch_dedup(c, (int)n, d.R, h->pbits, d.ctl, st);
    }
    if (d.world == 1) {
      {
        Prof p(h, "probe", st);
        launch_probe(d, c, (int)n, st);
      }
      {
        Prof p(h, "sync_fetch", st);
        launch_sync_fetch_install_local(d, c, (int)n, st);
      }
      h->launches += 2;
    } else {
      rc = mgpu_lookup(h->mg, d, c, h->prof ? (void*)h : nullptr, st);
      if (rc) return fail(h, rc, "multi-GPU lookup failed");
      h->launches += mgpu_take_launches(h->mg);
    }
    {
      Prof p(h, "gather", st);
      launch_gather(d, c, dout, st);
      h->launches += 1;
    }
  }
  if (d.pin_thr) h->launches += launch_pin_apply(d, st);   // light-LFU promotions of this lookup
  if (out_host) CUDA_TRY(h, cudaMemcpyAsync(out, dout, (size_t)n * h->D * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaGetLastError());
  h->have_lookup = true;
  h->last_n = n;
  h->overflow_bound += n;
  return HET_OK;
}

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

het_status_t het_update(het_cache_t h, const int64_t* keys, uint32_t n, const float* grads, float lr,
                        het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  (void)keys;
  if (!h->have_lookup || n != h->last_n) return fail(h, HET_ERR_PROTOCOL, "write without matching read");
  if (n && !grads) return fail(h, HET_ERR_ARG, "null grads");
  if (n && !is_device_ptr(grads)) {
    if (!h->stage_rows) CUDA_TRY(h, (dalloc(h, &h->stage_rows, (size_t)h->n_max * h->D)));
    CUDA_TRY(h, cudaMemcpyAsync(h->stage_rows, grads, (size_t)n * h->D * 4, cudaMemcpyHostToDevice, st));
    grads = h->stage_rows;
  }
  Dev& d = h->d;
  if (h->fused) {
    Prof p(h, "update_fused", st);
    h->launches += launch_update_fused(d, h->call, grads, lr, h->evbuf_host, st,
                                       d.world > 1 ? (const void*)p2p_view_ptr(mgpu_p2p(h->mg)) : nullptr);
    h->overflow_bound = 0;
  } else {
    {
      Prof p(h, "segreduce_apply", st);
      h->launches += launch_segreduce_apply(d, h->call, grads, lr, (int)n, st, h->side, h->ev_fork, h->ev_join);
    }
    het_status_t rc = evict_overflow(h, st);
    if (rc) return fail(h, rc, "evict failed");
  }
  CUDA_TRY(h, cudaGetLastError());
  h->have_lookup = false;
  return HET_OK;
}

het_status_t het_evict(het_cache_t h, const int64_t* keys, uint32_t n, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  Dev& d = h->d;
  if (!keys) {
    het_status_t rc = evict_overflow(h, st);
    if (rc) return fail(h, rc, "evict failed");
    return HET_OK;
  }
  if (n > h->n_max) return fail(h, HET_ERR_CAPACITY, "n exceeds max_keys_per_call");
  het_status_t rc = stage_keys(h, keys, n, st);
  if (rc) return rc;
  Call& c = h->call;
  c.n = (int)n;
  c.keys = keys;
  cudaMemsetAsync(&d.ctl->abort, 0, 4, st);
  h->launches += launch_dedup(c, (int)n, d.R, h->pbits, d.ctl, st);
  if (d.world == 1) {
    int blocks = std::max(1, ((int)n + 7) / 8);
    k_evict_keys_local<<<blocks, 256, 0, st>>>(d, c);
    h->launches += 1;
  } else {
    rc = mgpu_evict_keys(h->mg, d, c, st);
    if (rc) return fail(h, rc, "multi-GPU evict failed");
    h->launches += mgpu_take_launches(h->mg);
  }
  h->have_lookup = false;
  CUDA_TRY(h, cudaGetLastError());
  return HET_OK;
}

static het_status_t sticky(het_cache* h, cudaStream_t st) {
  Ctl ctl;
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (ctl.err) return fail(h, (het_status_t)ctl.err, "sticky device error");
  return HET_OK;
}

het_status_t het_sync(het_cache_t h, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  Dev& d = h->d;
  if (d.world == 1) {
    k_flush_local<<<148 * 4, 256, 0, st>>>(d);
    h->launches += 1;
  } else {
    het_status_t rc = mgpu_drain(h->mg, d, h->call, st);
    if (rc == HET_OK) rc = mgpu_flush(h->mg, d, st);
    if (rc) return fail(h, rc, "multi-GPU flush failed");
    h->launches += mgpu_take_launches(h->mg);
  }
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
  return sticky(h, st);
}

het_status_t het_check(het_cache_t h) {
  if (!h) return HET_ERR_ARG;
  return sticky(h, 0);
}

het_status_t het_stats(het_cache_t h, het_stats_t* out) {
  if (!h || !out) return HET_ERR_ARG;
  unsigned long long cnt[C_NUM];
  Ctl ctl;
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
  out->sticky_error = ctl.err;
  out->pinned = (uint32_t)ctl.npinned;
  return HET_OK;
}

het_status_t het_read_global(het_cache_t h, const int64_t* keys, uint32_t n, float* rows, uint32_t* cg,
                             het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (n == 0) return HET_OK;
  if (!keys) return HET_ERR_ARG;
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

het_status_t het_dense_allreduce(het_cache_t h, float* buf, uint64_t count, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h) return HET_ERR_ARG;
  if (count == 0 || h->d.world == 1) return HET_OK;
  if (!buf || !is_device_ptr(buf)) return fail(h, HET_ERR_ARG, "dense buffer must be device memory");
  Prof p(h, "dense_allreduce", st);
  int l = 0;
  het_status_t rc = mgpu_dense_p2p(h->mg, h->d, buf, count, st, &l);   // peer-memory one-shot mean
  if (rc == HET_OK) {
    h->launches += l;
    return HET_OK;
  }
  if (rc != HET_ERR_CAPACITY) return fail(h, rc, "peer all-reduce failed");
  rc = mgpu_allreduce_sum(h->mg, buf, count, st);
  if (rc) return fail(h, rc, "allreduce failed");
  k_scale<<<148 * 4, 256, 0, st>>>(buf, count, 1.0f / (float)h->d.world);
  h->launches += 1;
  return HET_OK;
}

het_status_t het_debug_lookup_log(het_cache_t h, int64_t* uniq, int32_t* inverse, int32_t* perm,
                                  int32_t* seg_off, uint8_t* status, uint32_t* U, het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !U) return HET_ERR_ARG;
  Ctl ctl;
  CUDA_TRY(h, cudaMemcpyAsync(&ctl, h->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  uint32_t u = (uint32_t)ctl.U;
  *U = u;
  size_t n = (size_t)h->call.n;
  Call& c = h->call;
  if (uniq) CUDA_TRY(h, cudaMemcpyAsync(uniq, c.uniq, u * 8, cudaMemcpyDefault, st));
  if (inverse) CUDA_TRY(h, cudaMemcpyAsync(inverse, c.inverse, n * 4, cudaMemcpyDefault, st));
  if (perm) CUDA_TRY(h, cudaMemcpyAsync(perm, c.perm, n * 4, cudaMemcpyDefault, st));
  if (seg_off) CUDA_TRY(h, cudaMemcpyAsync(seg_off, c.seg_off, (u + 1) * 4, cudaMemcpyDefault, st));
  if (status) CUDA_TRY(h, cudaMemcpyAsync(status, c.status, u, cudaMemcpyDefault, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return HET_OK;
}

het_status_t het_debug_victims(het_cache_t h, int64_t* keys, uint8_t* dirty, uint32_t cap, uint32_t* e,
                               het_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!h || !e) return HET_ERR_ARG;
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
