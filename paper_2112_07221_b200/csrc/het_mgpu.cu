// Multi-GPU path (N > 1): one worker per GPU, the global table hash-sharded
// over the workers (owner(k) = k mod N, local row = k div N; R15), exchanges
// by NCCL grouped send/recv all-to-alls over NVLink on the caller's stream.
//
// Lookup (Alg. 2 over N lock-step workers, reading R1):
//   probe            cond (1) locally; hits passing it become NEEDQ
//   C1  clock check  requester -> owner: keys;  owner -> requester: c_g
//                    ("we only send the clocks"); requester evaluates
//                    cond (2) -> HIT / EXP2.  Owners answer before applying any
//                    push of this iteration (stream order), i.e. L3 reads c_g
//                    after U4(t-1) and before L4(t).
//   C2  sync+fetch   requester -> owner: header (key, c_c, dirty) for every
//                    expired hit and miss + the pending row of dirty syncs
//                    (fused Evict(k)+Fetch(k); R5); the owner groups
//                    the requests of all sources by row (dedup kernel: ascending
//                    source rank within a row), applies the pushes in that order
//                    (W += p, c_g = max), then answers every request
//                    with (c_g, W row) read after all pushes (L4 before L5).
//   install          v = W row, c_s = c_c = c_g
// Update: segment-reduce/apply locally, select victims locally, then
//   C3  push         victim -> owner: (key, c_c, p row) for dirty victims;
//                    owners apply grouped by row in source-rank order (U4).
// Per-peer message counts are exchanged first (one int pair per peer) and
// read on the host, which sizes the NCCL calls.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "het_mgpu.h"
#include "het_p2p.h"

namespace het {

constexpr int MG_TPB = 256;

struct ReqHdr {       // C2 request header (16 B)
  int64_t key;
  uint32_t cc;
  int32_t push;       // index of the pending row in the sender's push region, -1 if clean/miss
};

struct MgpuState {
  ncclComm_t comm = nullptr;
  int N = 1, rank = 0;
  uint32_t D = 0;
  int64_t CAPS = 0;           // per-peer region capacity (records)
  int64_t REC = 0;            // floats per record with a row: 4 + D
  // C1
  int64_t* qkeys = nullptr;   // [N][CAPS] send
  int32_t* qidx = nullptr;    // [N][CAPS]
  int64_t* rqkeys = nullptr;  // [N][CAPS] recv
  uint32_t* ans = nullptr;    // [N][CAPS] owner answers
  uint32_t* ansr = nullptr;   // [N][CAPS] answers received
  // C2
  ReqHdr* hdr = nullptr;      // [N][CAPS]
  int32_t* ridx = nullptr;    // [N][CAPS]
  float* prow = nullptr;      // [N][CAPS][D]
  ReqHdr* rhdr = nullptr;     // [N][CAPS]
  float* rprow = nullptr;     // [N][CAPS][D]
  float* resp = nullptr;      // [N][CAPS][REC]
  float* rresp = nullptr;     // [N][CAPS][REC]
  // C3
  float* push = nullptr;      // [N][CAPS][REC]  {key lo, key hi, c_c, 0, row}
  float* rpush = nullptr;     // [N][CAPS][REC]
  // counts: [N][2] (records, pushes)
  int32_t* scnt = nullptr;
  int32_t* rcnt = nullptr;
  int32_t* h_scnt = nullptr;  // pinned host copies
  int32_t* h_rcnt = nullptr;
  // owner-side grouping (dedup of received rows)
  Call oc{};
  int64_t* okeys = nullptr;   // [N*CAPS] local rows of received records
  int32_t* osrc = nullptr;    // [N*CAPS] record location s*CAPS + j
  Ctl* octl = nullptr;
  int opbits = 1;
  uint64_t launches = 0;
  uint64_t bytes_clock_tx = 0, bytes_clock_rx = 0, bytes_emb_tx = 0, bytes_emb_rx = 0;
  std::vector<void*> allocs;
  P2PState* p2p = nullptr;     // device-initiated exchange (default); nullptr = NCCL v1
};

template <typename T>
static bool mg_alloc(MgpuState* m, T** p, size_t count) {
  void* q = nullptr;
  if (cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) return false;
  m->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return true;
}

static int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

P2PState* mgpu_p2p(MgpuState* mg) { return mg ? mg->p2p : nullptr; }

uint64_t mgpu_take_launches(MgpuState* mg) {
  uint64_t l = mg ? mg->launches : 0;
  if (mg) mg->launches = 0;
  return l;
}

void mgpu_bytes(MgpuState* mg, uint64_t* ctx, uint64_t* crx, uint64_t* etx, uint64_t* erx) {
  *ctx = mg ? mg->bytes_clock_tx : 0;
  *crx = mg ? mg->bytes_clock_rx : 0;
  *etx = mg ? mg->bytes_emb_tx : 0;
  *erx = mg ? mg->bytes_emb_rx : 0;
}

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ int owner_of(const Dev& s, int64_t key) { return (int)(key % s.world); }

// warp-aggregated slot claim in per-owner regions
__device__ __forceinline__ int claim(int32_t* cnt, int owner, bool pred) {
  unsigned act = __ballot_sync(0xffffffffu, pred);
  int slot = -1;
  if (pred) {
    unsigned grp = __match_any_sync(act, owner);
    int leader = __ffs(grp) - 1;
    int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cnt[owner * 2], __popc(grp));
    base = __shfl_sync(grp, base, leader);
    slot = base + __popc(grp & ((1u << lane) - 1));
  }
  return slot;
}

// C1 build: one thread per unique key
__global__ void k_build_queries(Dev s, Call c, MgpuState m_) {
  const MgpuState& m = m_;
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  int U = s.ctl->abort ? 0 : s.ctl->U;
  int limit = ((c.n + 31) / 32) * 32;
  if (u >= limit) return;
  bool q = u < U && c.status[u] == ST_NEEDQ;
  int64_t key = q ? c.uniq[u] : 0;
  int o = q ? owner_of(s, key) : 0;
  int slot = claim(m.scnt, o, q);
  if (q) {
    m.qkeys[o * m.CAPS + slot] = key;
    m.qidx[o * m.CAPS + slot] = u;
  }
}

// C1 owner: answer c_g for every received key
__global__ void k_answer(Dev s, MgpuState m_) {
  const MgpuState& m = m_;
  for (int src = 0; src < m.N; ++src) {
    int nq = m.rcnt[src * 2];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
      int64_t key = m.rqkeys[src * m.CAPS + j];
      m.ans[src * m.CAPS + j] = s.cg[key / s.world];
    }
  }
}

// C1 requester: condition (2) with the owner's c_g
__global__ void k_finish_classify(Dev s, Call c, MgpuState m_) {
  const MgpuState& m = m_;
  __shared__ unsigned bc[2];
  if (threadIdx.x < 2) bc[threadIdx.x] = 0;
  __syncthreads();
  for (int o = 0; o < m.N; ++o) {
    int nq = m.scnt[o * 2];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
      int u = m.qidx[o * m.CAPS + j];
      uint32_t g = m.ansr[o * m.CAPS + j];
      uint32_t ecc = s.cc[c.uentry[u]];
      bool ok = (g <= ecc) || (g - ecc <= s.s);     // c_g <= c_c + s
      c.status[u] = ok ? ST_HIT : ST_EXP2;
      atomicAdd(&bc[ok ? 0 : 1], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[1]);
  }
}

// C2 build: warp per unique key; header for every expired hit / miss, the
// pending row for dirty syncs
__global__ void k_build_requests(Dev s, Call c, MgpuState m_) {
  const MgpuState& m = m_;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s.ctl->abort || u >= s.ctl->U) return;
  uint8_t st = c.status[u];
  if (st == ST_HIT) return;
  int64_t key = c.uniq[u];
  int o = owner_of(s, key);
  int slot = 0, ps = -1;
  uint32_t ecc = 0;
  bool dirty = false;
  int32_t e = c.uentry[u];
  if (st != ST_MISS) {
    ecc = s.cc[e];
    dirty = ecc > s.cs[e];
  }
  if (lane == 0) {
    slot = atomicAdd(&m.scnt[o * 2], 1);
    if (dirty) ps = atomicAdd(&m.scnt[o * 2 + 1], 1);
    ReqHdr h;
    h.key = key;
    h.cc = ecc;
    h.push = ps;
    m.hdr[o * m.CAPS + slot] = h;
    m.ridx[o * m.CAPS + slot] = u;
  }
  ps = __shfl_sync(0xffffffffu, ps, 0);
  if (dirty) {
    const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
    float4* dst = reinterpret_cast<float4*>(m.prow + ((int64_t)o * m.CAPS + ps) * s.D);
    for (int d = lane; d < (int)(s.D >> 2); d += 32) dst[d] = pr[d];
  }
}

// owner: local rows of the received records (C2 headers or C3 pushes), in
// (source, record) order, for grouping by the dedup kernel
__global__ void k_owner_keys(Dev s, MgpuState m_, int kind) {
  const MgpuState& m = m_;
  __shared__ int offs[65];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int src = 0; src < m.N; ++src) { offs[src] = acc; acc += m.rcnt[src * 2]; }
    offs[m.N] = acc;
  }
  __syncthreads();
  for (int src = 0; src < m.N; ++src) {
    int nr = m.rcnt[src * 2];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nr; j += gridDim.x * blockDim.x) {
      int64_t key;
      if (kind == 0) key = m.rhdr[src * m.CAPS + j].key;
      else {
        const float* rec = m.rpush + ((int64_t)src * m.CAPS + j) * m.REC;
        key = *reinterpret_cast<const int64_t*>(rec);
      }
      m.okeys[offs[src] + j] = key / s.world;
      m.osrc[offs[src] + j] = src * (int)m.CAPS + j;
    }
  }
}

__device__ __forceinline__ float4 f4add_m(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// owner, C2: warp per distinct row: apply the sync pushes in source order
// (L4), then answer every request of the row with (c_g, W row) (L5)
__global__ void k_owner_sync_fetch(Dev s, MgpuState m_) {
  const MgpuState& m = m_;
  const Call& oc = m.oc;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  int U = m.octl->U;
  const int D4 = s.D >> 2;
  for (int u = w; u < U; u += nw) {
    int64_t row = oc.uniq[u];
    float4* Wr = reinterpret_cast<float4*>(s.W + row * s.D);
    uint32_t g = s.cg[row];
    int j0 = oc.seg_off[u], j1 = oc.seg_off[u + 1];
    for (int j = j0; j < j1; ++j) {
      int loc = m.osrc[oc.perm[j]];
      ReqHdr h = m.rhdr[loc];
      if (h.push >= 0) {
        int src = loc / (int)m.CAPS;
        const float4* pr = reinterpret_cast<const float4*>(m.rprow + ((int64_t)src * m.CAPS + h.push) * s.D);
        for (int d = lane; d < D4; d += 32) Wr[d] = f4add_m(Wr[d], pr[d]);
        g = g > h.cc ? g : h.cc;
      }
    }
    if (lane == 0) s.cg[row] = g;
    __syncwarp();
    for (int j = j0; j < j1; ++j) {
      int loc = m.osrc[oc.perm[j]];
      float* rec = m.resp + (int64_t)loc * m.REC;
      if (lane == 0) reinterpret_cast<uint32_t*>(rec)[0] = g;
      float4* dst = reinterpret_cast<float4*>(rec + 4);
      for (int d = lane; d < D4; d += 32) dst[d] = Wr[d];
    }
  }
}

// requester, C2: install the responses (L5): v = W row, c_s = c_c = c_g
__global__ void k_install(Dev s, Call c, MgpuState m_) {
  const MgpuState& m = m_;
  __shared__ int dpop[LFU_CB_MAX];
  dpop_init(dpop);
  __syncthreads();
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  Ctl* ctl = s.ctl;
  const int D4 = s.D >> 2;
  for (int o = 0; o < m.N && !ctl->abort; ++o) {
    int nr = m.scnt[o * 2];
    for (int j = w; j < nr; j += nw) {
      int u = m.ridx[o * m.CAPS + j];
      const float* rec = m.rresp + ((int64_t)o * m.CAPS + j) * m.REC;
      uint32_t g = reinterpret_cast<const uint32_t*>(rec)[0];
      int64_t key = c.uniq[u];
      int32_t e;
      if (c.status[u] == ST_MISS) {
        int32_t idx = 0;
        if (lane == 0) idx = atomicSub(&ctl->ftop, 1) - 1;
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx < 0) {
          if (lane == 0) raise_err(ctl, 4);
          continue;
        }
        HET_ASSERT(idx >= 0 && idx < s.Ecap);
        e = s.fstack[idx];
        HET_ASSERT(e >= 0 && e < s.Ecap);
        warp_insert(s, key, e, lane);
        if (lane == 0) {
          s.ekey[e] = key;
          uint32_t prim = s.policy == 0 ? (s.lfu_persist ? s.count_by_key[key] : 1u) : (uint32_t)ctl->t_cur;
          s.eprim[e] = prim;
          if (s.policy == 0) { lfu_move(s, key, EP_FREE, prim, dpop); pin_candidate(s, key, e, prim); }
          atomicMin(&ctl->min_install, prim);
          c.uentry[u] = e;
        }
      } else {
        e = c.uentry[u];
      }
      const float4* src = reinterpret_cast<const float4*>(rec + 4);
      float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
      for (int d = lane; d < D4; d += 32) vr[d] = src[d];
      if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
}

// requester, C3: push records of dirty entries, then delete + free.
// mode 0: overflow victims (ctl->vmode: keys or entries); mode 1: unique
// keys of the current call (explicit Evict(k)); mode 2: entries [e0, e1) (flush)
__global__ void k_build_pushes(Dev s, Call c, MgpuState m_, const int64_t* vsel, const int32_t* victims,
                               int64_t* vkeys, uint8_t* vdirty, int mode, int64_t e0, int64_t e1) {
  const MgpuState& m = m_;
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty, s_ev;
  dpop_init(dpop);
  if (threadIdx.x == 0) { s_dirty = 0; s_ev = 0; }
  __syncthreads();
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  const int D4 = s.D >> 2;
  int64_t count = 0;
  if (!ctl->abort) {
    if (mode == 0) count = ctl->need > 0 ? ctl->nvict : 0;
    else if (mode == 1) count = ctl->U;
    else count = e1 - e0;
  }
  for (int64_t i = w; i < count; i += nw) {
    int64_t key;
    int32_t e;
    uint64_t slot = 0;
    if (mode == 2) {
      e = (int32_t)(e0 + i);
      key = s.ekey[e];
      if (key < 0) continue;
      uint32_t ecc = s.cc[e];
      if (ecc <= s.cs[e]) continue;         // flush pushes dirty entries only, keeps none
    } else {
      if (mode == 0) key = ctl->vmode == 1 ? vsel[i] : s.ekey[victims[i]];
      else key = c.uniq[i];
      e = warp_find_slot(s, key, lane, &slot);
      if (e < 0) continue;
    }
    const uint32_t ecc = s.cc[e], ecs = s.cs[e], prim = s.eprim[e];
    const bool dirty = ecc > ecs;
    if (dirty) {
      int o = owner_of(s, key);
      int ps = 0;
      if (lane == 0) ps = atomicAdd(&m.scnt[o * 2], 1);
      ps = __shfl_sync(0xffffffffu, ps, 0);
      float* rec = m.push + ((int64_t)o * m.CAPS + ps) * m.REC;
      if (lane == 0) {
        *reinterpret_cast<int64_t*>(rec) = key;
        reinterpret_cast<uint32_t*>(rec)[2] = ecc;
        reinterpret_cast<uint32_t*>(rec)[3] = 0;
      }
      const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
      float4* dst = reinterpret_cast<float4*>(rec + 4);
      for (int d = lane; d < D4; d += 32) dst[d] = pr[d];
    }
    if (mode != 2 && lane == 0) {
      s.hslot[slot] = HS_TOMB;
      atomicAdd(&ctl->n_tomb, 1);
      if (mode == 0) { vkeys[i] = key; vdirty[i] = dirty ? 1 : 0; }
      if (s.policy == 0) lfu_move(s, key, prim, EP_FREE, dpop);
      unpin_count(s, prim);
      s.eprim[e] = EP_FREE;
      s.ekey[e] = -1;
      s.fstack[atomicAdd(&ctl->ftop, 1)] = e;
      atomicAdd(&s_ev, 1u);
      if (dirty) atomicAdd(&s_dirty, 1u);
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (s_ev) atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)s_ev);
    if (s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
  }
}

// owner, C3: warp per distinct row, pushes applied in source order (U4)
__global__ void k_owner_apply_pushes(Dev s, MgpuState m_) {
  const MgpuState& m = m_;
  const Call& oc = m.oc;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  int U = m.octl->U;
  const int D4 = s.D >> 2;
  for (int u = w; u < U; u += nw) {
    int64_t row = oc.uniq[u];
    float4* Wr = reinterpret_cast<float4*>(s.W + row * s.D);
    uint32_t g = s.cg[row];
    for (int j = oc.seg_off[u]; j < oc.seg_off[u + 1]; ++j) {
      int loc = m.osrc[oc.perm[j]];
      const float* rec = m.rpush + (int64_t)loc * m.REC;
      uint32_t cc = reinterpret_cast<const uint32_t*>(rec)[2];
      const float4* pr = reinterpret_cast<const float4*>(rec + 4);
      for (int d = lane; d < D4; d += 32) Wr[d] = f4add_m(Wr[d], pr[d]);
      g = g > cc ? g : cc;
    }
    if (lane == 0) s.cg[row] = g;
  }
}

__global__ void k_reset_ctl_u(Ctl* octl) {
  octl->abort = 0;
}

// ---------------------------------------------------------------- host helpers
static het_status_t nccl_ok(ncclResult_t r) { return r == ncclSuccess ? HET_OK : HET_ERR_NCCL; }

// all-to-all of the per-peer count pairs, then read both on the host
static het_status_t exchange_counts(MgpuState* m, cudaStream_t st) {
  ncclGroupStart();
  for (int p = 0; p < m->N; ++p) {
    ncclSend(m->scnt + 2 * p, 2, ncclInt32, p, m->comm, st);
    ncclRecv(m->rcnt + 2 * p, 2, ncclInt32, p, m->comm, st);
  }
  if (ncclGroupEnd() != ncclSuccess) return HET_ERR_NCCL;
  cudaMemcpyAsync(m->h_scnt, m->scnt, sizeof(int32_t) * 2 * m->N, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(m->h_rcnt, m->rcnt, sizeof(int32_t) * 2 * m->N, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return HET_ERR_CUDA;
  return HET_OK;
}

// grouped send/recv: sendcnt[p] / recvcnt[p] elements of `bytes` each, regions of `stride` bytes
static het_status_t alltoallv(MgpuState* m, const void* sbuf, void* rbuf, const int32_t* sendcnt,
                              const int32_t* recvcnt, int cstride, size_t bytes, size_t stride, cudaStream_t st) {
  ncclGroupStart();
  for (int p = 0; p < m->N; ++p) {
    size_t sb = (size_t)sendcnt[p * cstride] * bytes;
    size_t rb = (size_t)recvcnt[p * cstride] * bytes;
    if (sb) ncclSend((const char*)sbuf + p * stride, sb, ncclChar, p, m->comm, st);
    if (rb) ncclRecv((char*)rbuf + p * stride, rb, ncclChar, p, m->comm, st);
  }
  return nccl_ok(ncclGroupEnd());
}

static int grid_for(int64_t units, int per_block) {
  int64_t b = (units + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}

// owner-side grouping of the received records (kind 0: C2 headers, 1: C3 pushes)
static void owner_group(MgpuState* m, const Dev& d, int total, int kind, cudaStream_t st) {
  k_owner_keys<<<grid_for(total, MG_TPB), MG_TPB, 0, st>>>(d, *m, kind);
  k_reset_ctl_u<<<1, 1, 0, st>>>(m->octl);
  Call oc = m->oc;
  oc.keys = m->okeys;
  oc.n = total;
  int64_t rows_local = d.rows_local;
  m->launches += 2 + launch_dedup(oc, total, rows_local, m->opbits, m->octl, st);
}

// ---------------------------------------------------------------- API
het_status_t mgpu_create(MgpuState*& mg, const Dev& d, uint32_t n_max, const void* uid, uint64_t dense_cap,
                         cudaStream_t st) {
  MgpuState* m = new MgpuState();
  mg = m;
  m->N = d.world;
  m->rank = d.rank;
  m->D = d.D;
  m->CAPS = 3 * (int64_t)n_max;
  m->REC = 4 + d.D;
  const char* env = std::getenv("HET_P2P");
  const bool loopback = uid == nullptr;   // N workers on this device, driven by het_group_* (no NCCL)
  const bool p2p = loopback || !(env && env[0] == '0');
  if (p2p && d.world > P2P_MAX_WORLD) return HET_ERR_ARG;
  if (!loopback) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    // NCCL's kernels (the dense all-reduce fallback, overlapped on a side
    // stream) are capped at NCCL_CTAS blocks, and the cooperative hot-path
    // kernels leave that many SMs free (het::coop_sm_reserve), so neither
    // waits for the other's SMs.
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (!getenv("HET_NCCL_DEFAULT")) {   // diagnostic: NCCL's own CTA choice
      cfg.maxCTAs = coop_sm_reserve();
      cfg.minCTAs = std::min(4, cfg.maxCTAs);
    }
    if (ncclCommInitRankConfig(&m->comm, d.world, id, d.rank, &cfg) != ncclSuccess) return HET_ERR_NCCL;
  }
  if (p2p) return p2p_create(m->p2p, d, n_max, m->comm, dense_cap, st);
  // the NCCL send/recv exchange (HET_P2P=0): its staging regions
  const int64_t NC = (int64_t)m->N * m->CAPS;
  bool ok = mg_alloc(m, &m->qkeys, NC) && mg_alloc(m, &m->qidx, NC) && mg_alloc(m, &m->rqkeys, NC) &&
            mg_alloc(m, &m->ans, NC) && mg_alloc(m, &m->ansr, NC) && mg_alloc(m, &m->hdr, NC) &&
            mg_alloc(m, &m->ridx, NC) && mg_alloc(m, &m->prow, NC * d.D) && mg_alloc(m, &m->rhdr, NC) &&
            mg_alloc(m, &m->rprow, NC * d.D) && mg_alloc(m, &m->resp, NC * m->REC) &&
            mg_alloc(m, &m->rresp, NC * m->REC) && mg_alloc(m, &m->push, NC * m->REC) &&
            mg_alloc(m, &m->rpush, NC * m->REC) && mg_alloc(m, &m->scnt, 2 * m->N) &&
            mg_alloc(m, &m->rcnt, 2 * m->N) && mg_alloc(m, &m->okeys, NC) && mg_alloc(m, &m->osrc, NC) &&
            mg_alloc(m, &m->octl, 1);
  Call& oc = m->oc;
  ok = ok && mg_alloc(m, &oc.uniq, NC) && mg_alloc(m, &oc.inverse, NC) && mg_alloc(m, &oc.perm, NC) &&
       mg_alloc(m, &oc.seg_off, NC + 1) && mg_alloc(m, &oc.status, NC) && mg_alloc(m, &oc.uentry, NC) &&
       mg_alloc(m, &oc.sortbuf0, NC) && mg_alloc(m, &oc.sortbuf1, NC) && mg_alloc(m, &oc.blockbuf, NC / 1024 + 2);
  if (!ok) return HET_ERR_OOM;
  if (cudaMallocHost(&m->h_scnt, sizeof(int32_t) * 2 * m->N) != cudaSuccess) return HET_ERR_OOM;
  if (cudaMallocHost(&m->h_rcnt, sizeof(int32_t) * 2 * m->N) != cudaSuccess) return HET_ERR_OOM;
  m->opbits = std::max(1, bits_for((uint64_t)NC - 1));
  cudaMemsetAsync(m->octl, 0, sizeof(Ctl), st);
  cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * m->N, st);
  return HET_OK;
}

void mgpu_destroy(MgpuState* m) {
  if (!m) return;
  p2p_destroy(m->p2p);
  // abort rather than destroy: teardown is not collective, and a CUDA graph
  // that captured NCCL work of this communicator may still be alive
  if (m->comm) ncclCommAbort(m->comm);
  for (void* q : m->allocs) cudaFree(q);
  if (m->h_scnt) cudaFreeHost(m->h_scnt);
  if (m->h_rcnt) cudaFreeHost(m->h_rcnt);
  delete m;
}

het_status_t mgpu_lookup(MgpuState* m, const Dev& d, const Call& c, void* prof, cudaStream_t st) {
  const int n = c.n;
  het_status_t rc;
  {
    void* pr = prof_begin(prof, "probe", st);
    launch_probe(d, c, n, st);
    prof_end(prof, pr, st);
    m->launches += 1;
  }
  const int N = m->N;
  if (m->p2p) {
    void* pr = prof_begin(prof, "exchange", st);
    m->launches += p2p_round(m->p2p, d, c, 0, st);
    prof_end(prof, pr, st);
    return HET_OK;
  }
  if (d.s != S_INF) {
    void* pr = prof_begin(prof, "clock_check", st);
    cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * N, st);
    k_build_queries<<<grid_for(std::max(n, 1), MG_TPB), MG_TPB, 0, st>>>(d, c, *m);
    if ((rc = exchange_counts(m, st))) return rc;
    if ((rc = alltoallv(m, m->qkeys, m->rqkeys, m->h_scnt, m->h_rcnt, 2, 8, m->CAPS * 8, st))) return rc;
    k_answer<<<grid_for(N * m->CAPS, MG_TPB), MG_TPB, 0, st>>>(d, *m);
    if ((rc = alltoallv(m, m->ans, m->ansr, m->h_rcnt, m->h_scnt, 2, 4, m->CAPS * 4, st))) return rc;
    k_finish_classify<<<grid_for(N * m->CAPS, MG_TPB), MG_TPB, 0, st>>>(d, c, *m);
    for (int p = 0; p < N; ++p) {
      m->bytes_clock_tx += (uint64_t)m->h_scnt[2 * p] * 8 + (uint64_t)m->h_rcnt[2 * p] * 4;
      m->bytes_clock_rx += (uint64_t)m->h_rcnt[2 * p] * 8 + (uint64_t)m->h_scnt[2 * p] * 4;
    }
    m->launches += 3;
    prof_end(prof, pr, st);
  }
  {
    void* pr = prof_begin(prof, "sync_fetch", st);
    cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * N, st);
    // warp per unique key, not grid-strided: one warp for every key (n may exceed grid_for's cap)
    k_build_requests<<<std::max(1, (n + 7) / 8), MG_TPB, 0, st>>>(d, c, *m);
    if ((rc = exchange_counts(m, st))) return rc;
    if ((rc = alltoallv(m, m->hdr, m->rhdr, m->h_scnt, m->h_rcnt, 2, sizeof(ReqHdr), m->CAPS * sizeof(ReqHdr), st)))
      return rc;
    if ((rc = alltoallv(m, m->prow, m->rprow, m->h_scnt + 1, m->h_rcnt + 1, 2, (size_t)d.D * 4,
                        (size_t)m->CAPS * d.D * 4, st)))
      return rc;
    int total = 0;
    for (int p = 0; p < N; ++p) total += m->h_rcnt[2 * p];
    owner_group(m, d, total, 0, st);
    k_owner_sync_fetch<<<grid_for(std::max(total, 1), 8), MG_TPB, 0, st>>>(d, *m);
    if ((rc = alltoallv(m, m->resp, m->rresp, m->h_rcnt, m->h_scnt, 2, (size_t)m->REC * 4,
                        (size_t)m->CAPS * m->REC * 4, st)))
      return rc;
    k_install<<<grid_for(N * m->CAPS, 8), MG_TPB, 0, st>>>(d, c, *m);
    for (int p = 0; p < N; ++p) {
      uint64_t hs = m->h_scnt[2 * p], hr = m->h_rcnt[2 * p], ps = m->h_scnt[2 * p + 1], prr = m->h_rcnt[2 * p + 1];
      m->bytes_emb_tx += hs * sizeof(ReqHdr) + ps * d.D * 4 + hr * m->REC * 4;
      m->bytes_emb_rx += hr * sizeof(ReqHdr) + prr * d.D * 4 + hs * m->REC * 4;
    }
    m->launches += 3;
    prof_end(prof, pr, st);
  }
  return HET_OK;
}

// C3 exchange + owner apply for whatever k_build_pushes put in m->push
static het_status_t push_exchange_apply(MgpuState* m, const Dev& d, cudaStream_t st) {
  het_status_t rc;
  if ((rc = exchange_counts(m, st))) return rc;
  if ((rc = alltoallv(m, m->push, m->rpush, m->h_scnt, m->h_rcnt, 2, (size_t)m->REC * 4,
                      (size_t)m->CAPS * m->REC * 4, st)))
    return rc;
  int total = 0;
  for (int p = 0; p < m->N; ++p) {
    total += m->h_rcnt[2 * p];
    m->bytes_emb_tx += (uint64_t)m->h_scnt[2 * p] * m->REC * 4;
    m->bytes_emb_rx += (uint64_t)m->h_rcnt[2 * p] * m->REC * 4;
  }
  owner_group(m, d, total, 1, st);
  k_owner_apply_pushes<<<grid_for(std::max(total, 1), 8), MG_TPB, 0, st>>>(d, *m);
  m->launches += 1;
  return HET_OK;
}

struct EvBufView {  // leading fields of EvBuf (k_evict.cu)
  uint32_t* hist; uint32_t* khist; int32_t* victims; int32_t* cand; int32_t* sub; int32_t* flags;
  int64_t* vkeys; uint8_t* vdirty; int64_t* vsel;
};

het_status_t mgpu_evict_overflow(MgpuState* m, const Dev& d, void* evbuf, void* prof, cudaStream_t st) {
  void* pr = prof_begin(prof, "evict", st);
  m->launches += launch_evict_select(d, evbuf, st);
  if (m->p2p) {
    m->launches += p2p_pushes(m->p2p, d, evbuf, st);
    prof_end(prof, pr, st);
    return HET_OK;
  }
  const EvBufView& b = *reinterpret_cast<const EvBufView*>(evbuf);
  cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * m->N, st);
  Call dummy{};
  k_build_pushes<<<148 * 2, MG_TPB, 0, st>>>(d, dummy, *m, b.vsel, b.victims, b.vkeys, b.vdirty, 0, 0, 0);
  m->launches += 1;
  het_status_t rc = push_exchange_apply(m, d, st);
  prof_end(prof, pr, st);
  return rc;
}

het_status_t mgpu_evict_keys(MgpuState* m, const Dev& d, const Call& c, cudaStream_t st) {   // NCCL exchange only
  cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * m->N, st);
  k_build_pushes<<<grid_for(std::max(c.n, 1), 8), MG_TPB, 0, st>>>(d, c, *m, nullptr, nullptr, nullptr, nullptr, 1,
                                                                     0, 0);
  m->launches += 1;
  return push_exchange_apply(m, d, st);
}

// flush (het_sync; R16): every dirty entry pushes to its owner.
// A key's pushes from all workers must meet at the owner in the same round
// (applied in source-rank order), so rounds cover whole KEY ranges: a
// histogram of dirty entries over FBINS key bins is max-reduced across the
// workers and the host groups consecutive bins into rounds whose per-worker
// count fits the (temporary) flush buffers.

// dirty resident entries of keys [k0, k1) per bin: bin(key) = (key - k0) * FBINS / (k1 - k0)
__global__ void k_flush_hist(Dev s, int32_t* bins, int64_t k0, int64_t k1) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s.Ecap; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t key = s.ekey[e];
    if (key >= k0 && key < k1 && s.cc[e] > s.cs[e]) atomicAdd(&bins[(int)(((key - k0) * FBINS) / (k1 - k0))], 1);
  }
}

__global__ void k_flush_build(Dev s, MgpuState m_, int64_t k0, int64_t k1) {
  const MgpuState& m = m_;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  const int D4 = s.D >> 2;
  for (int64_t e0 = (int64_t)w * 32; e0 < s.Ecap; e0 += (int64_t)nw * 32) {
    int64_t e = e0 + lane;
    int64_t key = e < s.Ecap ? s.ekey[e] : -1;
    bool pick = key >= k0 && key < k1 && s.cc[e] > s.cs[e];
    unsigned mk = __ballot_sync(0xffffffffu, pick);
    while (mk) {
      int src = __ffs(mk) - 1;
      mk &= mk - 1;
      int64_t k = __shfl_sync(0xffffffffu, key, src);
      int64_t ee = e0 + src;
      int o = owner_of(s, k);
      int ps = 0;
      if (lane == 0) ps = atomicAdd(&m.scnt[o * 2], 1);
      ps = __shfl_sync(0xffffffffu, ps, 0);
      float* rec = m.push + ((int64_t)o * m.CAPS + ps) * m.REC;
      if (lane == 0) {
        *reinterpret_cast<int64_t*>(rec) = k;
        reinterpret_cast<uint32_t*>(rec)[2] = s.cc[ee];
        reinterpret_cast<uint32_t*>(rec)[3] = 0;
      }
      const float4* pr = reinterpret_cast<const float4*>(s.p + ee * s.D);
      float4* dst = reinterpret_cast<float4*>(rec + 4);
      for (int d = lane; d < D4; d += 32) dst[d] = pr[d];
    }
  }
}

het_status_t mgpu_flush_hist(MgpuState* m, const Dev& d, int64_t k0, int64_t k1, int32_t* bins_host,
                             cudaStream_t st) {
  int32_t* dbins;
  if (cudaMallocAsync((void**)&dbins, FBINS * 4, st) != cudaSuccess) return HET_ERR_OOM;
  cudaMemsetAsync(dbins, 0, FBINS * 4, st);
  k_flush_hist<<<148 * 4, 256, 0, st>>>(d, dbins, k0, k1);
  m->launches += 1;
  cudaMemcpyAsync(bins_host, dbins, FBINS * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbins, st);
  return cudaStreamSynchronize(st) == cudaSuccess ? HET_OK : HET_ERR_CUDA;
}

het_status_t mgpu_allreduce_max_host(MgpuState* m, int32_t* x, int count, cudaStream_t st) {
  if (!m->comm) return HET_ERR_ARG;
  int32_t* dx;
  if (cudaMallocAsync((void**)&dx, (size_t)count * 4, st) != cudaSuccess) return HET_ERR_OOM;
  cudaMemcpyAsync(dx, x, (size_t)count * 4, cudaMemcpyHostToDevice, st);
  if (ncclAllReduce(dx, dx, count, ncclInt32, ncclMax, m->comm, st) != ncclSuccess) return HET_ERR_NCCL;
  cudaMemcpyAsync(x, dx, (size_t)count * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dx, st);
  return cudaStreamSynchronize(st) == cudaSuccess ? HET_OK : HET_ERR_CUDA;
}

bool mgpu_loopback(MgpuState* m) { return m && m->p2p && p2p_loopback(m->p2p); }

het_status_t mgpu_comm_error(MgpuState* m) {
  if (!m || !m->comm) return HET_OK;
  ncclResult_t r = ncclSuccess;
  if (ncclCommGetAsyncError(m->comm, &r) != ncclSuccess || r != ncclSuccess) return HET_ERR_NCCL;
  return HET_OK;
}

het_status_t mgpu_flush(MgpuState* m, const Dev& d, cudaStream_t st) {
  const int N = m->N;
  int32_t *dbins, *rbins;
  if (cudaMallocAsync((void**)&dbins, FBINS * 4, st) || cudaMallocAsync((void**)&rbins, FBINS * 4, st))
    return HET_ERR_OOM;
  cudaMemsetAsync(dbins, 0, FBINS * 4, st);
  k_flush_hist<<<148 * 4, 256, 0, st>>>(d, dbins, 0, d.R);
  if (ncclAllReduce(dbins, rbins, FBINS, ncclInt32, ncclMax, m->comm, st) != ncclSuccess) return HET_ERR_NCCL;
  std::vector<int32_t> bins(FBINS);
  cudaMemcpyAsync(bins.data(), rbins, FBINS * 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return HET_ERR_CUDA;
  cudaFreeAsync(dbins, st);
  cudaFreeAsync(rbins, st);
  // flush buffer capacity per peer region: ~256 MB per direction, at least one bin
  int32_t maxbin = *std::max_element(bins.begin(), bins.end());
  int64_t FB = std::max<int64_t>((256ll << 20) / ((int64_t)N * m->REC * 4), m->CAPS);
  FB = std::max<int64_t>(FB, maxbin);
  // swap in temporary buffers sized N x FB
  MgpuState save = *m;
  const int64_t NC = (int64_t)N * FB;
  het_status_t rc = HET_OK;
  std::vector<void*> tmp;
  auto talloc = [&](void** p, size_t bytes) {
    if (rc) return;
    if (cudaMallocAsync(p, std::max<size_t>(bytes, 16), st) != cudaSuccess) { rc = HET_ERR_OOM; return; }
    tmp.push_back(*p);
  };
  talloc((void**)&m->push, NC * m->REC * 4);
  talloc((void**)&m->rpush, NC * m->REC * 4);
  talloc((void**)&m->okeys, NC * 8);
  talloc((void**)&m->osrc, NC * 4);
  talloc((void**)&m->oc.uniq, NC * 8);
  talloc((void**)&m->oc.inverse, NC * 4);
  talloc((void**)&m->oc.perm, NC * 4);
  talloc((void**)&m->oc.seg_off, (NC + 1) * 4);
  talloc((void**)&m->oc.sortbuf0, NC * 8);
  talloc((void**)&m->oc.sortbuf1, NC * 8);
  talloc((void**)&m->oc.blockbuf, (NC / 1024 + 2) * 4);
  m->CAPS = FB;
  m->opbits = std::max(1, bits_for((uint64_t)NC - 1));
  int b0 = 0;
  while (!rc && b0 < FBINS) {
    int64_t acc = 0;
    int b1 = b0;
    while (b1 < FBINS && acc + bins[b1] <= FB) acc += bins[b1++];
    if (b1 == b0) b1 = b0 + 1;  // cannot happen (FB >= maxbin)
    if (acc > 0) {
      int64_t k0 = ((int64_t)b0 * d.R + FBINS - 1) / FBINS, k1 = ((int64_t)b1 * d.R + FBINS - 1) / FBINS;
      // bin(key) = key*FBINS/R, so bins [b0, b1) are exactly keys [ceil(b0 R/F), ceil(b1 R/F))
      cudaMemsetAsync(m->scnt, 0, sizeof(int32_t) * 2 * N, st);
      k_flush_build<<<148 * 4, 256, 0, st>>>(d, *m, k0, k1);
      rc = push_exchange_apply(m, d, st);
    }
    b0 = b1;
  }
  cudaStreamSynchronize(st);
  for (void* q : tmp) cudaFreeAsync(q, st);
  uint64_t l = m->launches, a = m->bytes_emb_tx, b = m->bytes_emb_rx;
  *m = save;
  m->launches = l;
  m->bytes_emb_tx = a;
  m->bytes_emb_rx = b;
  return rc;
}

het_status_t mgpu_dense_p2p(MgpuState* m, const Dev& d, float* buf, uint64_t count, int phase, cudaStream_t st,
                            int* launches) {
  static const bool nccl_only = getenv("HET_DENSE_NCCL") != nullptr;   // diagnostic: NCCL all-reduce
  if (!m->p2p || (nccl_only && m->comm)) return HET_ERR_CAPACITY;
  return p2p_dense_allreduce(m->p2p, d, buf, count, phase, st, launches);
}

het_status_t mgpu_allreduce_sum(MgpuState* m, float* buf, uint64_t count, cudaStream_t st) {
  if (!m->comm) return HET_ERR_CAPACITY;   // loopback: no NCCL
  return nccl_ok(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, m->comm, st));
}

}  // namespace het
