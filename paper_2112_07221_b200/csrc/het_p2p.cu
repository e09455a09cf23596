// Multi-GPU exchange v2: device-initiated, over NVLink peer memory.
//
// Every rank exports one "inbox" allocation (CUDA IPC, mapped by every peer):
//   reqflag[N]    per source: {epoch, total records, pushes among them}
//   respflag[N]   per owner:  {epoch}
//   req[N][CAPS]  request records written by source s into region s
//   rows[N][CAPS][D]  rows of dirty records (same index as the record)
//   resp[N][CAPS][4 + D]  responses written by owner o into region o
// One lookup is one round: requesters write their records (the eviction
// pushes of their previous update first, then this lookup's requests)
// straight into the owners' inboxes with 128-bit peer stores and publish the
// round's epoch; owners link the records of each row (lock-free lists), apply
// them per row in source-rank order -- eviction pushes (U4 of t-1), clock
// checks against c_g after those pushes (L3), sync pushes (L4,
// P:442-443), then answer every request with (c_g, row) (L5) -- and
// write the responses straight into the requesters' inboxes.  No host
// synchronisation; the step is CUDA-graph capturable.
//
// A hit passing condition (1) sends its pending row speculatively (dirty
// entries); the owner applies it only if condition (2) fails (EXP2), which
// folds the clock check (C1) into the same round as the fetches (C2), and
// carrying the pushes of update t in round t+1 is the fusion of C3(t) with
// C1(t+1) that SURVEY §8(e) notes has identical semantics (U4(t) precedes
// L3(t+1) at every owner).
//
// Waits spin on flags in local memory written by peers (one process per GPU,
// so the waited-for kernel always runs on another GPU); every wait has a
// wall-clock timeout that raises a sticky error instead of hanging.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "het_internal.cuh"
#include "het_p2p.h"
#include "p2p_dev.cuh"

namespace het {

namespace cg = cooperative_groups;

// Row moves of one warp in batches of RB float4 per lane: the loads of a batch
// are issued before its stores, so wide rows (D = 4096: 32 float4 per lane)
// take D/(128*RB) memory round trips instead of D/128.
constexpr int RB = 4;
__device__ __forceinline__ void warp_copy_row(float4* dst, const float4* src, int D4, int lane) {
  for (int d0 = lane; d0 < D4; d0 += 32 * RB) {
    float4 t[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (d0 + 32 * b < D4) t[b] = src[d0 + 32 * b];
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (d0 + 32 * b < D4) dst[d0 + 32 * b] = t[b];
  }
}

#ifdef HET_TIMELINE
constexpr int PTLW = 8192;
__device__ unsigned long long g_ptl[16 * PTLW];
#define PTL(i) do { if ((threadIdx.x & 31) == 0) { int w_ = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; \
  if (w_ < PTLW) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); g_ptl[(i) * PTLW + w_] = t_; } } } while (0)
extern "C" int het_debug_timeline_p2p(unsigned long long* out) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_ptl, sizeof(g_ptl));
  static unsigned long long* zero = nullptr;
  if (!zero) zero = (unsigned long long*)calloc(16 * PTLW, 8);
  cudaMemcpyToSymbol(g_ptl, zero, sizeof(g_ptl));
  return 0;
}
#else
#define PTL(i) do {} while (0)
#endif

// ---------------------------------------------------------------- requester: build + publish
__global__ void k_p2p_build(Dev s, Call c, P2P m, int drain) {
  __shared__ unsigned long long sb[4];
  bytes_init(sb);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long ep = *m.epoch + 1;
  const int U = (drain || s.ctl->abort) ? 0 : s.ctl->U;
  const int D4 = s.D >> 2;
  for (int u = gw; u < U; u += nw) {
    const uint8_t st = c.status[u];
    if (st == ST_HIT) continue;
    const int64_t key = c.uniq[u];
    const int o = (int)(key % m.N);
    const int32_t e = st == ST_MISS ? -1 : c.uentry[u];
    uint32_t ecc = 0;
    bool dirty = false;
    if (e >= 0) { ecc = s.cc[e]; dirty = ecc > s.cs[e]; }
    const uint32_t kind = (st == ST_NEEDQ ? K_NEEDQ : st == ST_EXP1 ? K_EXP1 : K_MISS) | (dirty ? K_DIRTY : 0);
    int slot = 0;
    if (lane == 0) slot = atomicAdd(&m.lcnt[o], 1);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    const int64_t j = m.c3cnt[o] + slot;
    if (lane == 0) {
      Rec r;
      r.key = key; r.cc = ecc; r.kind = kind;
      reqrec(m, o, m.rank)[j] = r;
      m.ridx[(int64_t)o * m.CAPS + slot] = u;
      if (st == ST_NEEDQ) atomicAdd(&sb[0], 16ull);
      else atomicAdd(&sb[2], 16ull);
      if (dirty) atomicAdd(&sb[2], 4ull * s.D);
    }
    if (dirty) {
      warp_copy_row(reinterpret_cast<float4*>(reqrow(m, o, m.rank, j)),
                    reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D), D4, lane);
    }
  }
  __syncthreads();
  bytes_flush(s, sb);
  if (!last_block(&m.done[0])) return;
  if (threadIdx.x < m.N) {
    const int o = threadIdx.x;
    Flag* f = &reqflag(m, o)[m.rank];
    f->total = (uint32_t)(m.c3cnt[o] + m.lcnt[o]);
    f->pushes = (uint32_t)m.c3cnt[o];
    __threadfence_system();
    st_release(&f->epoch, ep);
    m.c3cnt[o] = 0;     // lcnt stays: k_p2p_install reads it, its last block zeroes it
  }
  if (threadIdx.x == 0) m.done[0] = 0;
}

// ---------------------------------------------------------------- owner: wait + link
// Link every received record into its row's list (grid-stride); tot[src] =
// records from src this round.
__device__ __forceinline__ void link_records(const P2P& m, const int32_t* tot) {
  int64_t all = 0;                        // every source's records as one index space: one pass
  for (int src = 0; src < m.N; ++src) all += tot[src];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g - threadIdx.x % 32 < all; g += stride) {
    bool live = g < all;
    int src = 0;
    int64_t j = g;
    while (live && src < m.N - 1 && j >= tot[src]) { j -= tot[src]; ++src; }
    int64_t row = 0;
    int32_t old = 0;
    if (live) {
      row = reqrec(m, m.rank, src)[j].key / m.N;
      const int32_t id = (int32_t)(src * m.CAPS + j);
      old = atomicExch(&m.head[row], id);
      m.next[id] = old;
    }
    // first record of a row: append the ROW to the leader list (one atomic per warp)
    const unsigned lm = __ballot_sync(0xffffffffu, live && old < 0);
    const int lane = threadIdx.x & 31;
    int b = 0;
    if (lane == 0 && lm) b = atomicAdd(m.nlead, __popc(lm));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (live && old < 0) m.leaders[b + __popc(lm & ((1u << lane) - 1))] = (int32_t)row;
  }
}

__global__ void k_p2p_link(Dev s, P2P m) {
  __shared__ int s_ok;
  __shared__ int32_t tot[64];
  const unsigned long long ep = *m.epoch + 1;
  Flag* flags = reqflag(m, m.rank);
  PTL(3);
  if (threadIdx.x == 0) s_ok = wait_flags(flags, m.N, ep, s.ctl);
  __syncthreads();
  PTL(4);
  if (!s_ok) return;
  if (threadIdx.x < m.N) {
    tot[threadIdx.x] = (int32_t)flags[threadIdx.x].total;
    if (blockIdx.x == 0) { m.qtot[threadIdx.x] = (int32_t)flags[threadIdx.x].total; m.qpush[threadIdx.x] = (int32_t)flags[threadIdx.x].pushes; }
  }
  __syncthreads();
  link_records(m, tot);
  PTL(5);
}

// ---------------------------------------------------------------- owner: apply + respond
// Warp per linked row (warp-strided): apply the row's records in source order
// and write the responses into the requesters' inboxes.  Wide rows: PG warps
// per row (a group inside one block), each walking the row's list and taking
// the same decisions, each moving its 1/PG of the columns; the group's first
// writes c_g, the response headers and the byte counters.  The lists' heads
// are reset after the phase (reset_heads), not by the walk.
__device__ __forceinline__ void process_rows(const Dev& s, const P2P& m, unsigned long long* sb) {
  __shared__ int32_t wbuf[32][32];   // per warp: the row's record ids, sorted
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int D4 = s.D >> 2;
  const int PG = wide_rows(s.D) ? 4 : 1;   // divides the 8 or 32 warps of a block
  const int nw = ((gridDim.x * blockDim.x) >> 5) / PG;
  const int gw0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int gw = gw0 / PG, sub = gw0 % PG;
  const bool lead = sub == 0;
  const int c0 = sub * (D4 / PG), c1 = c0 + D4 / PG;   // this warp's float4 columns
  const int nl = s.ctl->abort ? 0 : *m.nlead;
  const Rec* base = reqrec(m, m.rank, 0);
  for (int li = gw; li < nl; li += nw) {
    const int64_t row = m.leaders[li];
    // the row's server row and c_g do not depend on the list: load them first
    uint32_t g0 = 0;
    if (lane == 0) g0 = s.cg[row];
    const float4 wpre = c0 + lane < c1 ? reinterpret_cast<const float4*>(s.W + row * s.D)[c0 + lane]
                                       : make_float4(0.f, 0.f, 0.f, 0.f);   // this warp's first 32 float4
    if (PG > 1) {   // every warp of the group has read c_g before the group's first may write it
      g0 = __shfl_sync(0xffffffffu, g0, 0);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + wi / PG), "r"(PG * 32) : "memory");
    }
    // walk the row's list once (lane 0), sort by id = (source rank, pushes
    // before requests) across the lanes, hand record i to lane i
    int cnt = 0;
    if (lane == 0) {
      int32_t cur = m.head[row];
      while (cur >= 0 && cnt < 32) { wbuf[wi][cnt++] = cur; cur = m.next[cur]; }
    }
    __syncwarp();
    cnt = __shfl_sync(0xffffffffu, cnt, 0);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    {
      const int32_t mine = lane < cnt ? wbuf[wi][lane] : 0x7FFFFFFF;
      int rank = 0;
      for (int k = 0; k < cnt; ++k) rank += __shfl_sync(0xffffffffu, mine, k) < mine;
      __syncwarp();
      if (lane < cnt) wbuf[wi][rank] = mine;
      __syncwarp();
    }
    PTL(12);
    const bool have = lane < cnt;
    const int32_t id = have ? wbuf[wi][lane] : 0;
    const int src = id / (int)m.CAPS;
    const int64_t j = id - (int64_t)src * m.CAPS;
    Rec r{};
    bool push = false;
    if (have) { r = base[id]; push = j < m.qpush[src]; }
    // U4(t-1): eviction pushes raise c_g (max is order-free); L3: condition (2)
    // for clock-checked hits against c_g after them; L4: sync pushes of the
    // requests that are not valid hits
    uint32_t g = g0;
    const unsigned pushm = __ballot_sync(0xffffffffu, have && push);
    {
      uint32_t x = (have && push) ? r.cc : 0u;
      for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
      g = max(g, x);
    }
    const bool req = have && !push;
    const bool valid = req && (r.kind & 3) == K_NEEDQ && (g <= r.cc || g - r.cc <= s.s);
    const unsigned validm = __ballot_sync(0xffffffffu, valid);
    const bool syncp = req && !valid && (r.kind & K_DIRTY);
    const unsigned syncm = __ballot_sync(0xffffffffu, syncp);
    {
      uint32_t x = syncp ? r.cc : 0u;
      for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
      g = max(g, x);
    }
    if (lane == 0 && lead) s.cg[row] = g;
    // byte counters: pushes received, requests received / answered
    if (have && lead) {
      if (push) atomicAdd(&sb[3], 16ull + 4ull * s.D);
      else {
        atomicAdd(&sb[(r.kind & 3) == K_NEEDQ ? 1 : 3], 16ull);
        if (r.kind & K_DIRTY) atomicAdd(&sb[3], 4ull * s.D);
        atomicAdd(&sb[valid ? 0 : 2], valid ? 8ull : 8ull + 4ull * s.D);
      }
    }
    // response headers: (c_g, valid) straight into the requester's inbox (L5)
    float* rec_l = nullptr;
    if (req) {
      rec_l = resprec(m, src, m.rank, j - m.qpush[src]);
      if (lead) {
        reinterpret_cast<uint32_t*>(rec_l)[0] = g;
        reinterpret_cast<uint32_t*>(rec_l)[1] = valid ? 1u : 0u;
      }
    }
    PTL(13);
    // row data, lane per float4, records in sorted order: pushes, then sync pushes
    const unsigned needrow = (pushm | syncm);
    const unsigned answer = __ballot_sync(0xffffffffu, req && !valid);
    float4* Wr = reinterpret_cast<float4*>(s.W + row * s.D);
    for (int d0 = c0 + lane; d0 - lane < c1; d0 += 32 * RB) {   // RB columns per lane per pass (wide rows)
      float4 w[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b)
        w[b] = (d0 == c0 + lane && b == 0) ? wpre : (d0 + 32 * b < c1 ? Wr[d0 + 32 * b] : make_float4(0.f, 0.f, 0.f, 0.f));
      for (int pass = 0; pass < 2; ++pass) {
        unsigned mm = pass == 0 ? pushm : syncm;
        while (mm) {
          const int i = __ffs(mm) - 1;
          mm &= mm - 1;
          const int si = __shfl_sync(0xffffffffu, src, i);
          const int64_t ji = __shfl_sync(0xffffffffu, j, i);
          const float4* rr = reinterpret_cast<const float4*>(reqrow(m, m.rank, si, ji));
          float4 x[RB];
#pragma unroll
          for (int b = 0; b < RB; ++b) if (d0 + 32 * b < c1) x[b] = rr[d0 + 32 * b];
#pragma unroll
          for (int b = 0; b < RB; ++b) if (d0 + 32 * b < c1) w[b] = f4add_p(w[b], x[b]);
        }
      }
      if (needrow) {
#pragma unroll
        for (int b = 0; b < RB; ++b) if (d0 + 32 * b < c1) Wr[d0 + 32 * b] = w[b];
      }
      unsigned am = answer;
      while (am) {
        const int i = __ffs(am) - 1;
        am &= am - 1;
        float* rec = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rec_l), i));
#pragma unroll
        for (int b = 0; b < RB; ++b)
          if (d0 + 32 * b < c1) reinterpret_cast<float4*>(rec + 4)[d0 + 32 * b] = w[b];
      }
    }
    PTL(14);
    __syncwarp();
  }
}

// the row lists of this round's leaders, emptied for the next round's link
// (after every warp of the phase walked them); thread-strided over the grid
__device__ __forceinline__ void reset_heads(const P2P& m, int nl) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) m.head[m.leaders[i]] = -1;
}

__global__ void k_p2p_process(Dev s, P2P m) {
  __shared__ unsigned long long sb[4];
  bytes_init(sb);
  PTL(6);
  __syncthreads();
  const unsigned long long ep = *m.epoch + 1;
  process_rows(s, m, sb);
  PTL(7);
  __syncthreads();
  bytes_flush(s, sb);
  if (!last_block(&m.done[1])) return;
  if (threadIdx.x < m.N) {
    __threadfence_system();
    st_release(&respflag(m, threadIdx.x)[m.rank].epoch, ep);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < *m.nlead; i += blockDim.x) m.head[m.leaders[i]] = -1;   // every block has walked
  __syncthreads();
  if (threadIdx.x == 0) { *m.nlead = 0; m.done[1] = 0; }
  PTL(8);
}

// ---------------------------------------------------------------- requester: wait + install
__global__ void k_p2p_install(Dev s, Call c, P2P m) {
  __shared__ int s_ok;
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned bc[2];
  __shared__ int32_t lc[64];
  __shared__ unsigned long long sb[4];
  const unsigned long long ep = *m.epoch + 1;
  bytes_init(sb);
  dpop_init(dpop);
  if (threadIdx.x < 2) bc[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_ok = wait_flags(respflag(m, m.rank), m.N, ep, s.ctl);
  if (threadIdx.x < m.N) lc[threadIdx.x] = m.lcnt[threadIdx.x];
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int D4 = s.D >> 2;
  if (s_ok && !ctl->abort) {
    for (int o = 0; o < m.N; ++o) {
      for (int j = gw; j < lc[o]; j += nw) {
        const int u = m.ridx[(int64_t)o * m.CAPS + j];
        const float* rec = resprec(m, m.rank, o, j);
        const uint32_t g = reinterpret_cast<const uint32_t*>(rec)[0];
        const bool valid = reinterpret_cast<const uint32_t*>(rec)[1] != 0;
        const uint8_t st = c.status[u];
        if (lane == 0) atomicAdd(&sb[valid ? 1 : 3], valid ? 8ull : 8ull + 4ull * s.D);
        if (st == ST_NEEDQ) {
          if (lane == 0) {
            c.status[u] = valid ? ST_HIT : ST_EXP2;
            atomicAdd(&bc[valid ? 0 : 1], 1u);
          }
          if (valid) continue;
        }
        const int64_t key = c.uniq[u];
        int32_t e;
        if (st == ST_MISS) {
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
            const uint32_t prim = s.policy == 0 ? (s.lfu_persist ? s.count_by_key[key] : 1u) : (uint32_t)ctl->t_cur;
            s.eprim[e] = prim;
            if (s.policy == 0) { lfu_move(s, key, EP_FREE, prim, dpop); pin_candidate(s, key, e, prim); }
            atomicMin(&ctl->min_install, prim);
            c.uentry[u] = e;
          }
        } else {
          e = c.uentry[u];
        }
        warp_copy_row(reinterpret_cast<float4*>(s.v + (int64_t)e * s.D), reinterpret_cast<const float4*>(rec + 4),
                      D4, lane);
        if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
      }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  bytes_flush(s, sb);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[1]);
  }
  if (!last_block(&m.done[2])) return;
  if (threadIdx.x < m.N) m.lcnt[threadIdx.x] = 0;   // every block read it at entry; zero for the next round
  if (threadIdx.x == 0) { *m.epoch = ep; m.done[2] = 0; }
}

// ---------------------------------------------------------------- requester: eviction pushes
// overflow victims (keys or entries from the selection) -> PUSH records in the
// owners' inboxes, then delete + free locally.  Sent with the next round.
struct EvView {  // leading fields of EvBuf
  uint32_t* hist; uint32_t* khist; int32_t* victims; int32_t* cand; int32_t* sub; int32_t* flags;
  int64_t* vkeys; uint8_t* vdirty; int64_t* vsel;
};

__global__ void k_p2p_pushes(Dev s, P2P m, EvView b) {
  __shared__ unsigned long long sb[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty, s_ev;
  dpop_init(dpop);
  bytes_init(sb);
  if (threadIdx.x == 0) { s_dirty = 0; s_ev = 0; }
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int D4 = s.D >> 2;
  const int count = (!ctl->abort && ctl->need > 0) ? ctl->nvict : 0;
  for (int i = gw; i < count; i += nw) {
    const int64_t key = ctl->vmode == 1 ? b.vsel[i] : s.ekey[b.victims[i]];
    uint64_t slot = 0;
    const int32_t e = warp_find_slot(s, key, lane, &slot);
    if (e < 0) continue;
    const uint32_t ecc = s.cc[e], ecs = s.cs[e], prim = s.eprim[e];
    const bool dirty = ecc > ecs;
    if (dirty) {
      const int o = (int)(key % m.N);
      int ps = 0;
      if (lane == 0) ps = atomicAdd(&m.c3cnt[o], 1);
      ps = __shfl_sync(0xffffffffu, ps, 0);
      if (lane == 0) {
        Rec r;
        r.key = key; r.cc = ecc; r.kind = K_PUSH | K_DIRTY;
        reqrec(m, o, m.rank)[ps] = r;
        atomicAdd(&sb[2], 16ull + 4ull * s.D);
      }
      warp_copy_row(reinterpret_cast<float4*>(reqrow(m, o, m.rank, ps)),
                    reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D), D4, lane);
    }
    if (lane == 0) {
      s.hslot[slot] = HS_TOMB;
      atomicAdd(&ctl->n_tomb, 1);
      b.vkeys[i] = key;
      b.vdirty[i] = dirty ? 1 : 0;
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
  bytes_flush(s, sb);
  if (threadIdx.x == 0) {
    if (s_ev) atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)s_ev);
    if (s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
  }
}

// ---------------------------------------------------------------- fused round (n <= 8192)
// probe + request build (warp per unique key; rmode: per sorted position,
// non-heads skip), in two phases around a block barrier so that the request
// slots in each owner's inbox are reserved with one atomic per (block, owner)
// instead of one per key (thousands of records per owner per round):
//  A: Cache.Find, condition (1), the LFU/LRU touch, the inverse and the
//     lookup -> update record; a request takes a block-local slot
//  B: the record (+ pending row of a dirty entry) straight into the owner's
//     inbox at its reserved slot
struct PBKey {            // phase A -> phase B (warp-uniform)
  int64_t key;
  int32_t e;
  uint32_t ecc;
  int32_t o;              // owner, -1: no request
  int32_t lslot;          // block-local slot among this block's requests to o
  uint8_t st;
  bool dirty;
};

__device__ __forceinline__ PBKey probe_build_a(const Dev& s, const Call& c, const P2P& m, int u, int lane,
                                               unsigned* bc, int* dpop, int* s_cnt, float* __restrict__ out) {
  Ctl* ctl = s.ctl;
  PBKey k{};
  k.o = -1;
  int64_t key;
  int j0, cnt, pos_lane;
  if (c.rmode) {
    if (!key_run(c, u, lane, &key, &cnt, &pos_lane)) {   // not the key's first sorted position
      if (lane == 0) { c.urec[u].x = -1; c.status[u] = ST_SKIP; }
      k.st = ST_SKIP;
      return k;
    }
    j0 = u;
  } else {
    key = c.uniq[u];
    j0 = c.seg_off[u];
    cnt = c.seg_off[u + 1] - j0;
    pos_lane = lane < cnt ? c.perm[j0 + lane] : 0;
  }
  uint32_t cntk = 0;
  if (lane == 0 && s.lfu_persist) cntk = s.count_by_key[key];
  uint64_t cslot = ~0ull, cword = 0;
  const int32_t e = warp_find_cand(s, key, lane, &cslot, &cword);
  uint32_t ecs = 0, ecc = 0;
  if (e >= 0) { ecs = s.cs[e]; ecc = s.cc[e]; }
  else if (lane == 0) { c.ucslot[u] = cslot; c.ucword[u] = cword; }   // the install's CAS slot
  uint8_t st = ST_MISS;
  if (lane == 0) {
    const uint32_t oldc = (e >= 0 && s.policy == 0) ? s.eprim[e] : 0u;
    const bool pinned = oldc == EP_PIN;                    // light-LFU: no frequency maintenance
    if (s.lfu_persist && !pinned) { cntk += 1; s.count_by_key[key] = cntk; }
    if (e >= 0) {
      if (s.s == S_INF) st = ST_HIT;                       // R4
      else if (ecc - ecs > s.s) st = ST_EXP1;              // cond (1)
      else st = ST_NEEDQ;                                  // cond (2) at the owner
      if (s.policy == 0) {
        if (!pinned) {
          uint32_t newc = s.lfu_persist ? cntk : oldc + 1;
          s.eprim[e] = newc;
          lfu_move(s, key, oldc, newc, dpop);
          pin_candidate(s, key, e, newc);
        }
      } else {
        s.eprim[e] = (uint32_t)ctl->t_cur;
      }
    }
    c.status[u] = st;
    c.uentry[u] = e;
    atomicAdd(&bc[st == ST_HIT ? 0 : st == ST_EXP1 ? 1 : st == ST_MISS ? 3 : 2], 1u);   // 2: NEEDQ (finished at install)
  }
  st = __shfl_sync(0xffffffffu, st, 0);
  for (int q = lane; q < cnt; q += 32) c.inverse[q < 32 ? pos_lane : c.perm[j0 + q]] = u;
  write_urec(c, u, e, j0, cnt, ecc > ecs, ecc, pos_lane, lane);   // resident: a hit keeps it, a refetch rewrites it
  if (c.rmode && lane == 0) { c.uniq[u] = key; c.ucnt[u] = cnt; }   // for the install phase
  k.key = key; k.e = e; k.ecc = ecc; k.st = st;
  if ((st == ST_HIT || st == ST_NEEDQ) && !(c.rmode && wide_rows(s.D))) {   // wide: launch_scatter_wide
    // Cache.Get now: a hit's row, and a clock-checked hit's row (the
    // install overwrites the occurrences of the rare one condition (2) refuses)
    const int D4 = s.D >> 2;
    const float4* vr = reinterpret_cast<const float4*>(s.v + (int64_t)e * s.D);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (int d0 = lane; d0 - lane < D4; d0 += 32 * RB) {   // RB columns per lane in flight (wide rows)
      float4 val[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) val[b] = d0 + 32 * b < D4 ? vr[d0 + 32 * b] : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int kb = 0; kb < cnt; kb += 32) {
        const int srcp = kb == 0 ? pos_lane : (kb + lane < cnt ? c.perm[j0 + kb + lane] : 0);
        const int mm = min(32, cnt - kb);
        for (int q = 0; q < mm; ++q) {
          const int pos = __shfl_sync(0xffffffffu, srcp, q);
#pragma unroll
          for (int b = 0; b < RB; ++b)
            if (d0 + 32 * b < D4) __stcs(o4 + (int64_t)pos * D4 + d0 + 32 * b, val[b]);
        }
      }
    }
  }
  if (st != ST_HIT) {
    k.o = (int)(key % m.N);
    k.dirty = e >= 0 && ecc > ecs;
    int ls = 0;
    if (lane == 0) ls = atomicAdd(&s_cnt[k.o], 1);
    k.lslot = __shfl_sync(0xffffffffu, ls, 0);
  }
  return k;
}

__device__ __forceinline__ void probe_build_b(const Dev& s, const Call& c, const P2P& m, int u, int lane,
                                              const PBKey& k, const int* s_base, unsigned long long* sb) {
  if (k.o < 0) return;
  const int D4 = s.D >> 2;
  const int slot = s_base[k.o] + k.lslot;
  const int64_t j = m.c3cnt[k.o] + slot;
  if (lane == 0) {
    Rec r;
    r.key = k.key; r.cc = k.ecc;
    r.kind = (k.st == ST_NEEDQ ? K_NEEDQ : k.st == ST_EXP1 ? K_EXP1 : K_MISS) | (k.dirty ? K_DIRTY : 0);
    HET_ASSERT(j >= 0 && j < m.CAPS);
    reqrec(m, k.o, m.rank)[j] = r;
    m.uslot[u] = (int32_t)(k.o * m.CAPS + slot);
    atomicAdd(&sb[k.st == ST_NEEDQ ? 0 : 2], 16ull);
    if (k.dirty) atomicAdd(&sb[2], 4ull * s.D);
  }
  if (k.dirty)
    warp_copy_row(reinterpret_cast<float4*>(reqrow(m, k.o, m.rank, j)),
                  reinterpret_cast<const float4*>(s.p + (int64_t)k.e * s.D), D4, lane);
}

// every warp of the block takes keys u = base + warp, base over the grid in
// steps of gridDim * warps-per-block (the same trip count in every warp, so
// the block barriers line up)
__device__ __forceinline__ void probe_build_all(const Dev& s, const Call& c, const P2P& m, int U, unsigned* bc,
                                                int* dpop, unsigned long long* sb, float* __restrict__ out) {
  __shared__ int s_cnt[P2P_MAX_WORLD], s_base[P2P_MAX_WORLD];
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  if (threadIdx.x < P2P_MAX_WORLD) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int base = blockIdx.x * wpb; base < U; base += gridDim.x * wpb) {
    const int u = base + (threadIdx.x >> 5);
    PBKey k{};
    k.o = -1;
    if (u < U) k = probe_build_a(s, c, m, u, lane, bc, dpop, s_cnt, out);
    __syncthreads();
    if (threadIdx.x < m.N) {
      s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&m.lcnt[threadIdx.x], s_cnt[threadIdx.x]) : 0;
      s_cnt[threadIdx.x] = 0;
    }
    __syncthreads();
    if (u < U) probe_build_b(s, c, m, u, lane, k, s_base, sb);
  }
}

__device__ __forceinline__ void probe_build_flush(const Dev& s, const Call& c, unsigned* bc, int* dpop,
                                                  unsigned long long* sb, int U) {
  dpop_flush(s, dpop);
  bytes_flush(s, sb);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP1], (unsigned long long)bc[1]);
    if (bc[3]) atomicAdd(&s.cnt[C_MISSES], (unsigned long long)bc[3]);
    if (c.rmode) {   // heads of this block: hits + exp1 + misses + clock-checked (finished at install)
      const unsigned nu = bc[0] + bc[1] + bc[2] + bc[3];
      if (nu) atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)nu);
    } else if (blockIdx.x == 0 && !s.ctl->abort) {
      atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)U);
    }
  }
}

// the round's request flags: records to owner o = carried pushes + requests
__device__ __forceinline__ void publish_requests(const P2P& m, unsigned long long ep) {
  if (threadIdx.x < m.N) {
    const int o = threadIdx.x;
    Flag* f = &reqflag(m, o)[m.rank];
    f->total = (uint32_t)(m.c3cnt[o] + m.lcnt[o]);
    f->pushes = (uint32_t)m.c3cnt[o];
    __threadfence_system();
    st_release(&f->epoch, ep);
    m.c3cnt[o] = 0;
    m.lcnt[o] = 0;   // counted; zero for the next round (no memset node in the step graph)
  }
}

__global__ void __launch_bounds__(256)
k_probe_build(Dev s, Call c, P2P m, float* __restrict__ out) {
  __shared__ unsigned bc[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned long long sb[4];
  PTL(0);
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  dpop_init(dpop);
  bytes_init(sb);
  __syncthreads();
  Ctl* ctl = s.ctl;
  const unsigned long long ep = *m.epoch + 1;
  const int U = ctl->abort ? 0 : (c.rmode ? c.n : ctl->U);
  probe_build_all(s, c, m, U, bc, dpop, sb, out);
  __syncthreads();
  probe_build_flush(s, c, bc, dpop, sb, U);
  PTL(1);
  if (!last_block(&m.done[0])) return;
  publish_requests(m, ep);
  if (threadIdx.x == 0) m.done[0] = 0;
  PTL(2);
}

// install + gather for one unique key (warp): finish the status of a
// clock-checked hit from the owner's answer, install a fetched row, scatter
// the key's row to its occurrences (Cache.Get)
// mnext: this warp's next index into its block's free-stack reservation
// (misses in u order, descending); nullptr: one atomic pop per miss
__device__ __forceinline__ void install_gather_key(const Dev& s, const Call& c, const P2P& m, int u, int lane,
                                                   float* __restrict__ out, unsigned* bc, int* dpop,
                                                   unsigned long long* sb, int* mnext = nullptr) {
  Ctl* ctl = s.ctl;
  const int D4 = s.D >> 2;
  uint8_t st = c.status[u];
  if (st == ST_SKIP) return;   // rmode: not a key's first sorted position
  int32_t e = c.uentry[u];
  const int64_t key = c.uniq[u];
  const int j0 = c.rmode ? u : c.seg_off[u];
  const int cnt = c.rmode ? c.ucnt[u] : c.seg_off[u + 1] - j0;
  const int pos_lane = lane < cnt ? c.perm[j0 + lane] : 0;
  bool ok = true;
  if (st != ST_HIT) {
    const int loc = m.uslot[u];
    const int o = loc / (int)m.CAPS;
    const float* rec = resprec(m, m.rank, o, loc - o * m.CAPS);
    const uint32_t g = reinterpret_cast<const uint32_t*>(rec)[0];
    const bool valid = reinterpret_cast<const uint32_t*>(rec)[1] != 0;
    if (lane == 0) atomicAdd(&sb[valid ? 1 : 3], valid ? 8ull : 8ull + 4ull * s.D);
    if (st == ST_NEEDQ) {
      if (lane == 0) { c.status[u] = valid ? ST_HIT : ST_EXP2; atomicAdd(&bc[valid ? 0 : 1], 1u); }
    }
    if (!(st == ST_NEEDQ && valid)) {
      if (st == ST_MISS) {
        int32_t idx = 0;
        if (mnext) {
          idx = (*mnext)--;                   // warp-uniform: the block reserved these entries
        } else {
          if (lane == 0) idx = atomicSub(&ctl->ftop, 1) - 1;
          idx = __shfl_sync(0xffffffffu, idx, 0);
        }
        if (idx < 0) {
          if (lane == 0) raise_err(ctl, 4);
          ok = false;
        } else {
          HET_ASSERT(idx >= 0 && idx < s.Ecap);
          e = s.fstack[idx];
          HET_ASSERT(e >= 0 && e < s.Ecap);
          warp_insert_at(s, key, e, lane, c.ucslot[u], c.ucword[u]);
          if (lane == 0) {
            s.ekey[e] = key;
            const uint32_t prim = s.policy == 0 ? (s.lfu_persist ? s.count_by_key[key] : 1u) : (uint32_t)ctl->t_cur;
            s.eprim[e] = prim;
            if (s.policy == 0) { lfu_move(s, key, EP_FREE, prim, dpop); pin_candidate(s, key, e, prim); }
            atomicMin(&ctl->min_install, prim);
            c.uentry[u] = e;
          }
        }
      }
      if (ok) {
        if (!(c.rmode && wide_rows(s.D)))   // wide rows: launch_scatter_wide copies the response row
          warp_copy_row(reinterpret_cast<float4*>(s.v + (int64_t)e * s.D), reinterpret_cast<const float4*>(rec + 4),
                        D4, lane);
        if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
        write_urec(c, u, e, j0, cnt, false, g, pos_lane, lane);   // fetched: clean, c_c = c_g
      }
    }
  }
  bool fresh = st != ST_HIT;   // the probe already scattered hits and clock-checked hits condition (2) kept
  if (st == ST_NEEDQ) fresh = reinterpret_cast<const uint32_t*>(
                                  resprec(m, m.rank, m.uslot[u] / (int)m.CAPS, m.uslot[u] % (int)m.CAPS))[1] == 0;
  if (ok && e >= 0 && fresh && !(c.rmode && wide_rows(s.D))) {   // wide rows: launch_scatter_wide after the round
    const float4* vr = reinterpret_cast<const float4*>(s.v + (int64_t)e * s.D);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (int d0 = lane; d0 - lane < D4; d0 += 32 * RB) {
      float4 val[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) val[b] = d0 + 32 * b < D4 ? vr[d0 + 32 * b] : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int kb = 0; kb < cnt; kb += 32) {
        const int srcp = kb == 0 ? pos_lane : (kb + lane < cnt ? c.perm[j0 + kb + lane] : 0);
        const int mm = min(32, cnt - kb);
        for (int k = 0; k < mm; ++k) {
          const int pos = __shfl_sync(0xffffffffu, srcp, k);
#pragma unroll
          for (int b = 0; b < RB; ++b)
            if (d0 + 32 * b < D4) __stcs(o4 + (int64_t)pos * D4 + d0 + 32 * b, val[b]);
        }
      }
    }
  }
}

__device__ __forceinline__ void install_gather_flush(const Dev& s, unsigned* bc, int* dpop, unsigned long long* sb) {
  dpop_flush(s, dpop);
  bytes_flush(s, sb);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[1]);
  }
}

__global__ void __launch_bounds__(256)
k_install_gather(Dev s, Call c, P2P m, float* __restrict__ out) {
  __shared__ int s_ok;
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned bc[2];
  __shared__ unsigned long long sb[4];
  const unsigned long long ep = *m.epoch + 1;
  dpop_init(dpop);
  bytes_init(sb);
  if (threadIdx.x < 2) bc[threadIdx.x] = 0;
  PTL(9);
  if (threadIdx.x == 0) s_ok = wait_flags(respflag(m, m.rank), m.N, ep, s.ctl);
  __syncthreads();
  PTL(10);
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int U = (s_ok && !ctl->abort) ? (c.rmode ? c.n : ctl->U) : 0;
  if (u < U) install_gather_key(s, c, m, u, lane, out, bc, dpop, sb);
  __syncthreads();
  install_gather_flush(s, bc, dpop, sb);
  if (!last_block(&m.done[2])) return;
  if (threadIdx.x == 0) { *m.epoch = ep; m.done[2] = 0; }
}

// ---------------------------------------------------------------- the whole round, one cooperative kernel
constexpr int EX_THREADS = 1024;   // 32 warps per SM: a WDL-sized batch's keys in one pass per phase
// One block per SM (so concurrent NCCL kernels always find room: no
// cross-GPU resource cycle), grid syncs between the phases instead of kernel
// boundaries.  Every block reaches every grid sync (no early returns).
__global__ void __launch_bounds__(EX_THREADS)
k_exchange(Dev s, Call c, P2P m, float* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: launched while the dedup runs
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned bc[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned long long sb[4];
  __shared__ int s_ok;
  __shared__ int32_t tot[64];
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long ep = *m.epoch + 1;
  // ---- requester: probe + build
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  dpop_init(dpop);
  bytes_init(sb);
  __syncthreads();
  PTL(0);
  const int U = ctl->abort ? 0 : (c.rmode ? c.n : ctl->U);   // rmode: sorted positions, heads carry the work
  probe_build_all(s, c, m, U, bc, dpop, sb, out);
  __syncthreads();
  probe_build_flush(s, c, bc, dpop, sb, U);
  PTL(1);
  __threadfence();
  grid.sync();
  if (blockIdx.x == 0) publish_requests(m, ep);
  PTL(2);
  // ---- owner: wait for every source, link
  PTL(3);
  if (threadIdx.x == 0) s_ok = wait_flags(reqflag(m, m.rank), m.N, ep, ctl);
  __syncthreads();
  PTL(4);
  const bool ok1 = s_ok;
  if (threadIdx.x < m.N) {
    const Flag* flags = reqflag(m, m.rank);
    tot[threadIdx.x] = ok1 ? (int32_t)flags[threadIdx.x].total : 0;
    if (blockIdx.x == 0) {
      m.qtot[threadIdx.x] = ok1 ? (int32_t)flags[threadIdx.x].total : 0;
      m.qpush[threadIdx.x] = ok1 ? (int32_t)flags[threadIdx.x].pushes : 0;
    }
  }
  bytes_init(sb);
  __syncthreads();
  link_records(m, tot);
  PTL(5);
  grid.sync();
  // ---- owner: apply + respond
  PTL(6);
  const int nlr = *m.nlead;   // this round's leaders (block 0 zeroes the counter after the next grid sync)
  process_rows(s, m, sb);
  PTL(7);
  __syncthreads();
  bytes_flush(s, sb);
  __threadfence();
  grid.sync();
  reset_heads(m, nlr);   // every warp has walked its rows' lists
  if (blockIdx.x == 0) {
    if (threadIdx.x < m.N) {
      __threadfence_system();
      st_release(&respflag(m, threadIdx.x)[m.rank].epoch, ep);
    }
    if (threadIdx.x == 0) *m.nlead = 0;
  }
  PTL(8);
  // ---- requester: wait for every owner, install + gather
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  dpop_init(dpop);
  bytes_init(sb);
  PTL(9);
  if (threadIdx.x == 0) s_ok = wait_flags(respflag(m, m.rank), m.N, ep, ctl);
  __syncthreads();
  PTL(10);
  const int U2 = (s_ok && !ctl->abort) ? (c.rmode ? c.n : ctl->U) : 0;
  {
    // the block's misses take one free-stack reservation (one atomic per
    // block instead of one per miss: the Reddit-shaped batches miss ~7K keys)
    __shared__ int s_mcount, s_mbase;
    if (threadIdx.x == 0) s_mcount = 0;
    __syncthreads();
    int my = 0;
    for (int i0 = 0; gw + i0 * nw < U2; i0 += 32) {
      const int uu = gw + (i0 + lane) * nw;
      my += __popc(__ballot_sync(0xffffffffu, uu < U2 && c.status[uu] == ST_MISS));
    }
    int woff = 0;
    if (lane == 0 && my) woff = atomicAdd(&s_mcount, my);
    woff = __shfl_sync(0xffffffffu, woff, 0);
    __syncthreads();
    if (threadIdx.x == 0 && s_mcount) s_mbase = atomicSub(&ctl->ftop, s_mcount);
    __syncthreads();
    int mnext = s_mbase - 1 - woff;
    for (int u = gw; u < U2; u += nw) install_gather_key(s, c, m, u, lane, out, bc, dpop, sb, &mnext);
  }
  PTL(11);
  __syncthreads();
  install_gather_flush(s, bc, dpop, sb);
  // every block read the epoch at entry, before three grid syncs: block 0 can
  // advance it without a fence (the next round is ordered by the kernel boundary)
  if (blockIdx.x == 0 && threadIdx.x == 0) *m.epoch = ep;
}

// ---------------------------------------------------------------- host side
// ---------------------------------------------------------------- dense all-reduce over peer memory
// Eq. 2: buf <- mean over the N workers.  Every rank stages its
// buffer in an IPC-exported region (two buffers by epoch parity), publishes
// an epoch flag into every peer's flag array, and then each rank sums ALL
// staged buffers itself in rank order (one-shot: every rank computes the same
// fp32 sums in the same order, so the result is bitwise identical on every
// rank).  A second flag ("done reading epoch e") guards the reuse of a
// staging buffer two epochs later.  No grid-wide barrier: last-block
// election publishes, every block waits for the peers before its share of
// the sum; the grid (coop_sm_reserve() blocks) fits in the SMs the
// cooperative hot-path kernels leave free, so a spinning block never starves
// a peer's kernel.
struct DenseView {
  int N, rank;
  char* const* peer;            // [N] dense-region bases (own included)
  uint64_t cap;                 // floats per staging buffer
  unsigned long long* epoch;    // completed all-reduces (device)
  int32_t* done;                // [2] last-block counters
};
__device__ __forceinline__ Flag* dready(const DenseView& v, int r) { return (Flag*)v.peer[r]; }
__device__ __forceinline__ Flag* ddone(const DenseView& v, int r) { return (Flag*)v.peer[r] + 64; }
__device__ __forceinline__ float* dbuf(const DenseView& v, int r, int par) {
  return (float*)(v.peer[r] + 2 * 64 * sizeof(Flag)) + (uint64_t)par * v.cap;
}

// phase 0: the whole all-reduce (one process per GPU: every wait is for
// another GPU's kernel); phase 1: stage + publish only; phase 2: wait + sum
// only.  The loopback driver (one GPU, N workers) runs phase 1 of every
// worker before phase 2 of any, so no wait ever spins.
__global__ void __launch_bounds__(512) k_dense_ar(DenseView v, float* __restrict__ buf, uint64_t count,
                                                  float scale, Ctl* ctl, int phase) {
  __shared__ int s_ok;
  const unsigned long long e = *v.epoch + 1;
  const int par = (int)(e & 1);
  const uint64_t n4 = count / 4;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
  constexpr int U = 8;   // float4 per thread in flight (peer reads cross NVLink: latency-bound)
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (phase != 2) {
    // staging buffer `par` is free once every peer finished reading epoch e - 2
    if (threadIdx.x == 0) s_ok = e <= 2 || wait_flags(ddone(v, v.rank), v.N, e - 2, ctl);
    __syncthreads();
    float4* mine = reinterpret_cast<float4*>(dbuf(v, v.rank, par));
    if (s_ok) {
      const float4* b4 = reinterpret_cast<const float4*>(buf);
      for (uint64_t i0 = tid; i0 < n4; i0 += U * nth) {
        float4 t[U];
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * nth < n4) t[k] = b4[i0 + k * nth];
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * nth < n4) mine[i0 + k * nth] = t[k];
      }
      for (uint64_t i = n4 * 4 + tid; i < count; i += nth) ((float*)mine)[i] = buf[i];
    }
    if (last_block(&v.done[0]) && threadIdx.x < v.N) {   // fence.sys done by last_block
      st_release(&dready(v, threadIdx.x)[v.rank].epoch, e);
      if (threadIdx.x == 0) v.done[0] = 0;
    }
    if (phase == 1) return;
  }
  if (threadIdx.x == 0) s_ok = s_ok && wait_flags(dready(v, v.rank), v.N, e, ctl);
  __syncthreads();
  if (s_ok) {
    for (uint64_t i0 = tid; i0 < n4; i0 += U * nth) {
      float4 a[U];
      const float4* s0 = reinterpret_cast<const float4*>(dbuf(v, 0, par));
#pragma unroll
      for (int k = 0; k < U; ++k) if (i0 + k * nth < n4) a[k] = s0[i0 + k * nth];
      for (int r = 1; r < v.N; ++r) {              // rank order: the same sums on every rank
        const float4* sr = reinterpret_cast<const float4*>(dbuf(v, r, par));
        float4 x[U];
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * nth < n4) x[k] = sr[i0 + k * nth];
#pragma unroll
        for (int k = 0; k < U; ++k) a[k] = f4add_p(a[k], x[k]);
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (i0 + k * nth < n4)
          reinterpret_cast<float4*>(buf)[i0 + k * nth] = make_float4(
              __fmul_rn(a[k].x, scale), __fmul_rn(a[k].y, scale), __fmul_rn(a[k].z, scale), __fmul_rn(a[k].w, scale));
    }
    for (uint64_t i = n4 * 4 + tid; i < count; i += nth) {
      float a = dbuf(v, 0, par)[i];
      for (int r = 1; r < v.N; ++r) a = __fadd_rn(a, dbuf(v, r, par)[i]);
      buf[i] = __fmul_rn(a, scale);
    }
  }
  if (last_block(&v.done[1])) {
    if (threadIdx.x < v.N) st_release(&ddone(v, threadIdx.x)[v.rank].epoch, e);
    if (threadIdx.x == 0) { v.done[1] = 0; *v.epoch = e; }
  }
}

// ---------------------------------------------------------------- flush / explicit evict (pushes only)
// het_sync (R16): every dirty resident entry with key in [k0, k1)
// sends a PUSH record {key, c_c} + its pending row to the owner's inbox at the
// source's push cursor; the next drain round applies them (per row in source
// rank order, so the key ranges keep every worker's push of a key in one round).
__global__ void k_p2p_flush_build(Dev s, P2P m, int64_t k0, int64_t k1) {
  __shared__ unsigned long long sb[4];
  bytes_init(sb);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t e0 = (int64_t)w * 32; e0 < s.Ecap; e0 += (int64_t)nw * 32) {
    const int64_t e = e0 + lane;
    const int64_t key = e < s.Ecap ? s.ekey[e] : -1;
    const bool pick = key >= k0 && key < k1 && s.cc[e] > s.cs[e];
    unsigned mk = __ballot_sync(0xffffffffu, pick);
    while (mk) {
      const int src = __ffs(mk) - 1;
      mk &= mk - 1;
      const int64_t k = __shfl_sync(0xffffffffu, key, src);
      const int32_t ee = (int32_t)(e0 + src);
      push_record(s, m, ee, k, s.cc[ee], lane);
      if (lane == 0) atomicAdd(&sb[2], 16ull + 4ull * s.D);
    }
  }
  __syncthreads();
  bytes_flush(s, sb);
}

// Cache.Evict(key) of the call's unique keys at N > 1: a resident
// dirty entry sends its PUSH record (delivered by the next drain round), then
// delete + free.  Warp per unique key.
__global__ void k_p2p_evict_keys(Dev s, Call c, P2P m) {
  __shared__ unsigned long long sb[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty, s_ev;
  bytes_init(sb);
  dpop_init(dpop);
  if (threadIdx.x == 0) { s_dirty = 0; s_ev = 0; }
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (!ctl->abort && u < ctl->U) {
    const int64_t key = c.uniq[u];
    uint64_t slot = 0;
    const int32_t e = warp_find_slot(s, key, lane, &slot);
    if (e >= 0) {
      const uint32_t ecc = s.cc[e], ecs = s.cs[e], prim = s.eprim[e];
      const bool dirty = ecc > ecs;
      if (dirty) push_record(s, m, e, key, ecc, lane);
      if (lane == 0) {
        if (dirty) atomicAdd(&sb[2], 16ull + 4ull * s.D);
        s.hslot[slot] = HS_TOMB;
        atomicAdd(&ctl->n_tomb, 1);
        if (s.policy == 0) lfu_move(s, key, prim, EP_FREE, dpop);
        unpin_count(s, prim);
        s.eprim[e] = EP_FREE;
        s.ekey[e] = -1;
        s.fstack[atomicAdd(&ctl->ftop, 1)] = e;
        atomicAdd(&s_ev, 1u);
        if (dirty) atomicAdd(&s_dirty, 1u);
      }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  bytes_flush(s, sb);
  if (threadIdx.x == 0) {
    if (s_ev) atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)s_ev);
    if (s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
  }
}

struct P2PState {
  P2P v{};
  char* inbox = nullptr;
  std::vector<char*> mapped;     // opened peer bases (to close)
  std::vector<void*> allocs;
  bool loopback = false;         // N workers on one device: plain pointers, no IPC
  // dense all-reduce staging (allocated at create; nullptr = NCCL fallback)
  char* dense = nullptr;
  DenseView dv{};
};

template <typename T>
static bool p_alloc(P2PState* p, T** q, size_t count) {
  void* x = nullptr;
  if (cudaMalloc(&x, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) return false;
  p->allocs.push_back(x);
  *q = reinterpret_cast<T*>(x);
  return true;
}

// IPC export of one allocation, import of every peer's (collective over comm)
static het_status_t exchange_bases(P2PState* p, char* mine_base, int N, int rank, ncclComm_t comm,
                                   cudaStream_t st, char** dbases) {
  cudaIpcMemHandle_t mine;
  if (cudaIpcGetMemHandle(&mine, mine_base) != cudaSuccess) return HET_ERR_CUDA;
  char* dh;
  if (cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * N) != cudaSuccess) return HET_ERR_OOM;
  cudaMemcpyAsync(dh + sizeof(cudaIpcMemHandle_t) * rank, &mine, sizeof(mine), cudaMemcpyHostToDevice, st);
  if (ncclAllGather(dh + sizeof(cudaIpcMemHandle_t) * rank, dh, sizeof(cudaIpcMemHandle_t), ncclChar, comm, st) !=
      ncclSuccess)
    return HET_ERR_NCCL;
  std::vector<cudaIpcMemHandle_t> all(N);
  cudaMemcpyAsync(all.data(), dh, sizeof(cudaIpcMemHandle_t) * N, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return HET_ERR_CUDA;
  cudaFree(dh);
  std::vector<char*> bases(N);
  for (int r = 0; r < N; ++r) {
    if (r == rank) { bases[r] = mine_base; continue; }
    void* q = nullptr;
    if (cudaIpcOpenMemHandle(&q, all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HET_ERR_CUDA;
    bases[r] = (char*)q;
    p->mapped.push_back((char*)q);
  }
  cudaMemcpyAsync(dbases, bases.data(), sizeof(char*) * N, cudaMemcpyHostToDevice, st);
  return HET_OK;
}

// comm == nullptr: loopback worker (p2p_loopback_connect fills the peer tables)
het_status_t p2p_create(P2PState*& out, const Dev& d, uint32_t n_max, ncclComm_t comm, uint64_t dense_cap,
                        cudaStream_t st) {
  P2PState* p = new P2PState();
  out = p;
  p->loopback = comm == nullptr;
  P2P& v = p->v;
  v.N = d.world;
  v.rank = d.rank;
  v.CAPS = 3 * (int64_t)n_max;
  v.REC = 4 + d.D;
  v.D = d.D;
  const int N = v.N;
  if (N > P2P_MAX_WORLD) return HET_ERR_ARG;   // per-row record lists hold <= 32 records (2 per source)
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  v.off_reqflag = off; off = al(off + sizeof(Flag) * N);
  v.off_respflag = off; off = al(off + sizeof(Flag) * N);
  v.off_req = off; off = al(off + sizeof(Rec) * N * v.CAPS);
  v.off_rows = off; off = al(off + sizeof(float) * N * v.CAPS * d.D);
  v.off_resp = off; off = al(off + sizeof(float) * N * v.CAPS * v.REC);
  if (cudaMalloc(&p->inbox, off) != cudaSuccess) return HET_ERR_OOM;
  cudaMemsetAsync(p->inbox, 0, v.off_req, st);                      // flags: epoch 0
  char** dbases;
  if (!p_alloc(p, &dbases, N)) return HET_ERR_OOM;
  v.peer = dbases;
  if (!p->loopback) {
    het_status_t rc = exchange_bases(p, p->inbox, N, d.rank, comm, st, dbases);
    if (rc) return rc;
  }
  const int64_t NC = (int64_t)N * v.CAPS;
  bool ok = p_alloc(p, &v.lcnt, N) && p_alloc(p, &v.c3cnt, N) && p_alloc(p, &v.ridx, NC) &&
            p_alloc(p, &v.head, d.rows_local) && p_alloc(p, &v.next, NC) && p_alloc(p, &v.leaders, NC) &&
            p_alloc(p, &v.nlead, 1) && p_alloc(p, &v.done, 4) && p_alloc(p, &v.epoch, 1) &&
            p_alloc(p, &v.qtot, N) && p_alloc(p, &v.qpush, N) && p_alloc(p, &v.uslot, n_max);
  if (!ok) return HET_ERR_OOM;
  cudaMemsetAsync(v.lcnt, 0, 4 * N, st);
  cudaMemsetAsync(v.c3cnt, 0, 4 * N, st);
  cudaMemsetAsync(v.head, 0xFF, 4 * d.rows_local, st);
  cudaMemsetAsync(v.nlead, 0, 4, st);
  cudaMemsetAsync(v.done, 0, 16, st);
  cudaMemsetAsync(v.epoch, 0, 8, st);
  // dense all-reduce staging (Eq. 2), set up here -- outside any graph capture,
  // and agreed by every rank: a rank whose allocation failed makes all of
  // them use the NCCL all-reduce (no rank-local path choice)
  const uint64_t cap = (std::max<uint64_t>(dense_cap, 4) + 3) & ~3ull;
  const size_t flags = 2 * 64 * sizeof(Flag);
  int ok_dense = cudaMalloc(&p->dense, flags + 2 * cap * sizeof(float)) == cudaSuccess ? 1 : 0;
  if (!ok_dense) { cudaGetLastError(); p->dense = nullptr; }
  if (p->dense) cudaMemsetAsync(p->dense, 0, flags, st);
  DenseView& dv = p->dv;
  dv.N = N; dv.rank = d.rank; dv.cap = cap;
  char** dd;
  if (!p_alloc(p, &dd, N) || !p_alloc(p, &dv.epoch, 1) || !p_alloc(p, &dv.done, 2)) return HET_ERR_OOM;
  dv.peer = dd;
  cudaMemsetAsync(dv.epoch, 0, 8, st);
  cudaMemsetAsync(dv.done, 0, 8, st);
  if (!p->loopback) {
    int32_t* dok;
    if (!p_alloc(p, &dok, 1)) return HET_ERR_OOM;
    cudaMemcpyAsync(dok, &ok_dense, 4, cudaMemcpyHostToDevice, st);
    if (ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, st) != ncclSuccess) return HET_ERR_NCCL;
    cudaMemcpyAsync(&ok_dense, dok, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return HET_ERR_CUDA;
    if (ok_dense) {
      het_status_t rc = exchange_bases(p, p->dense, N, d.rank, comm, st, dd);
      if (rc) return rc;
    } else if (p->dense) {
      cudaFree(p->dense);
      p->dense = nullptr;
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return HET_ERR_CUDA;
  return HET_OK;
}

het_status_t p2p_loopback_connect(P2PState* const* ps, int N, cudaStream_t st) {
  std::vector<char*> inb(N), den(N);
  bool dense = true;
  for (int r = 0; r < N; ++r) {
    if (!ps[r] || !ps[r]->loopback) return HET_ERR_ARG;
    inb[r] = ps[r]->inbox;
    den[r] = ps[r]->dense;
    dense = dense && ps[r]->dense != nullptr && ps[r]->dv.cap == ps[0]->dv.cap;
  }
  for (int r = 0; r < N; ++r) {
    if (cudaMemcpyAsync((void*)ps[r]->v.peer, inb.data(), sizeof(char*) * N, cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
      return HET_ERR_CUDA;
    if (dense) {
      cudaMemcpyAsync((void*)ps[r]->dv.peer, den.data(), sizeof(char*) * N, cudaMemcpyHostToDevice, st);
    } else if (ps[r]->dense) {
      cudaFree(ps[r]->dense);
      ps[r]->dense = nullptr;
    }
  }
  return cudaStreamSynchronize(st) == cudaSuccess ? HET_OK : HET_ERR_CUDA;
}

void p2p_destroy(P2PState* p) {
  if (!p) return;
  for (char* q : p->mapped) cudaIpcCloseMemHandle(q);
  for (void* q : p->allocs) cudaFree(q);
  if (p->inbox) cudaFree(p->inbox);
  if (p->dense) cudaFree(p->dense);
  delete p;
}

bool p2p_loopback(const P2PState* p) { return p && p->loopback; }
int64_t p2p_caps(const P2PState* p) { return p->v.CAPS; }

het_status_t p2p_dense_allreduce(P2PState* p, const Dev& d, float* buf, uint64_t count, int phase, cudaStream_t st,
                                 int* launches) {
  if (!p->dense || count > p->dv.cap) return HET_ERR_CAPACITY;   // the caller falls back to NCCL
  k_dense_ar<<<coop_sm_reserve(), 512, 0, st>>>(p->dv, buf, count, 1.0f / (float)d.world, d.ctl, phase);
  *launches += 1;
  return HET_OK;
}

static int grid_p(int64_t units_warps) {
  int64_t b = (units_warps + 7) / 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 4));
}

// one phase of a drain round (drain = no requests, only the pending pushes)
// or of the non-fused lookup round (after k_probe)
int p2p_round_phase(P2PState* p, const Dev& d, const Call& c, int drain, int phase, cudaStream_t st) {
  P2P& v = p->v;
  switch (phase) {
    case RP_BUILD:
      cudaMemsetAsync(v.lcnt, 0, 4 * v.N, st);
      k_p2p_build<<<grid_p(std::max(c.n, 1)), 256, 0, st>>>(d, c, v, drain);
      return 1;
    case RP_LINK: k_p2p_link<<<148, 256, 0, st>>>(d, v); return 1;
    case RP_PROCESS: k_p2p_process<<<148 * 2, 256, 0, st>>>(d, v); return 1;
    default: k_p2p_install<<<148 * 2, 256, 0, st>>>(d, c, v); return 1;
  }
}

int p2p_round(P2PState* p, const Dev& d, const Call& c, int drain, cudaStream_t st) {
  int l = 0;
  for (int ph = 0; ph < RP_NUM; ++ph) l += p2p_round_phase(p, d, c, drain, ph, st);
  return l;
}

// one phase of the fused lookup round (after the dedup): probe+build, link,
// process, install+gather -- the device functions k_exchange runs between its
// grid syncs
int p2p_lookup_phase(P2PState* p, const Dev& d, const Call& c, float* out, int phase, cudaStream_t st) {
  P2P& v = p->v;   // lcnt is zero here: the previous round's publish reset it
  const int blocks = std::max(1, (c.n + 7) / 8);
  switch (phase) {
    case RP_BUILD: k_probe_build<<<blocks, 256, 0, st>>>(d, c, v, out); return 1;
    case RP_LINK: k_p2p_link<<<148, 256, 0, st>>>(d, v); return 1;
    case RP_PROCESS: k_p2p_process<<<148 * 2, 256, 0, st>>>(d, v); return 1;
    default:
      k_install_gather<<<blocks, 256, 0, st>>>(d, c, v, out);
      return 1 + (c.rmode && wide_rows(d.D) ? launch_scatter_wide(d, c, out, st, reinterpret_cast<const float*>(p->inbox + v.off_resp), v.REC, v.uslot) : 0);
  }
}

// fused round as ONE cooperative kernel (one process per GPU)
int p2p_round_fused(P2PState* p, const Dev& d, const Call& c, float* out, cudaStream_t st) {
  P2P& v = p->v;
  static const bool split = getenv("HET_P2P_SPLIT") != nullptr;   // diagnostic: the four-kernel round
  if (!split) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nsm - coop_sm_reserve());
    cfg.blockDim = dim3(EX_THREADS);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlaps the dedup's tail
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, k_exchange, d, c, v, out) == cudaSuccess)
      return 1 + (c.rmode && wide_rows(d.D) ? launch_scatter_wide(d, c, out, st, reinterpret_cast<const float*>(p->inbox + v.off_resp), v.REC, v.uslot) : 0);
    cudaGetLastError();   // fall through to the split round
  }
  int l = 0;
  for (int ph = 0; ph < RP_NUM; ++ph) l += p2p_lookup_phase(p, d, c, out, ph, st);
  return l;
}

P2P* p2p_view_ptr(P2PState* p) { return &p->v; }

int p2p_pushes(P2PState* p, const Dev& d, void* evbuf, cudaStream_t st) {
  EvView b = *reinterpret_cast<EvView*>(evbuf);
  k_p2p_pushes<<<148 * 2, 256, 0, st>>>(d, p->v, b);
  return 1;
}

int p2p_flush_build(P2PState* p, const Dev& d, int64_t k0, int64_t k1, cudaStream_t st) {
  k_p2p_flush_build<<<148 * 4, 256, 0, st>>>(d, p->v, k0, k1);
  return 1;
}

int p2p_evict_keys(P2PState* p, const Dev& d, const Call& c, cudaStream_t st) {
  k_p2p_evict_keys<<<std::max(1, (c.n + 7) / 8), 256, 0, st>>>(d, c, p->v);
  return 1;
}

}  // namespace het
