// Cache kernels of the hot path (sm_100a).  Each kernel cites the passage of
// PAPER.md that defines the operation; readings Rn are listed in DESIGN.md.
//
//   K10 k_init_shard      W0 / c_g = 0 for this rank's rows (R14)
//   K2  k_probe           Cache.Find + CheckValid cond (1) [+ cond (2) at N=1]
//                         + LFU/LRU touch (R3, R7, R8)
//   K45 k_sync_fetch_local  N=1: Evict(k) push + Fetch(k) fused (P:439, P:442-443,
//                         P:495-500; R5, R6) and the miss install
//   K6  k_gather          Cache.Get: out[pos] = v[entry(inverse[pos])]
//   (K7 segment reduce + apply: k_segreduce.cu; K8/K9 eviction: k_evict.cu)
#include <algorithm>

#include "het_internal.cuh"

namespace het {

constexpr int WARPS_PER_BLOCK = 8;
constexpr int TPB = WARPS_PER_BLOCK * 32;
constexpr int NBIN = 2048;
constexpr int SUBMAX = 16384;

// ------------------------------------------------------------------ init
__global__ void k_init_shard(Dev s) {
  int64_t total = s.rows_local * (int64_t)s.D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / s.D;
    uint32_t d = (uint32_t)(i - r * s.D);
    int64_t key = r * s.world + s.rank;
    s.W[i] = init_w0(s.seed0, key, d);
  }
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < s.rows_local;
       r += (int64_t)gridDim.x * blockDim.x)
    s.cg[r] = 0;
}

__global__ void k_reset_cache(Dev s) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < s.Ecap; i += stride) {
    s.ekey[i] = -1;
    s.eprim[i] = EP_FREE;
    s.fstack[i] = (int32_t)(s.Ecap - 1 - i);
  }
  for (int64_t i = i0; i <= (int64_t)s.hmask; i += stride) s.hslot[i] = HS_EMPTY;
  if (i0 == 0) {
    s.ctl->ftop = (int32_t)s.Ecap;
    s.ctl->n_tomb = 0;
    s.ctl->npinned = 0;      // light-LFU: the cache is empty
    s.ctl->npin_cand = 0;
    s.ctl->T_last = 0;
    s.ctl->min_install = 0xFFFFFFFFu;
  }
}

// first kernel of every lookup: reset the per-call abort flag, fix the
// clock t of this call (the caller's, or the device counter for
// HET_CLOCK_AUTO so captured CUDA graphs advance it on replay), count it.
__global__ void k_begin(Dev s, uint64_t t, int n) {
  Ctl* ctl = s.ctl;
  ctl->abort = 0;
  if (t == CLOCK_AUTO) { t = ctl->t_auto; ctl->t_auto = t + 1; }
  ctl->t_cur = t;
  ctl->lk_seq = ctl->lk_seq + 1;
  ctl->nsel = 0;   // the fused update's victim list (its extraction blocks append)
  s.cnt[C_LOOKUPS] += 1;
  s.cnt[C_KEYS] += (unsigned long long)n;
}

void launch_begin(const Dev& s, uint64_t t, int n, cudaStream_t st) { k_begin<<<1, 1, 0, st>>>(s, t, n); }

void launch_init_shard(const Dev& s, cudaStream_t st) {
  k_init_shard<<<148 * 8, 256, 0, st>>>(s);
}
void launch_reset_cache(const Dev& s, cudaStream_t st) {
  k_reset_cache<<<148 * 8, 256, 0, st>>>(s);
}

// ------------------------------------------------------------------ block counters

// ------------------------------------------------------------------ K2 probe
__global__ void __launch_bounds__(TPB)
k_probe(Dev s, Call c) {
  __shared__ unsigned bc[4];  // hits, exp1, exp2, misses
  __shared__ int dpop[LFU_CB_MAX];
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  dpop_init(dpop);
  __syncthreads();
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int U = ctl->U;
  if (!ctl->abort && u < U) {
    int64_t key = c.uniq[u];
    // issue the count and (N = 1) global-clock loads alongside the hash probe
    uint32_t cnt = 0, gpre = 0;
    if (lane == 0 && s.lfu_persist) cnt = s.count_by_key[key];
    if (lane == 1 && s.world == 1 && s.s != S_INF) gpre = s.cg[key];
    int32_t e = warp_find(s, key, lane);
    gpre = __shfl_sync(0xffffffffu, gpre, 1);
    if (lane == 0) {
      uint8_t st;
      const uint32_t oldc = (e >= 0 && s.policy == 0) ? s.eprim[e] : 0u;
      const bool pinned = oldc == EP_PIN;            // light-LFU: no frequency maintenance
      if (s.lfu_persist && !pinned) { cnt += 1; s.count_by_key[key] = cnt; }
      if (e < 0) {
        st = ST_MISS;
      } else {
        uint32_t ecs = s.cs[e], ecc = s.cc[e];
        if (s.s == S_INF) st = ST_HIT;                      // R4: no clock check
        else if (ecc - ecs > s.s) st = ST_EXP1;             // cond (1) fails
        else if (s.world == 1) {                            // cond (2), c_g read now (R1, R3)
          uint32_t g = gpre;
          st = (g <= ecc || g - ecc <= s.s) ? ST_HIT : ST_EXP2;
        } else st = ST_NEEDQ;                               // ask the owner (C1)
        // L6: LFU count +1 / LRU tick = t for resident entries
        if (s.policy == 0) {
          if (!pinned) {
            uint32_t newc = s.lfu_persist ? cnt : oldc + 1;
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
      if (st < 4) atomicAdd(&bc[st == ST_HIT ? 0 : st == ST_EXP1 ? 1 : st == ST_EXP2 ? 2 : 3], 1u);
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP1], (unsigned long long)bc[1]);
    if (bc[2]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[2]);
    if (bc[3]) atomicAdd(&s.cnt[C_MISSES], (unsigned long long)bc[3]);
    if (blockIdx.x == 0 && !ctl->abort) atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)U);
  }
}

void launch_probe(const Dev& s, const Call& c, int n_units, cudaStream_t st) {
  int blocks = (n_units + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
  if (blocks < 1) blocks = 1;
  k_probe<<<blocks, TPB, 0, st>>>(s, c);
}

// ------------------------------------------------------------------ row helpers
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// ------------------------------------------------------------------ K45 (N = 1)
// Server == this rank: apply the sync push of an expired dirty hit (L4) and
// refetch (L5) in one pass per key; keys are distinct within the call.  Warp
// per key.  Misses take free entries and report their primary for the
// eviction lower bound; both go through one global atomic per block (free
// stack pop, min_install) -- with ~10^5 misses per call, per-warp atomics on
// those two addresses serialise in L2.  Which free entry a key gets is not
// observable.
__global__ void __launch_bounds__(TPB)
k_sync_fetch_local(Dev s, Call c) {
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ int s_nmiss, s_base;
  __shared__ unsigned s_minp;
  dpop_init(dpop);
  if (threadIdx.x == 0) { s_nmiss = 0; s_minp = 0xFFFFFFFFu; }
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool live = !ctl->abort && u < ctl->U;
  const uint8_t st = live ? c.status[u] : (uint8_t)ST_HIT;
  const int64_t key = live ? c.uniq[u] : 0;
  const bool miss = live && st == ST_MISS;
  int moff = 0;
  uint32_t prim = 0;
  if (miss) {
    prim = s.policy == 0 ? (s.lfu_persist ? s.count_by_key[key] : 1u) : (uint32_t)ctl->t_cur;
    if (lane == 0) {
      moff = atomicAdd(&s_nmiss, 1);
      atomicMin(&s_minp, prim);
    }
    moff = __shfl_sync(0xffffffffu, moff, 0);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_nmiss) {
    s_base = atomicSub(&ctl->ftop, s_nmiss);   // entries fstack[s_base - s_nmiss, s_base)
    atomicMin(&ctl->min_install, s_minp);
  }
  __syncthreads();
  if (live && st != ST_HIT) {
    const int64_t row = key;  // N = 1: local row = key
    const int D4 = s.D >> 2;
    float4* Wr = reinterpret_cast<float4*>(s.W + row * s.D);
    int32_t e = 0;
    uint32_t g = 0;
    bool ok = true;
    if (st == ST_EXP1 || st == ST_EXP2) {
      e = c.uentry[u];
      const uint32_t ecs = s.cs[e], ecc = s.cc[e];
      g = s.cg[row];
      if (ecc > ecs) {  // dirty (R13): W += p, c_g = max(c_g, c_c)
        const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
        for (int d = lane; d < D4; d += 32) Wr[d] = f4add(Wr[d], pr[d]);
        g = g > ecc ? g : ecc;
        if (lane == 0) s.cg[row] = g;
      }
    } else {  // MISS: take a free entry, insert into the hash table
      const int idx = s_base - 1 - moff;
      if (idx < 0) {
        if (lane == 0) raise_err(ctl, 4 /*HET_ERR_CAPACITY*/);
        ok = false;
      } else {
        HET_ASSERT(idx >= 0 && idx < s.Ecap);
        e = s.fstack[idx];
        HET_ASSERT(e >= 0 && e < s.Ecap);
        warp_insert(s, key, e, lane);
        g = s.cg[row];
        if (lane == 0) {
          s.ekey[e] = key;
          s.eprim[e] = prim;
          if (s.policy == 0) { lfu_move(s, key, EP_FREE, prim, dpop); pin_candidate(s, key, e, prim); }
          c.uentry[u] = e;
        }
      }
    }
    if (ok) {
      // L5: v = W[k], c_s = c_c = c_g  (p need not be zeroed: R13)
      float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
      for (int d = lane; d < D4; d += 32) vr[d] = Wr[d];
      if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
}

void launch_sync_fetch_install_local(const Dev& s, const Call& c, int n_units, cudaStream_t st) {
  int blocks = (n_units + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
  if (blocks < 1) blocks = 1;
  k_sync_fetch_local<<<blocks, TPB, 0, st>>>(s, c);
}

// ------------------------------------------------------------------ K6 gather
// one float4 per thread, consecutive threads along the row: 128-bit coalesced
// stores of out, 128-bit loads of the (L2-friendly) cached rows.
__global__ void __launch_bounds__(256)
k_gather(const float* __restrict__ v, const int32_t* __restrict__ uentry,
         const int32_t* __restrict__ inverse, float* __restrict__ out, int n, int D4,
         const Ctl* __restrict__ ctl) {
  if (ctl->abort) return;
  int64_t total = (int64_t)n * D4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int pos = (int)(i / D4);
    int d = (int)(i - (int64_t)pos * D4);
    int32_t e = __ldg(&uentry[__ldg(&inverse[pos])]);
    float4 x = __ldg(reinterpret_cast<const float4*>(v) + (int64_t)e * D4 + d);
    __stcs(reinterpret_cast<float4*>(out) + i, x);
  }
}

void launch_gather(const Dev& s, const Call& c, float* out, cudaStream_t st) {
  int D4 = s.D >> 2;
  int64_t total = (int64_t)c.n * D4;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_gather<<<(int)blocks, 256, 0, st>>>(s.v, c.uentry, c.inverse, out, c.n, D4, s.ctl);
}

// ------------------------------------------------------------------ hash rebuild
// Hash maintenance: when tombstones exceed S/8 the table is rebuilt from the
// resident entries.  Every block of k_rebuild_clear takes the same decision
// from n_tomb (unchanged during the kernel); k_rebuild_insert reads it back.
__global__ void k_rebuild_clear(Dev s) {
  const int64_t S = (int64_t)s.hmask + 1;
  const bool go = (int64_t)s.ctl->n_tomb > S / 8;
  if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->rebuild = go ? 1 : 0;
  if (!go) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x)
    s.hslot[i] = HS_EMPTY;
}
__global__ void k_rebuild_insert(Dev s) {
  if (!s.ctl->rebuild) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) s.ctl->n_tomb = 0;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t e0 = (int64_t)w * 32; e0 < s.Ecap; e0 += (int64_t)nw * 32) {
    int64_t e = e0 + lane;
    int64_t key = e < s.Ecap ? s.ekey[e] : -1;
    unsigned m = __ballot_sync(0xffffffffu, key >= 0);
    while (m) {
      int src = __ffs(m) - 1;
      int64_t k = __shfl_sync(0xffffffffu, key, src);
      warp_insert(s, k, (int32_t)(e0 + src), lane);
      m &= m - 1;
    }
  }
}

void launch_hash_rebuild(const Dev& s, cudaStream_t st) {
  k_rebuild_clear<<<148 * 4, 256, 0, st>>>(s);
  k_rebuild_insert<<<148 * 4, 256, 0, st>>>(s);
}

}  // namespace het
