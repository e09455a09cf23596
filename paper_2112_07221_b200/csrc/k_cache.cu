// Cache kernels of the hot path (sm_100a).  Each kernel cites the passage of
// PAPER.md that defines the operation; readings Rn are listed in DESIGN.md.
//
//   K10 k_init_shard      W0 / c_g = 0 for this rank's rows (R14)
//   K2  k_probe           Cache.Find + CheckValid cond (1) [+ cond (2) at N=1]
//                         + LFU/LRU touch (R3, R7, R8)
//   K45 k_sync_fetch_local  N=1: Evict(k) push + Fetch(k) fused (P:439, P:442-443,
//                         P:495-500; R5, R6) and the miss install
//   K6  k_gather          Cache.Get: out[pos] = v[entry(inverse[pos])]
//   K7  k_segreduce_apply Cache.Update + Cache.Clock: acc = sum G (ascending
//                         position), d = -lr*acc, v += d, p += d, c_c += 1
//                         (R11, R13, R17)
//   K8  k_ev_*            Cache.Evict(): exact selection of |cache| - C victims
//                         by (count,key) [LFU] or (tick,key) [LRU] (R9)
//   K9  k_ev_apply        victim push W += p, c_g = max + free
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
    s.fstack[i] = (int32_t)(s.Ecap - 1 - i);
  }
  for (int64_t i = i0; i <= (int64_t)s.hmask; i += stride) s.hkey[i] = HK_EMPTY;
  if (i0 == 0) {
    s.ctl->ftop = (int32_t)s.Ecap;
    s.ctl->n_tomb = 0;
    s.ctl->T_last = 0;
    s.ctl->min_install = 0xFFFFFFFFu;
  }
}

void launch_init_shard(const Dev& s, cudaStream_t st) {
  k_init_shard<<<148 * 8, 256, 0, st>>>(s);
}
void launch_reset_cache(const Dev& s, cudaStream_t st) {
  k_reset_cache<<<148 * 8, 256, 0, st>>>(s);
}

// ------------------------------------------------------------------ block counters
struct BlockCnt {
  unsigned c[4];
};

// ------------------------------------------------------------------ K2 probe
__global__ void __launch_bounds__(TPB)
k_probe(Dev s, Call c) {
  __shared__ unsigned bc[4];  // hits, exp1, exp2, misses
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  __syncthreads();
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int U = ctl->U;
  if (!ctl->abort && u < U) {
    int64_t key = c.uniq[u];
    int32_t e = warp_find(s, key, lane);
    if (lane == 0) {
      uint8_t st;
      uint32_t cnt = 0;
      if (s.lfu_persist) { cnt = s.count_by_key[key] + 1; s.count_by_key[key] = cnt; }
      if (e < 0) {
        st = ST_MISS;
      } else {
        uint32_t ecs = s.cs[e], ecc = s.cc[e];
        if (s.s == S_INF) st = ST_HIT;                      // R4: no clock check
        else if (ecc - ecs > s.s) st = ST_EXP1;             // cond (1) fails
        else if (s.world == 1) {                            // cond (2), c_g read now (R1, R3)
          uint32_t g = s.cg[key];
          st = (g <= ecc || g - ecc <= s.s) ? ST_HIT : ST_EXP2;
        } else st = ST_NEEDQ;                               // ask the owner (C1)
        // L6: LFU count +1 / LRU tick = t for resident entries
        if (s.policy == 0) s.eprim[e] = s.lfu_persist ? cnt : s.eprim[e] + 1;
        else s.eprim[e] = (uint32_t)c.t;
      }
      c.status[u] = st;
      c.uentry[u] = e;
      if (st < 4) atomicAdd(&bc[st == ST_HIT ? 0 : st == ST_EXP1 ? 1 : st == ST_EXP2 ? 2 : 3], 1u);
    }
  }
  __syncthreads();
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
// refetch (L5) in one pass per key; keys are distinct within the call.
__global__ void __launch_bounds__(TPB)
k_sync_fetch_local(Dev s, Call c) {
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ctl->abort || u >= ctl->U) return;
  uint8_t st = c.status[u];
  if (st == ST_HIT) return;
  int64_t key = c.uniq[u];
  int64_t row = key;  // N = 1: local row = key
  const int D4 = s.D >> 2;
  float4* Wr = reinterpret_cast<float4*>(s.W + row * s.D);
  int32_t e;
  uint32_t g;
  if (st == ST_EXP1 || st == ST_EXP2) {
    e = c.uentry[u];
    uint32_t ecs = s.cs[e], ecc = s.cc[e];
    g = s.cg[row];
    if (ecc > ecs) {  // dirty (R13): W += p, c_g = max(c_g, c_c)
      const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
      for (int d = lane; d < D4; d += 32) Wr[d] = f4add(Wr[d], pr[d]);
      g = g > ecc ? g : ecc;
      if (lane == 0) s.cg[row] = g;
    }
  } else {  // MISS: take a free entry, insert into the hash table
    int32_t idx = 0;
    if (lane == 0) idx = atomicSub(&ctl->ftop, 1) - 1;
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx < 0) {
      if (lane == 0) raise_err(ctl, 4 /*HET_ERR_CAPACITY*/);
      return;
    }
    e = s.fstack[idx];
    warp_insert(s, key, e, lane);
    g = s.cg[row];
    if (lane == 0) {
      s.ekey[e] = key;
      uint32_t prim = s.policy == 0 ? (s.lfu_persist ? s.count_by_key[key] : 1u) : (uint32_t)c.t;
      s.eprim[e] = prim;
      atomicMin(&ctl->min_install, prim);
      c.uentry[u] = e;
    }
  }
  // L5: v = W[k], c_s = c_c = c_g  (p need not be zeroed: R13)
  float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
  for (int d = lane; d < D4; d += 32) vr[d] = Wr[d];
  if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
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

// ------------------------------------------------------------------ K7 segment-reduce + apply
__global__ void __launch_bounds__(TPB)
k_segreduce_apply(Dev s, Call c, const float* __restrict__ G, float lr) {
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ctl->abort || u >= ctl->U) return;
  int32_t e = c.uentry[u];
  int j0 = c.seg_off[u], j1 = c.seg_off[u + 1];
  bool dirty = s.cc[e] > s.cs[e];
  const int D4 = s.D >> 2;
  const float nlr = -lr;
  float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
  float4* pr = reinterpret_cast<float4*>(s.p + (int64_t)e * s.D);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  for (int d = lane; d < D4; d += 32) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);       // U1: +0.0f, ascending position
    for (int j = j0; j < j1; ++j) {
      int pos = __ldg(&c.perm[j]);
      acc = f4add(acc, __ldcs(G4 + (int64_t)pos * D4 + d));
    }
    float4 dl = make_float4(__fmul_rn(nlr, acc.x), __fmul_rn(nlr, acc.y), __fmul_rn(nlr, acc.z),
                            __fmul_rn(nlr, acc.w));  // U2: delta = (-lr) * acc
    vr[d] = f4add(vr[d], dl);
    pr[d] = dirty ? f4add(pr[d], dl) : f4add(make_float4(0.f, 0.f, 0.f, 0.f), dl);
  }
  __syncwarp();
  if (lane == 0) s.cc[e] = s.cc[e] + 1;  // Cache.Clock
}

void launch_segreduce_apply(const Dev& s, const Call& c, const float* grads, float lr, int n_units,
                            cudaStream_t st) {
  int blocks = (n_units + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
  if (blocks < 1) blocks = 1;
  k_segreduce_apply<<<blocks, TPB, 0, st>>>(s, c, grads, lr);
}

// ------------------------------------------------------------------ K8 eviction selection
struct EvBuf {
  uint32_t* hist;    // [NBIN] primary histogram relative to base
  uint32_t* khist;   // [NBIN] key-top histogram of candidates
  int32_t* victims;  // [vcap] entry indices
  int32_t* cand;     // [Ecap]
  int32_t* sub;      // [Ecap]
  int32_t* flags;    // [4]: base_invalid
  int64_t* vkeys;    // [vcap] victim keys (debug/parity export)
  uint8_t* vdirty;   // [vcap]
};

__device__ __forceinline__ int64_t resident_count(const Dev& s) {
  return s.Ecap - (int64_t)s.ctl->ftop;
}

__device__ __forceinline__ uint32_t ev_base(const Dev& s) {
  uint32_t b = s.ctl->T_last;
  if (s.policy == 0) b = min(b, s.ctl->min_install);
  return b;
}

// smem histogram increment aggregated across lanes holding the same bin
__device__ __forceinline__ void hist_add(uint32_t* h, unsigned active, int bin, bool pred) {
  unsigned m = __ballot_sync(active, pred);
  if (!pred) return;
  unsigned grp = __match_any_sync(m, bin);
  if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&h[bin], (uint32_t)__popc(grp));
}

// E1: histogram of primaries of all resident entries
__global__ void __launch_bounds__(256)
k_ev_hist(Dev s, EvBuf b) {
  __shared__ uint32_t h[NBIN];
  int64_t need = resident_count(s) - s.C;
  if (s.ctl->abort || need <= 0) return;
  if (need >= resident_count(s)) return;  // everything goes: no histogram needed
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t base = ev_base(s);
  int bad = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t limit = ((s.Ecap + 31) / 32) * 32;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < limit + 0; e += stride) {
    bool res = false;
    int bin = 0;
    if (e < s.Ecap && s.ekey[e] >= 0) {
      uint32_t prim = s.eprim[e];
      if (prim < base) bad = 1;
      uint32_t rel = prim - base;
      bin = rel < (uint32_t)(NBIN - 1) ? (int)rel : NBIN - 1;
      res = true;
    }
    hist_add(h, 0xffffffffu, bin, res);
  }
  if (bad) b.flags[0] = 1;
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x)
    if (h[i]) atomicAdd(&b.hist[i], h[i]);
}

// CTA-wide exact k-th selection over a u32 key space by 3 radix passes
// (11, 11, 10 bits), reading the values through `get(i, &val)` for i < count.
// Returns the threshold V with #(val < V) < m <= #(val <= V); *below = #(val < V).
template <typename Get>
__device__ uint32_t cta_select_u32(Get get, int64_t count, int64_t m, int64_t* below, uint32_t* sh_hist) {
  uint32_t prefix = 0;
  int64_t acc_below = 0;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  uint32_t pmask = 0;  // bits of prefix fixed so far
  for (int pass = 0; pass < 3; ++pass) {
    int nb = 1 << widths[pass];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
      uint32_t val;
      if (!get(i, &val)) continue;
      if ((val & pmask) != prefix) continue;
      atomicAdd(&sh_hist[(val >> shifts[pass]) & (nb - 1)], 1u);
    }
    __syncthreads();
    __shared__ int sel;
    __shared__ long long selbelow;
    if (threadIdx.x == 0) {
      int64_t cum = acc_below;
      int bsel = nb - 1;
      for (int bb = 0; bb < nb; ++bb) {
        if (cum + sh_hist[bb] >= m) { bsel = bb; break; }
        cum += sh_hist[bb];
      }
      sel = bsel;
      selbelow = cum;
    }
    __syncthreads();
    prefix |= (uint32_t)sel << shifts[pass];
    pmask |= (uint32_t)(nb - 1) << shifts[pass];
    acc_below = selbelow;
    __syncthreads();
  }
  *below = acc_below;
  return prefix;
}

// E2: resolve the threshold primary T and needT (one CTA)
__global__ void __launch_bounds__(1024)
k_ev_resolve(Dev s, EvBuf b) {
  __shared__ uint32_t sh[NBIN];
  __shared__ int s_found;
  Ctl* ctl = s.ctl;
  int64_t res = resident_count(s);
  int64_t need = res - s.C;
  if (threadIdx.x == 0) {
    ctl->nvict = 0; ctl->ncand = 0; ctl->nsub = 0;
    ctl->need = (ctl->abort || need < 0) ? 0 : need;
    ctl->resolved = 0;
  }
  if (ctl->abort || need <= 0) {
    __syncthreads();
    if (threadIdx.x == 0) { ctl->needT = 0; ctl->T = 0; }
    return;
  }
  if (need >= res) {  // evict everything
    if (threadIdx.x == 0) { ctl->T = 0xFFFFFFFFu; ctl->needT = -1; ctl->min_install = 0xFFFFFFFFu; }
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x) b.hist[i] = 0;
    return;
  }
  uint32_t base = ev_base(s);
  // fast path: exact bins 0..NBIN-2 of the histogram
  if (threadIdx.x == 0) {
    s_found = 0;
    if (!b.flags[0]) {
      int64_t cum = 0;
      for (int bb = 0; bb < NBIN - 1; ++bb) {
        uint32_t hb = b.hist[bb];
        if (cum + hb >= need) {
          ctl->T = base + (uint32_t)bb;
          ctl->needT = need - cum;
          ctl->ncand = 0;
          s_found = 1;
          break;
        }
        cum += hb;
      }
    }
  }
  __syncthreads();
  if (!s_found) {
    // slow exact path: radix select over absolute primaries of residents
    int64_t below;
    auto get = [&](int64_t i, uint32_t* val) -> bool {
      if (s.ekey[i] < 0) return false;
      *val = s.eprim[i];
      return true;
    };
    uint32_t T = cta_select_u32(get, s.Ecap, need, &below, sh);
    if (threadIdx.x == 0) { ctl->T = T; ctl->needT = need - below; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) b.hist[i] = 0;
  if (threadIdx.x == 0) {
    b.flags[0] = 0;
    ctl->T_last = ctl->T;
    ctl->min_install = 0xFFFFFFFFu;
  }
}

// block-level compaction helper: returns global slot for flagged threads
__device__ __forceinline__ int block_compact(bool flag, int32_t* counter, int* sh_warp, int* sh_base) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned m = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sh_warp[wid] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { int x = sh_warp[w]; sh_warp[w] = tot; tot += x; }
    *sh_base = tot ? atomicAdd(counter, tot) : 0;
  }
  __syncthreads();
  int slot = *sh_base + sh_warp[wid] + __popc(m & ((1u << lane) - 1));
  __syncthreads();
  return slot;
}

__device__ __forceinline__ int key_top(const Dev& s, int64_t key) {
  int sh = s.kbits > 11 ? s.kbits - 11 : 0;
  return (int)(key >> sh) & (NBIN - 1);
}

// E3: victims with prim < T, candidates with prim == T (+ key-top histogram)
__global__ void __launch_bounds__(256)
k_ev_collect(Dev s, EvBuf b) {
  __shared__ uint32_t kh[NBIN];
  __shared__ int sh_warp[8], sh_base;
  Ctl* ctl = s.ctl;
  if (ctl->abort || ctl->need <= 0) return;
  uint32_t T = ctl->T;
  int64_t needT = ctl->needT;
  bool all = needT < 0;
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) kh[i] = 0;
  __syncthreads();
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t limit = ((s.Ecap + stride - 1) / stride) * stride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < limit; e += stride) {
    bool isv = false, isc = false;
    int64_t key = -1;
    if (e < s.Ecap) {
      key = s.ekey[e];
      if (key >= 0) {
        uint32_t prim = s.eprim[e];
        if (all || prim < T) isv = true;
        else if (prim == T && needT > 0) isc = true;
      }
    }
    int vs = block_compact(isv, &ctl->nvict, sh_warp, &sh_base);
    if (isv) b.victims[vs] = (int32_t)e;
    int cs = block_compact(isc, &ctl->ncand, sh_warp, &sh_base);
    if (isc) b.cand[cs] = (int32_t)e;
    hist_add(kh, 0xffffffffu, isc ? key_top(s, key) : 0, isc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x)
    if (kh[i]) atomicAdd(&b.khist[i], kh[i]);
}

// E4: choose the key-top bucket among candidates (one CTA)
__global__ void k_ev_resolve_key(Dev s, EvBuf b) {
  Ctl* ctl = s.ctl;
  if (threadIdx.x == 0) {
    ctl->kb1 = 0xFFFFFFFFu;
    ctl->need2 = 0;
    int64_t needT = ctl->needT;
    if (!ctl->abort && ctl->need > 0 && needT > 0) {
      if (needT >= ctl->ncand) {
        ctl->kb1 = NBIN;  // every candidate is a victim
      } else {
        int64_t cum = 0;
        for (int bb = 0; bb < NBIN; ++bb) {
          uint32_t hb = b.khist[bb];
          if (cum + hb >= needT) { ctl->kb1 = bb; ctl->need2 = needT - cum; break; }
          cum += hb;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) b.khist[i] = 0;
}

// E5: candidates below the bucket are victims, the bucket itself is the sub list
__global__ void __launch_bounds__(256)
k_ev_collect_key(Dev s, EvBuf b) {
  __shared__ int sh_warp[8], sh_base;
  Ctl* ctl = s.ctl;
  uint32_t kb1 = ctl->kb1;
  if (ctl->abort || ctl->need <= 0 || kb1 == 0xFFFFFFFFu) return;
  int nc = ctl->ncand;
  int stride = gridDim.x * blockDim.x;
  int limit = ((nc + stride - 1) / stride) * stride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < limit; i += stride) {
    bool isv = false, iss = false;
    int32_t e = -1;
    if (i < nc) {
      e = b.cand[i];
      uint32_t kt = (uint32_t)key_top(s, s.ekey[e]);
      if (kb1 == NBIN || kt < kb1) isv = true;
      else if (kt == kb1) iss = true;
    }
    int vs = block_compact(isv, &ctl->nvict, sh_warp, &sh_base);
    if (isv) b.victims[vs] = e;
    int ss = block_compact(iss, &ctl->nsub, sh_warp, &sh_base);
    if (iss) b.sub[ss] = e;
  }
}

__device__ __forceinline__ void bitonic_smem64(uint64_t* a, int npad) {
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (npad >> 1); i += blockDim.x) {
        int lo = 2 * j * (i / j) + (i % j);
        int hi = lo + j;
        bool up = (lo & k) == 0;
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
      }
      __syncthreads();
    }
  }
}

// E6: the need2 smallest keys of the sub list (one CTA)
__global__ void __launch_bounds__(1024)
k_ev_select_sub(Dev s, EvBuf b) {
  extern __shared__ uint64_t sm[];
  __shared__ uint32_t sh[NBIN];
  Ctl* ctl = s.ctl;
  uint32_t kb1 = ctl->kb1;
  if (ctl->abort || ctl->need <= 0 || kb1 == 0xFFFFFFFFu || kb1 == NBIN) return;
  int nsub = ctl->nsub;
  int64_t need2 = ctl->need2;
  if (need2 <= 0) return;
  if (nsub <= SUBMAX) {
    int npad = 2;
    while (npad < nsub) npad <<= 1;
    for (int i = threadIdx.x; i < npad; i += blockDim.x)
      sm[i] = i < nsub ? (((uint64_t)s.ekey[b.sub[i]] << 24) | (uint64_t)i) : ~0ull;
    __syncthreads();
    bitonic_smem64(sm, npad);
    int base = ctl->nvict;
    for (int i = threadIdx.x; i < need2; i += blockDim.x)
      b.victims[base + i] = b.sub[(int)(sm[i] & 0xFFFFFF)];
    __syncthreads();
    if (threadIdx.x == 0) ctl->nvict = base + (int)need2;
  } else {
    // slow exact path: keys below 2^32 (kbits <= 32 enforced at create)
    int64_t below;
    auto get = [&](int64_t i, uint32_t* val) -> bool { *val = (uint32_t)s.ekey[b.sub[i]]; return true; };
    uint32_t K = cta_select_u32(get, nsub, need2, &below, sh);
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = ctl->nvict;
    __syncthreads();
    for (int i = threadIdx.x; i < nsub; i += blockDim.x) {
      int32_t e = b.sub[i];
      if ((uint32_t)s.ekey[e] <= K) b.victims[atomicAdd(&cnt, 1)] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) ctl->nvict = cnt;
  }
}

// E7 (N = 1): push dirty victims to the local server, delete, free
__global__ void __launch_bounds__(TPB)
k_ev_apply_local(Dev s, EvBuf b) {
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  if (ctl->abort || ctl->need <= 0) return;
  int nv = ctl->nvict;
  const int D4 = s.D >> 2;
  for (int i = w; i < nv; i += nw) {
    int32_t e = b.victims[i];
    int64_t key = s.ekey[e];
    uint32_t ecs = s.cs[e], ecc = s.cc[e];
    bool dirty = ecc > ecs;
    if (lane == 0) { b.vkeys[i] = key; b.vdirty[i] = dirty ? 1 : 0; }
    if (dirty) {
      float4* Wr = reinterpret_cast<float4*>(s.W + key * s.D);
      const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
      for (int d = lane; d < D4; d += 32) Wr[d] = f4add(Wr[d], pr[d]);
      if (lane == 0) { uint32_t g = s.cg[key]; s.cg[key] = g > ecc ? g : ecc; }
    }
    warp_erase(s, key, lane);
    if (lane == 0) {
      s.ekey[e] = -1;
      int32_t slot = atomicAdd(&ctl->ftop, 1);
      s.fstack[slot] = e;
      atomicAdd(&s.cnt[C_EVICTIONS], 1ull);
      if (dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], 1ull);
    }
  }
}

int launch_evict_select(const Dev& s, void* evbuf, cudaStream_t st) {
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  k_ev_hist<<<148 * 4, 256, 0, st>>>(s, b);
  k_ev_resolve<<<1, 1024, 0, st>>>(s, b);
  k_ev_collect<<<148 * 4, 256, 0, st>>>(s, b);
  k_ev_resolve_key<<<1, 256, 0, st>>>(s, b);
  k_ev_collect_key<<<148, 256, 0, st>>>(s, b);
  k_ev_select_sub<<<1, 1024, SUBMAX * 8, st>>>(s, b);
  return 6;
}

int launch_evict_overflow(const Dev& s, void* evbuf, int n_max, cudaStream_t st) {
  int n = launch_evict_select(s, evbuf, st);
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  k_ev_apply_local<<<148 * 2, TPB, 0, st>>>(s, b);
  return n + 1;
}

void cache_set_attrs() {
  cudaFuncSetAttribute(k_ev_select_sub, cudaFuncAttributeMaxDynamicSharedMemorySize, SUBMAX * 8);
}

size_t evbuf_struct_size() { return sizeof(EvBuf); }

void evbuf_init(void* evbuf, uint32_t* hist, uint32_t* khist, int32_t* victims, int32_t* cand,
                int32_t* sub, int32_t* flags, int64_t* vkeys, uint8_t* vdirty) {
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  b.hist = hist; b.khist = khist; b.victims = victims; b.cand = cand; b.sub = sub; b.flags = flags;
  b.vkeys = vkeys; b.vdirty = vdirty;
}

// ------------------------------------------------------------------ hash rebuild
__global__ void k_rebuild_decide(Dev s) {
  Ctl* ctl = s.ctl;
  int64_t S = (int64_t)s.hmask + 1;
  ctl->rebuild = (int64_t)ctl->n_tomb > S / 8 ? 1 : 0;
  if (ctl->rebuild) ctl->n_tomb = 0;
}
__global__ void k_rebuild_clear(Dev s) {
  if (!s.ctl->rebuild) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= (int64_t)s.hmask;
       i += (int64_t)gridDim.x * blockDim.x)
    s.hkey[i] = HK_EMPTY;
}
__global__ void k_rebuild_insert(Dev s) {
  if (!s.ctl->rebuild) return;
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
  k_rebuild_decide<<<1, 1, 0, st>>>(s);
  k_rebuild_clear<<<148 * 4, 256, 0, st>>>(s);
  k_rebuild_insert<<<148 * 4, 256, 0, st>>>(s);
}

}  // namespace het
