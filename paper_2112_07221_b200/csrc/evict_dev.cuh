// Eviction device code shared by k_evict.cu and k_fused.cu (internal).
#pragma once
#include <cooperative_groups.h>

#include "het_internal.cuh"

namespace het {
namespace cg = cooperative_groups;

constexpr int NBIN = 2048;
constexpr int SUBMAX = 8192;
constexpr int GEN_THREADS = 512;

struct EvBuf {
  uint32_t* hist;    // [NBIN] primary histogram relative to base
  uint32_t* khist;   // [NBIN] key-top histogram of candidates
  int32_t* victims;  // [vcap] entry indices (generic path)
  int32_t* cand;     // [Ecap]
  int32_t* sub;      // [Ecap]
  int32_t* flags;    // [4]: base_invalid
  int64_t* vkeys;    // [vcap] victim keys (export)
  uint8_t* vdirty;   // [vcap]
  int64_t* vsel;     // [vcap] victim keys chosen by the bitmap path
};

__device__ __forceinline__ int64_t resident_count(const Dev& s) { return s.Ecap - (int64_t)s.ctl->ftop; }

// exclusive block scan of one int per thread
__device__ __forceinline__ int64_t block_excl_scan64(int64_t x, long long* warp_sums, long long* tot) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_sums[wid] = v;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  long long base = wid ? warp_sums[wid - 1] : 0;
  *tot = warp_sums[nw - 1];
  __syncthreads();
  return base + v - x;
}

__device__ __forceinline__ int warp_append(bool pred, int32_t* counter) {
  unsigned m = __ballot_sync(0xffffffffu, pred);
  int lane = threadIdx.x & 31;
  int base = 0;
  if (m) {
    int leader = __ffs(m) - 1;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  return base + __popc(m & ((1u << lane) - 1));
}

__device__ __forceinline__ void hist_add(uint32_t* h, int bin, bool pred) {
  unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!pred) return;
  unsigned grp = __match_any_sync(m, bin);
  if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&h[bin], (uint32_t)__popc(grp));
}

// ============================================================ generic path
__device__ __forceinline__ uint32_t ev_base(const Dev& s) {
  uint32_t b = s.ctl->T_last;
  if (s.policy == 0) b = min(b, s.ctl->min_install);
  return b;
}

// CTA-wide exact selection over u32 values by 3 radix passes (11, 11, 10 bits).
// Returns V with #(val < V) < m <= #(val <= V); *below = #(val < V).
template <typename Get>
__device__ uint32_t cta_select_u32(Get get, int64_t count, int64_t m, int64_t* below, uint32_t* sh_hist) {
  __shared__ int sel;
  __shared__ long long selbelow;
  uint32_t prefix = 0, pmask = 0;
  int64_t acc_below = 0;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
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

__device__ __forceinline__ int key_top(const Dev& s, int64_t key) {
  int sh = s.kbits > 11 ? s.kbits - 11 : 0;
  return (int)(key >> sh) & (NBIN - 1);
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

__device__ __forceinline__ float4 f4add_(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// First bin where the running count of a shared-memory histogram reaches
// `need` (block-wide: per-thread chunks, one block scan, then a short serial
// walk in the crossing chunk).  *s_bin = -1 if the total stays below need.
__device__ __forceinline__ void block_find_cross(const uint32_t* hs, int nb, int64_t need, int* s_bin,
                                                 long long* s_before) {
  __shared__ long long ws[32];
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  long long loc = 0;
  for (int q = b0; q < b1; ++q) loc += hs[q];
  if (threadIdx.x == 0) *s_bin = -1;
  long long tot;
  const long long ex = block_excl_scan64(loc, ws, &tot);
  if (loc > 0 && ex < need && ex + loc >= need) {
    long long cum = ex;
    for (int q = b0; q < b1; ++q) {
      if (cum + hs[q] >= need) { *s_bin = q; *s_before = cum; break; }
      cum += hs[q];
    }
  }
  __syncthreads();
}

// generic exact selection (all blocks of a cooperative grid); sm64 needs SUBMAX*8 bytes
__device__ __forceinline__ void generic_select(const Dev& s, const EvBuf& b, uint64_t* sm64, uint32_t* h,
                                              cg::grid_group& grid) {
  Ctl* ctl = s.ctl;
  const int64_t need = ctl->need;
  const int64_t res = resident_count(s);
  const bool all = need >= res;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t elimit = ((s.Ecap + gstride - 1) / gstride) * gstride;
  // P1: histogram of primaries relative to the lower bound `base`
  uint32_t base = ev_base(s);
  if (!all) {
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int bad = 0;
    for (int64_t e = gtid; e < elimit; e += gstride) {
      bool r = false;
      int bin = 0;
      if (e < s.Ecap) {
        uint32_t prim = s.eprim[e];
        if (prim != EP_FREE) {
          if (prim < base) bad = 1;
          uint32_t rel = prim - base;
          bin = rel < (uint32_t)(NBIN - 1) ? (int)rel : NBIN - 1;
          r = true;
        }
      }
      hist_add(h, bin, r);
    }
    if (bad) b.flags[0] = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x)
      if (h[i]) atomicAdd(&b.hist[i], h[i]);
  }
  grid.sync();
  // P2: threshold T, needT (block 0; the histogram scanned block-wide)
  if (blockIdx.x == 0) {
    __shared__ int s_found, s_bin;
    __shared__ long long s_before;
    if (all) {
      if (threadIdx.x == 0) { ctl->T = 0xFFFFFFFFu; ctl->needT = -1; s_found = 1; }
    } else {
      if (threadIdx.x == 0) s_found = 0;
      const bool bad = b.flags[0] != 0;
      for (int i = threadIdx.x; i < NBIN; i += blockDim.x) h[i] = b.hist[i];
      __syncthreads();
      if (!bad) {
        block_find_cross(h, NBIN - 1, need, &s_bin, &s_before);
        if (threadIdx.x == 0 && s_bin >= 0) {
          ctl->T = base + (uint32_t)s_bin; ctl->needT = need - s_before; s_found = 1;
        }
      }
    }
    __syncthreads();
    if (!s_found) {
      int64_t below;
      auto get = [&](int64_t i, uint32_t* val) -> bool {
        uint32_t p = s.eprim[i];
        *val = p;
        return p != EP_FREE;
      };
      uint32_t T = cta_select_u32(get, s.Ecap, need, &below, h);
      if (threadIdx.x == 0) { ctl->T = T; ctl->needT = need - below; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x) b.hist[i] = 0;
    if (threadIdx.x == 0) {
      b.flags[0] = 0;
      if (!all) ctl->T_last = ctl->T;
      ctl->min_install = 0xFFFFFFFFu;
    }
  }
  grid.sync();
  // P3: victims (prim < T) and candidates (prim == T) + key-top histogram
  const uint32_t T = ctl->T;
  const int64_t needT = ctl->needT;
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t e = gtid; e < elimit; e += gstride) {
    bool isv = false, isc = false;
    int kt = 0;
    if (e < s.Ecap) {
      uint32_t prim = s.eprim[e];
      if (prim != EP_FREE) {
        if (all || prim < T) isv = true;
        else if (prim == T && needT > 0) { isc = true; kt = key_top(s, s.ekey[e]); }
      }
    }
    int vs = warp_append(isv, &ctl->nvict);
    if (isv) b.victims[vs] = (int32_t)e;
    int cs = warp_append(isc, &ctl->ncand);
    if (isc) b.cand[cs] = (int32_t)e;
    hist_add(h, kt, isc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x)
    if (h[i]) atomicAdd(&b.khist[i], h[i]);
  grid.sync();
  // P4: key-top bucket kb1 of the boundary (block 0; block-wide scan)
  if (blockIdx.x == 0) {
    __shared__ int s_kb;
    __shared__ long long s_kbefore;
    const bool scan = needT > 0 && needT < ctl->ncand;
    if (threadIdx.x == 0) {
      ctl->kb1 = 0xFFFFFFFFu;
      ctl->need2 = 0;
      if (needT > 0 && !scan) ctl->kb1 = NBIN;
    }
    if (scan) {
      for (int i = threadIdx.x; i < NBIN; i += blockDim.x) h[i] = b.khist[i];
      __syncthreads();
      block_find_cross(h, NBIN, needT, &s_kb, &s_kbefore);
      if (threadIdx.x == 0 && s_kb >= 0) { ctl->kb1 = (uint32_t)s_kb; ctl->need2 = needT - s_kbefore; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NBIN; i += blockDim.x) b.khist[i] = 0;
  }
  grid.sync();
  // P5: candidates below the bucket are victims, the bucket is the sub list
  const uint32_t kb1 = ctl->kb1;
  if (kb1 != 0xFFFFFFFFu) {
    const int nc = ctl->ncand;
    const int64_t climit = ((nc + gstride - 1) / gstride) * gstride;
    for (int64_t i = gtid; i < climit; i += gstride) {
      bool isv = false, iss = false;
      int32_t e = -1;
      if (i < nc) {
        e = b.cand[i];
        uint32_t kt = (uint32_t)key_top(s, s.ekey[e]);
        if (kb1 == NBIN || kt < kb1) isv = true;
        else if (kt == kb1) iss = true;
      }
      int vs = warp_append(isv, &ctl->nvict);
      if (isv) b.victims[vs] = e;
      int ss = warp_append(iss, &ctl->nsub);
      if (iss) b.sub[ss] = e;
    }
  }
  grid.sync();
  // P6: the need2 smallest keys of the sub list (block 0)
  if (blockIdx.x == 0 && kb1 != 0xFFFFFFFFu && kb1 != NBIN && ctl->need2 > 0) {
    const int nsub = ctl->nsub;
    const int64_t need2 = ctl->need2;
    if (nsub <= SUBMAX) {
      int npad = 2;
      while (npad < nsub) npad <<= 1;
      for (int i = threadIdx.x; i < npad; i += blockDim.x)
        sm64[i] = i < nsub ? (((uint64_t)s.ekey[b.sub[i]] << 24) | (uint64_t)i) : ~0ull;
      __syncthreads();
      bitonic_smem64(sm64, npad);
      int vb = ctl->nvict;
      for (int i = threadIdx.x; i < need2; i += blockDim.x) b.victims[vb + i] = b.sub[(int)(sm64[i] & 0xFFFFFF)];
      __syncthreads();
      if (threadIdx.x == 0) ctl->nvict = vb + (int)need2;
    } else {
      int64_t below;
      auto get = [&](int64_t i, uint32_t* val) -> bool { *val = (uint32_t)s.ekey[b.sub[i]]; return true; };
      uint32_t K = cta_select_u32(get, nsub, need2, &below, h);
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
}

// "When the frequency of an embedding is high enough, it will be
// assigned a direct access index, bypassing the cost of frequency
// maintenance."  The lookup kernels list the entries whose count reached
// pin_thr (pin_candidate); here they are pinned -- eprim = EP_PIN, out of the
// LFU count bitmaps, so never a victim -- in ascending key order while fewer
// than pin_max = floor(C/2) entries are pinned (reading R27).  One CTA (any
// block size), after every touch of the lookup.
__device__ __forceinline__ void pin_apply_block(const Dev& s) {
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ uint32_t h[NBIN];
  __shared__ uint32_t s_K;
  Ctl* ctl = s.ctl;
  const int nc = __ldcg(&ctl->npin_cand);   // other blocks' appends (L2)
  if (nc == 0) return;
  dpop_init(dpop);
  const int64_t budget = s.pin_max - __ldcg(&ctl->npinned);
  uint32_t K = 0xFFFFFFFFu;          // pin the candidates with key <= K
  if (budget > 0 && budget < nc) {          // the budget smallest keys (candidate keys are distinct)
    int64_t below;
    auto get = [&](int64_t i, uint32_t* val) -> bool { *val = (uint32_t)__ldcg(&s.pin_k[i]); return true; };
    const uint32_t T = cta_select_u32(get, nc, budget, &below, h);
    if (threadIdx.x == 0) s_K = T;
    __syncthreads();
    K = s_K;
  }
  __shared__ int s_np;
  if (threadIdx.x == 0) s_np = 0;
  __syncthreads();
  if (budget > 0) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const int64_t key = __ldcg(&s.pin_k[i]);
      if ((uint64_t)key > (uint64_t)K) continue;
      const int32_t e = __ldcg(&s.pin_e[i]);
      const uint32_t oldc = __ldcg(&s.eprim[e]);
      lfu_move(s, key, oldc, EP_PIN, dpop);   // EP_PIN >= lfu_cb: out of the bitmaps
      s.eprim[e] = EP_PIN;
      atomicAdd(&s_np, 1);
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    ctl->npinned += s_np;
    ctl->npin_cand = 0;
  }
}

}  // namespace het
