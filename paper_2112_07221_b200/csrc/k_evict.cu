// K8/K9 — Cache.Evict() overflow eviction ("evict the overflowed
// embeddings selected by certain cache policies", Alg. 3 line 4):
// exactly |cache| - C victims, the smallest by (count, key) under LFU or
// (tick, key) under LRU among ALL resident entries (reading R9), then the
// Evict push of each dirty victim: W += p, c_g = max(c_g, c_c).
//
// Two exact selection paths:
//  * LFU bitmap path (k_ev_select): resident keys with count c < lfu_cb are
//    kept in per-count key bitmaps with per-4096-key block counters and
//    per-count populations, maintained incrementally by probe/install/evict.
//    The threshold count T comes from the populations; victims are all keys
//    of counts < T plus the first needT keys (ascending) of count T, found
//    with one CTA-wide scan of T's block counters and a warp-parallel bit
//    extraction.  Cost O(R/4096 + victims) per step, no scan of the cache.
//  * generic path (k_ev_generic, one cooperative kernel): histogram of the
//    residents' primaries relative to a proven lower bound, threshold,
//    collection of victims/candidates, key-top histogram of the candidates,
//    and a final sort of the boundary bucket.  Used for LRU and whenever the
//    LFU threshold count is >= lfu_cb.
#include "evict_dev.cuh"

namespace het {

size_t evbuf_struct_size() { return sizeof(EvBuf); }

void evbuf_init(void* evbuf, uint32_t* hist, uint32_t* khist, int32_t* victims, int32_t* cand,
                int32_t* sub, int32_t* flags, int64_t* vkeys, uint8_t* vdirty, int64_t* vsel) {
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  b.hist = hist; b.khist = khist; b.victims = victims; b.cand = cand; b.sub = sub; b.flags = flags;
  b.vkeys = vkeys; b.vdirty = vdirty; b.vsel = vsel;
}

// ============================================================ light-LFU promotion
// (pin_apply_block in evict_dev.cuh; the fused N = 1 lookups run it in their
// last block, the other lookup paths launch this kernel after the lookup)
__global__ void __launch_bounds__(1024) k_pin_apply(Dev s) { pin_apply_block(s); }

int launch_pin_apply(const Dev& s, cudaStream_t st) {
  k_pin_apply<<<1, 1024, 0, st>>>(s);
  return 1;
}

// ============================================================ LFU bitmap path
// first `limit` set bits (ascending key) of count-c bitmap -> vsel[out ...]
__device__ void bitmap_extract(const Dev& s, const EvBuf& b, int c, int64_t limit, int64_t out,
                               long long* warp_sums, int* s_nlist) {
  const uint32_t* bc = s.bcnt + (int64_t)c * s.nbk;
  const uint32_t* bm = s.bm + (int64_t)c * s.bm_words;
  int64_t per = (s.nbk + blockDim.x - 1) / blockDim.x;
  int64_t b0 = threadIdx.x * per, b1 = min(b0 + per, s.nbk);
  int64_t local = 0;
  for (int64_t k = b0; k < b1; ++k) local += bc[k];
  long long tot;
  if (threadIdx.x == 0) *s_nlist = 0;
  int64_t off = block_excl_scan64(local, warp_sums, &tot);
  // blocks holding positions < limit -> work list (block id, first position)
  for (int64_t k = b0; k < b1 && off < limit; ++k) {
    uint32_t cnt = bc[k];
    if (cnt) {
      int li = atomicAdd(s_nlist, 1);
      b.sub[li] = (int32_t)k;
      b.cand[li] = (int32_t)off;
      off += cnt;
    }
  }
  __syncthreads();
  int nlist = *s_nlist;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int li = wid; li < nlist; li += nw) {
    int64_t blk = b.sub[li];
    int64_t pos0 = b.cand[li];
    uint32_t w[4];
    int cntl = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t wi = (blk << (LFU_BLK_SHIFT - 5)) + lane * 4 + q;
      w[q] = wi < s.bm_words ? bm[wi] : 0u;
      cntl += __popc(w[q]);
    }
    int incl = cntl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int64_t pos = pos0 + incl - cntl;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t bits = w[q];
      int64_t wbase = ((blk << (LFU_BLK_SHIFT - 5)) + lane * 4 + q) << 5;
      while (bits && pos < limit) {
        int bi = __ffs(bits) - 1;
        b.vsel[out + pos] = wbase + bi;
        ++pos;
        bits &= bits - 1;
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024)
k_ev_select(Dev s, EvBuf b) {
  __shared__ long long warp_sums[32];
  __shared__ int s_nlist, s_mode, s_T;
  __shared__ long long s_needT;
  Ctl* ctl = s.ctl;
  int64_t res = resident_count(s);
  int64_t need = res - s.C;
  if (threadIdx.x == 0) {
    ctl->nvict = 0; ctl->ncand = 0; ctl->nsub = 0; ctl->vmode = 0;
    bool none = ctl->abort || need <= 0;
    ctl->need = none ? 0 : need;
    int mode = 0;  // 0 nothing, 1 bitmap, 2 generic
    if (!none) {
      mode = 2;
      if (s.lfu_cb && need < res) {
        int64_t cum = 0;
        for (int c = 0; c < s.lfu_cb; ++c) {
          int64_t pc = s.pop[c];
          if (cum + pc >= need) { s_T = c; s_needT = need - cum; mode = 1; break; }
          cum += pc;
        }
      }
    }
    ctl->generic = mode == 2;
    s_mode = mode;
  }
  __syncthreads();
  if (s_mode != 1) return;
  int T = s_T;
  int64_t out = 0;
  for (int c = 0; c <= T; ++c) {
    int64_t limit = c < T ? (int64_t)s.pop[c] : (int64_t)s_needT;
    if (limit <= 0) continue;
    bitmap_extract(s, b, c, limit, out, warp_sums, &s_nlist);
    out += limit;
  }
  if (threadIdx.x == 0) {
    ctl->nvict = (int32_t)need;
    ctl->vmode = 1;
  }
}

__global__ void __launch_bounds__(GEN_THREADS)
k_ev_generic(Dev s, EvBuf b) {
  extern __shared__ uint64_t sm64[];
  __shared__ uint32_t h[NBIN];
  cg::grid_group grid = cg::this_grid();
  if (!s.ctl->generic) return;
  generic_select(s, b, sm64, h, grid);
}

__global__ void __launch_bounds__(256)
k_ev_apply_local(Dev s, EvBuf b) {
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty;
  dpop_init(dpop);
  if (threadIdx.x == 0) s_dirty = 0;
  __syncthreads();
  Ctl* ctl = s.ctl;
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  if (!ctl->abort && ctl->need > 0) {
    const int nv = ctl->nvict;
    const bool bykey = ctl->vmode == 1;
    const int D4 = s.D >> 2;
    for (int i = w; i < nv; i += nw) {
      int32_t e;
      int64_t key;
      uint64_t slot = 0;
      if (bykey) { key = b.vsel[i]; e = warp_find_slot(s, key, lane, &slot); }
      else { e = b.victims[i]; key = s.ekey[e]; e = warp_find_slot(s, key, lane, &slot); }
      const uint32_t ecs = s.cs[e], ecc = s.cc[e], prim = s.eprim[e];
      // row loads issued before the dirty test (victims are almost always dirty)
      float4* Wr = reinterpret_cast<float4*>(s.W + key * s.D);
      const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
      const bool dirty = ecc > ecs;
      for (int d = lane; d < D4; d += 32) {
        float4 wv = Wr[d], pv = pr[d];
        if (dirty) Wr[d] = f4add_(wv, pv);     // Evict push: W += p
      }
      if (lane == 0) {
        if (dirty) { uint32_t g = s.cg[key]; s.cg[key] = g > ecc ? g : ecc; }
        s.hslot[slot] = HS_TOMB;
        atomicAdd(&ctl->n_tomb, 1);
        b.vkeys[i] = key;
        b.vdirty[i] = dirty ? 1 : 0;
        if (dirty) atomicAdd(&s_dirty, 1u);
        if (s.policy == 0) lfu_move(s, key, prim, EP_FREE, dpop);
    unpin_count(s, prim);
        s.eprim[e] = EP_FREE;
        s.ekey[e] = -1;
        s.fstack[atomicAdd(&ctl->ftop, 1)] = e;
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)nv);
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0 && s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
}

static int g_coop_blocks = 0;

int launch_evict_select(const Dev& s, void* evbuf, cudaStream_t st) {
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  k_ev_select<<<1, 1024, 0, st>>>(s, b);
  if (!g_coop_blocks) {
    int dev, sms, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_ev_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, SUBMAX * 8);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ev_generic, GEN_THREADS, SUBMAX * 8);
    g_coop_blocks = sms * (per > 0 ? per : 1);
  }
  void* args[] = {(void*)&s, (void*)&b};
  cudaLaunchCooperativeKernel((void*)k_ev_generic, dim3(g_coop_blocks), dim3(GEN_THREADS), args,
                              SUBMAX * 8, st);
  return 2;
}

int launch_evict_apply_local(const Dev& s, void* evbuf, cudaStream_t st) {
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  k_ev_apply_local<<<148 * 2, 256, 0, st>>>(s, b);
  return 1;
}

void cache_set_attrs() {}

}  // namespace het
