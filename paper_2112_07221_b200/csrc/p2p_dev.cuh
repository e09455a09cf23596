// Peer-memory exchange device view and helpers (shared by het_p2p.cu and k_fused.cu).
#pragma once
#include "het_internal.cuh"

namespace het {

enum : uint32_t { K_PUSH = 0, K_NEEDQ = 1, K_EXP1 = 2, K_MISS = 3, K_DIRTY = 4 };
constexpr unsigned long long WAIT_NS = 20ull * 1000 * 1000 * 1000;  // 20 s

struct alignas(16) Flag {
  unsigned long long epoch;
  uint32_t total;
  uint32_t pushes;
};
struct alignas(16) Rec {
  int64_t key;
  uint32_t cc;
  uint32_t kind;
};

// POD view passed to kernels
struct P2P {
  int N, rank;
  int64_t CAPS, REC;
  uint32_t D;
  char* const* peer;            // [N] base of every rank's inbox (own included)
  size_t off_reqflag, off_respflag, off_req, off_rows, off_resp;
  int32_t* lcnt;                // [N] this round's requests per owner
  int32_t* c3cnt;               // [N] pending eviction pushes per owner
  int32_t* ridx;                // [N][CAPS] unique index of each request
  int32_t* head;                // [rows_local] list head per local row (-1)
  int32_t* next;                // [N*CAPS]
  int32_t* leaders;             // [N*CAPS]
  int32_t* nlead;
  int32_t* done;                // [4] last-block counters
  unsigned long long* epoch;    // completed rounds
  int32_t* qtot;                // [N] received totals (owner, this round)
  int32_t* qpush;               // [N] received pushes (owner, this round)
  int32_t* uslot;               // [n_max] request location (owner*CAPS + slot) per unique key
};

__device__ __forceinline__ Flag* reqflag(const P2P& m, int r) { return (Flag*)(m.peer[r] + m.off_reqflag); }
__device__ __forceinline__ Flag* respflag(const P2P& m, int r) { return (Flag*)(m.peer[r] + m.off_respflag); }
__device__ __forceinline__ Rec* reqrec(const P2P& m, int r, int src) {
  return (Rec*)(m.peer[r] + m.off_req) + (int64_t)src * m.CAPS;
}
__device__ __forceinline__ float* reqrow(const P2P& m, int r, int src, int64_t j) {
  return (float*)(m.peer[r] + m.off_rows) + ((int64_t)src * m.CAPS + j) * m.D;
}
__device__ __forceinline__ float* resprec(const P2P& m, int r, int owner, int64_t j) {
  return (float*)(m.peer[r] + m.off_resp) + ((int64_t)owner * m.CAPS + j) * m.REC;
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait until flags[0..N) carry `epoch`; false on timeout (sticky error raised)
__device__ __forceinline__ bool wait_flags(Flag* flags, int N, unsigned long long epoch, Ctl* ctl) {
  unsigned long long t0 = gtime();
  for (int r = 0; r < N; ++r) {
    while (ld_acquire(&flags[r].epoch) < epoch) {
      if (gtime() - t0 > WAIT_NS) {
        raise_err(ctl, 7 /*HET_ERR_NCCL: peer exchange timeout*/);
        return false;
      }
      __nanosleep(64);
    }
  }
  return true;
}

__device__ __forceinline__ float4 f4add_p(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// block-aggregated wire-byte counters (clock tx/rx, embedding tx/rx)
struct Bytes {
  unsigned long long v[4];
};
__device__ __forceinline__ void bytes_init(unsigned long long* b) {
  if (threadIdx.x < 4) b[threadIdx.x] = 0;
}
__device__ __forceinline__ void bytes_flush(const Dev& s, unsigned long long* b) {
  if (threadIdx.x < 4 && b[threadIdx.x]) atomicAdd(&s.cnt[C_BCLK_TX + threadIdx.x], b[threadIdx.x]);
}

// Last-block election.  Each block orders its writes with a GPU-scope fence
// before the counter; the elected block then issues the system-scope fence
// and the release store of the flag (causality is transitive: block writes
// -> fence.gpu -> counter -> elected block -> fence.sys -> st.release.sys),
// so only the publishing thread pays for system scope.
__device__ __forceinline__ bool last_block(int32_t* counter) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) __threadfence_system();
  return s_last;
}

// Eviction push of one dirty entry to its owner's inbox (carried by the next
// round): record {key, c_c, PUSH} + pending row at the source's push cursor.
__device__ __forceinline__ void push_record(const Dev& s, const P2P& m, int32_t e, int64_t key, uint32_t ecc,
                                            int lane) {
  const int o = (int)(key % m.N);
  int ps = 0;
  if (lane == 0) ps = atomicAdd(&m.c3cnt[o], 1);
  ps = __shfl_sync(0xffffffffu, ps, 0);
  HET_ASSERT(ps >= 0 && ps < m.CAPS);
  if (lane == 0) {
    Rec r;
    r.key = key; r.cc = ecc; r.kind = K_PUSH | K_DIRTY;
    reqrec(m, o, m.rank)[ps] = r;
  }
  const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
  float4* dst = reinterpret_cast<float4*>(reqrow(m, o, m.rank, ps));
  const int D4 = (int)(s.D >> 2);
  for (int d0 = lane; d0 < D4; d0 += 32 * 4) {   // loads of 4 columns before their stores (wide rows)
    float4 t[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) if (d0 + 32 * b < D4) t[b] = pr[d0 + 32 * b];
#pragma unroll
    for (int b = 0; b < 4; ++b) if (d0 + 32 * b < D4) dst[d0 + 32 * b] = t[b];
  }
}

}  // namespace het
