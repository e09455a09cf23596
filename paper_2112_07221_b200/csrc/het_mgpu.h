// Multi-GPU orchestration (one worker per GPU, hash-sharded server, NCCL
// all-to-all exchanges over NVLink).  Internal to libhet.
#pragma once
#include <cuda_runtime.h>

#include "../../include/het.h"
#include "het_internal.cuh"

namespace het {

struct MgpuState;
struct P2PState;
P2PState* mgpu_p2p(MgpuState* mg);   // device-initiated exchange state, nullptr if NCCL v1

het_status_t mgpu_create(MgpuState*& mg, const Dev& d, uint32_t n_max, const void* uid, cudaStream_t st);
void mgpu_destroy(MgpuState* mg);
het_status_t mgpu_lookup(MgpuState* mg, const Dev& d, const Call& c, void* prof, cudaStream_t st);
het_status_t mgpu_evict_overflow(MgpuState* mg, const Dev& d, void* evbuf, void* prof, cudaStream_t st);
het_status_t mgpu_evict_keys(MgpuState* mg, const Dev& d, const Call& c, cudaStream_t st);
het_status_t mgpu_flush(MgpuState* mg, const Dev& d, cudaStream_t st);
// deliver the eviction pushes still waiting for the next exchange round
het_status_t mgpu_drain(MgpuState* mg, const Dev& d, const Call& c, cudaStream_t st);
het_status_t mgpu_allreduce_sum(MgpuState* mg, float* buf, uint64_t count, cudaStream_t st);
// Eq. 2 mean over peer memory (p2p exchange only); HET_ERR_CAPACITY -> use NCCL
het_status_t mgpu_dense_p2p(MgpuState* mg, const Dev& d, float* buf, uint64_t count, cudaStream_t st,
                            int* launches);
void mgpu_bytes(MgpuState* mg, uint64_t* ctx, uint64_t* crx, uint64_t* etx, uint64_t* erx);
uint64_t mgpu_take_launches(MgpuState* mg);

void* prof_begin(void* h, const char* name, cudaStream_t st);
void prof_end(void* h, void* rec, cudaStream_t st);

}  // namespace het
