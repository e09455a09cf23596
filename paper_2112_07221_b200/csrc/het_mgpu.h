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

// uid == nullptr: a loopback worker (no NCCL communicator; see het_group_create)
het_status_t mgpu_create(MgpuState*& mg, const Dev& d, uint32_t n_max, const void* uid, uint64_t dense_cap,
                         cudaStream_t st);
bool mgpu_loopback(MgpuState* mg);
void mgpu_destroy(MgpuState* mg);
het_status_t mgpu_lookup(MgpuState* mg, const Dev& d, const Call& c, void* prof, cudaStream_t st);
het_status_t mgpu_evict_overflow(MgpuState* mg, const Dev& d, void* evbuf, void* prof, cudaStream_t st);
// NCCL exchange (HET_P2P=0) only: explicit evict and flush
het_status_t mgpu_evict_keys(MgpuState* mg, const Dev& d, const Call& c, cudaStream_t st);
het_status_t mgpu_flush(MgpuState* mg, const Dev& d, cudaStream_t st);
// het_sync over the peer-memory exchange: dirty entries per key bin (host copy),
// max over ranks (NCCL, one process per GPU)
constexpr int FBINS = 1024;
het_status_t mgpu_flush_hist(MgpuState* mg, const Dev& d, int64_t k0, int64_t k1, int32_t* bins_host,
                             cudaStream_t st);
het_status_t mgpu_allreduce_max_host(MgpuState* mg, int32_t* x, int count, cudaStream_t st);
// latched asynchronous NCCL error of the communicator (ncclCommGetAsyncError)
het_status_t mgpu_comm_error(MgpuState* mg);
het_status_t mgpu_allreduce_sum(MgpuState* mg, float* buf, uint64_t count, cudaStream_t st);
// Eq. 2 mean over peer memory (p2p exchange only); HET_ERR_CAPACITY -> use NCCL
het_status_t mgpu_dense_p2p(MgpuState* mg, const Dev& d, float* buf, uint64_t count, int phase, cudaStream_t st,
                            int* launches);
void mgpu_bytes(MgpuState* mg, uint64_t* ctx, uint64_t* crx, uint64_t* etx, uint64_t* erx);
uint64_t mgpu_take_launches(MgpuState* mg);

void* prof_begin(void* h, const char* name, cudaStream_t st);
void prof_end(void* h, void* rec, cudaStream_t st);

}  // namespace het
