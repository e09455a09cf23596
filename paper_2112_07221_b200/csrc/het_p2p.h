// Device-initiated multi-GPU exchange over NVLink peer memory (internal).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/het.h"
#include "het_internal.cuh"

namespace het {

struct P2PState;

het_status_t p2p_create(P2PState*& out, const Dev& d, uint32_t n_max, ncclComm_t comm, cudaStream_t st);
void p2p_destroy(P2PState* p);
// one lookup round after the probe: build + publish, owner link + process, install
int p2p_round(P2PState* p, const Dev& d, const Call& c, int drain, cudaStream_t st);
// fused round (n <= 8192, after k_dd_fused): probe+build, link, process, install+gather
int p2p_round_fused(P2PState* p, const Dev& d, const Call& c, float* out, cudaStream_t st);
// device view of the exchange state (for the fused update's eviction pushes)
struct P2P;
P2P* p2p_view_ptr(P2PState* p);
// eviction pushes of the current update (sent with the next round)
int p2p_pushes(P2PState* p, const Dev& d, void* evbuf, cudaStream_t st);
// Eq. 2 dense all-reduce (mean) over peer memory; HET_ERR_CAPACITY when
// count exceeds the staging set up by the first call (the caller falls back
// to NCCL).  The first call allocates and exchanges the staging (collective,
// outside graph capture).
het_status_t p2p_dense_allreduce(P2PState* p, const Dev& d, float* buf, uint64_t count, ncclComm_t comm,
                                 cudaStream_t st, int* launches);

}  // namespace het
