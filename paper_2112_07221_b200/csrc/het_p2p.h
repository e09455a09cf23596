// Device-initiated multi-GPU exchange over NVLink peer memory (internal).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/het.h"
#include "het_internal.cuh"

namespace het {

struct P2PState;

// A row's record list holds at most 32 records and a source sends at most two
// per row (a carried eviction push + a request), so N <= 16.
constexpr int P2P_MAX_WORLD = 16;

// Phases of one exchange round.  One process per GPU runs them back to back
// (or as one cooperative kernel); the loopback driver (N workers on one GPU)
// runs each phase for every worker before the next phase of any, so every
// flag a phase waits for is already set.
enum { RP_BUILD = 0, RP_LINK = 1, RP_PROCESS = 2, RP_INSTALL = 3, RP_NUM = 4 };

// comm == nullptr: a loopback worker (no CUDA IPC; p2p_loopback_connect fills
// the peer tables).  dense_cap: floats of the dense all-reduce staging.
het_status_t p2p_create(P2PState*& out, const Dev& d, uint32_t n_max, ncclComm_t comm, uint64_t dense_cap,
                        cudaStream_t st);
het_status_t p2p_loopback_connect(P2PState* const* ps, int N, cudaStream_t st);
void p2p_destroy(P2PState* p);
bool p2p_loopback(const P2PState* p);
int64_t p2p_caps(const P2PState* p);
// one round after the probe (drain = no requests, only pending pushes)
int p2p_round(P2PState* p, const Dev& d, const Call& c, int drain, cudaStream_t st);
int p2p_round_phase(P2PState* p, const Dev& d, const Call& c, int drain, int phase, cudaStream_t st);
// fused round (after the dedup): probe+build, link, process, install+gather
int p2p_round_fused(P2PState* p, const Dev& d, const Call& c, float* out, cudaStream_t st);
int p2p_lookup_phase(P2PState* p, const Dev& d, const Call& c, float* out, int phase, cudaStream_t st);
// device view of the exchange state (for the fused update's eviction pushes)
struct P2P;
P2P* p2p_view_ptr(P2PState* p);
// eviction pushes of the current update (sent with the next round)
int p2p_pushes(P2PState* p, const Dev& d, void* evbuf, cudaStream_t st);
// het_sync: PUSH records of the dirty entries with key in [k0, k1) (sent by the next drain round)
int p2p_flush_build(P2PState* p, const Dev& d, int64_t k0, int64_t k1, cudaStream_t st);
// explicit Evict(key) of the call's unique keys: PUSH records + local delete
int p2p_evict_keys(P2PState* p, const Dev& d, const Call& c, cudaStream_t st);
// Eq. 2 dense all-reduce (mean) over peer memory; phase 0 whole, 1 stage +
// publish, 2 wait + sum.  HET_ERR_CAPACITY when count exceeds the staging set
// up at create (every rank then takes the NCCL all-reduce: count is collective).
het_status_t p2p_dense_allreduce(P2PState* p, const Dev& d, float* buf, uint64_t count, int phase, cudaStream_t st,
                                 int* launches);

}  // namespace het
