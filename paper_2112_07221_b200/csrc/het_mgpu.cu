// Multi-GPU path: placeholder until the sharded exchange lands.
#include "het_mgpu.h"

namespace het {

struct MgpuState {
  int dummy;
};

het_status_t mgpu_create(MgpuState*& mg, const Dev&, uint32_t, const void*, cudaStream_t) {
  mg = nullptr;
  return HET_ERR_ARG;
}
void mgpu_destroy(MgpuState* mg) { delete mg; }
het_status_t mgpu_lookup(MgpuState*, const Dev&, const Call&, void*, cudaStream_t) { return HET_ERR_ARG; }
het_status_t mgpu_evict_overflow(MgpuState*, const Dev&, void*, void*, cudaStream_t) { return HET_ERR_ARG; }
het_status_t mgpu_evict_keys(MgpuState*, const Dev&, const Call&, cudaStream_t) { return HET_ERR_ARG; }
het_status_t mgpu_flush(MgpuState*, const Dev&, cudaStream_t) { return HET_ERR_ARG; }
het_status_t mgpu_allreduce_sum(MgpuState*, float*, uint64_t, cudaStream_t) { return HET_ERR_ARG; }
void mgpu_bytes(MgpuState*, uint64_t* a, uint64_t* b, uint64_t* c, uint64_t* d) { *a = *b = *c = *d = 0; }
uint64_t mgpu_take_launches(MgpuState*) { return 0; }

}  // namespace het
