// Instantiations of the fused search kernel for engine BPQ_ENGINE_HBPQ
// (split per engine so the instantiations compile in parallel).
#include "search_impl.cuh"

namespace bpq {

void set_prof_buffer_e2(unsigned long long *p) { g_prof_buffer = p; }

int launch_search_e2(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                      int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc,
                      int64_t *on, int64_t *op, cudaStream_t s) {
    return dispatch_m<BPQ_ENGINE_HBPQ>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
}

}  // namespace bpq
