// Instantiations of the fused search kernel for engine BPQ_ENGINE_FBPQ
// (split per engine so the instantiations compile in parallel).
#include "search_impl.cuh"

namespace bpq {

void set_prof_buffer_e1(unsigned long long *p) { g_prof_buffer = p; }

int launch_search_e1(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                      int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc,
                      int64_t *on, int64_t *op, cudaStream_t s) {
    return dispatch_m<BPQ_ENGINE_FBPQ>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
}

int search_grid_ctas(int engine, int M) {
    // upper bound over launches: the smallest dynamic footprint gives the most CTAs
    (void)engine;
    (void)M;
    int n = 0;
    if (configure<BPQ_ENGINE_FBPQ, 8, float, uint32_t>(dyn_smem_bytes(4, 0, 4, topk_capacity(1)), &n)) return -1;
    return n;
}

}  // namespace bpq
