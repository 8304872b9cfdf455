// One instantiation of the fused search kernel, selected at compile time by
// -DBPQ_INST_ENGINE=<0|1|2> -DBPQ_INST_M=<8|16|0> (see the Makefile): one
// (engine, M) pair per translation unit so the nine ptxas runs go parallel.
#include "search_impl.cuh"

#ifndef BPQ_INST_ENGINE
#error "compile with -DBPQ_INST_ENGINE=... -DBPQ_INST_M=..."
#endif

namespace bpq {

template <>
int launch_search_inst<BPQ_INST_ENGINE, BPQ_INST_M>(const Index &ix, const float *queries, int64_t q0,
                                                    int64_t nq, int64_t budget, int32_t k,
                                                    const SearchWorkspace &ws, float *od, uint32_t *oi,
                                                    int32_t *oc, int64_t *on, int64_t *op, cudaStream_t s) {
    return launch_one<BPQ_INST_ENGINE, BPQ_INST_M>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
}

#if BPQ_INST_ENGINE == 1 && BPQ_INST_M == 8  // FBPQ
int search_grid_ctas(int engine, int M) {
    // upper bound over launches: the smallest dynamic footprint gives the most CTAs
    (void)engine;
    (void)M;
    int n = 0;
    if (configure<BPQ_ENGINE_FBPQ, 8, float, uint32_t>(dyn_smem_bytes(4, 0, 4, topk_capacity(1)), &n)) return -1;
    return n;
}
#endif

}  // namespace bpq
