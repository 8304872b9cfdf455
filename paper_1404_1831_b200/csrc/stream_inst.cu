// The large-cell stream kernels (point-term FBPQ) for one M, selected by
// -DBPQ_INST_M=<8|16> (see the Makefile): their own translation units so they
// rebuild without the fused search kernel.
#include "stream_impl.cuh"

#ifndef BPQ_INST_M
#error "compile with -DBPQ_INST_M=8 or 16"
#endif

namespace bpq {

template <>
int launch_big_inst<BPQ_INST_M>(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                                int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc,
                                cudaStream_t s) {
    return launch_big_one<BPQ_INST_M>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, s);
}

}  // namespace bpq
