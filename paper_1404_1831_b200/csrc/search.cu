// Stage mirrors of the reference kernel backend (traverse_cells, scan_*)
// and the engine dispatch of the batched search.
#include <cub/device/device_radix_sort.cuh>

#include "search_impl.cuh"

namespace bpq {
unsigned long long *g_prof_buffer = nullptr;

#define BPQ_DECL_INST(E, M)                                                                        \
    template <>                                                                                    \
    int launch_search_inst<E, M>(const Index &, const float *, int64_t, int64_t, int64_t, int32_t, \
                                 const SearchWorkspace &, float *, uint32_t *, int32_t *, int64_t *, \
                                 int64_t *, cudaStream_t);
BPQ_DECL_INST(0, 8) BPQ_DECL_INST(0, 16) BPQ_DECL_INST(0, 0)
BPQ_DECL_INST(1, 8) BPQ_DECL_INST(1, 16) BPQ_DECL_INST(1, 0)
BPQ_DECL_INST(2, 8) BPQ_DECL_INST(2, 16) BPQ_DECL_INST(2, 0)

template <>
int launch_big_inst<8>(const Index &, const float *, int64_t, int64_t, int64_t, int32_t, const SearchWorkspace &,
                       float *, uint32_t *, int32_t *, cudaStream_t);
template <>
int launch_big_inst<16>(const Index &, const float *, int64_t, int64_t, int64_t, int32_t, const SearchWorkspace &,
                        float *, uint32_t *, int32_t *, cudaStream_t);

int effective_lut_min() {
    static const int env = getenv("BPQ_LUT_MIN") ? atoi(getenv("BPQ_LUT_MIN")) : 0;  // A/B experiments
    return env > 0 ? env : kLutMin;
}

int launch_big_scan(const Index &ix, int engine, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                    int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc, cudaStream_t s) {
    if (nq == 0 || engine != BPQ_ENGINE_FBPQ || ws.big_cells == nullptr || ix.pterm == nullptr) return BPQ_OK;
    if (ix.M == 8) return launch_big_inst<8>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, s);
    if (ix.M == 16) return launch_big_inst<16>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, s);
    return BPQ_OK;
}

template <int ENGINE>
int dispatch_m(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
               int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc,
               int64_t *on, int64_t *op, cudaStream_t s) {
    switch (ix.M) {
        case 8: return launch_search_inst<ENGINE, 8>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 16: return launch_search_inst<ENGINE, 16>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 2: case 4: case 6: case 10: case 12: case 14:
            return launch_search_inst<ENGINE, 0>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
    }
    return fail(BPQ_ERR_UNSUPPORTED, "num_parts must be even and in [2, 16]");
}

namespace {
// ------------------------------------------- stage mirrors: per-candidate scans
__global__ void stage_scan_kernel(int engine, const int32_t *__restrict__ vis_i,
                                  const int32_t *__restrict__ vis_j,
                                  const int64_t *__restrict__ starts,
                                  const int64_t *__restrict__ cand_start, int64_t nvis,
                                  int64_t ncand, const uint32_t *__restrict__ ids,
                                  const uint8_t *__restrict__ codes, int m, int K, int ds,
                                  float q_norm, const float *__restrict__ qd1,
                                  const float *__restrict__ qd2, const float *__restrict__ cn1,
                                  const float *__restrict__ cn2, const float *__restrict__ fold,
                                  const float *__restrict__ t1, const float *__restrict__ t2,
                                  const float *__restrict__ e1, const float *__restrict__ e2,
                                  const float *__restrict__ books, uint32_t *__restrict__ out_ids,
                                  float *__restrict__ out_d) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncand) return;
    int64_t lo = 0, hi = nvis;  // largest v with cand_start[v] <= c
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (cand_start[mid] <= c) lo = mid; else hi = mid;
    }
    const int64_t v = lo;
    const int64_t entry = starts[v] + (c - cand_start[v]);
    const int64_t i = vis_i[v], j = vis_j[v];
    const int m2 = m / 2;
    const uint8_t *cp = codes + entry * m;
    float acc;
    if (engine == BPQ_ENGINE_FBPQ) {
        acc = __fadd_rn(__fadd_rn(__fsub_rn(q_norm, __fmul_rn(2.f, __fadd_rn(qd1[i], qd2[j]))), cn1[i]), cn2[j]);
        for (int p = 0; p < m2; p++) {
            int cc = cp[p];
            acc = __fadd_rn(acc, __fadd_rn(fold[p * K + cc], __fmul_rn(2.f, t1[(i * m2 + p) * K + cc])));
        }
        for (int p = m2; p < m; p++) {
            int cc = cp[p];
            acc = __fadd_rn(acc, __fadd_rn(fold[p * K + cc], __fmul_rn(2.f, t2[(j * m2 + (p - m2)) * K + cc])));
        }
        if (acc < 0.f) acc = 0.f;
    } else {
        const int dh = m2 * ds;
        acc = 0.f;
        for (int p = 0; p < m; p++) {
            const int hp = p < m2 ? p : p - m2;
            const float *er = (p < m2 ? e1 + i * dh : e2 + j * dh) + hp * ds;
            const int cc = cp[p];
            const float *bk;
            if (engine == BPQ_ENGINE_HBPQ)
                bk = (p < m2 ? t1 + ((i * m2 + hp) * (int64_t)K + cc) * ds
                             : t2 + ((j * m2 + hp) * (int64_t)K + cc) * ds);
            else
                bk = books + ((int64_t)p * K + cc) * ds;
            for (int u = 0; u < ds; u++) {
                float d = __fsub_rn(er[u], bk[u]);
                acc = __fadd_rn(acc, __fmul_rn(d, d));
            }
        }
    }
    out_ids[c] = ids[entry];
    out_d[c] = acc;
}

__global__ void traverse_finish_kernel(const uint32_t *__restrict__ lin_sorted,
                                       const int64_t *__restrict__ st, const int64_t *__restrict__ en,
                                       const uint32_t *__restrict__ perm, const unsigned long long *n,
                                       int64_t t, int32_t *vi, int32_t *vj, int64_t *so,
                                       int64_t *eo, int64_t *nvis_out) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nn = (int64_t)*n;
    if (x == 0) *nvis_out = nn;
    if (x >= nn) return;
    uint32_t lin = lin_sorted[x];
    vi[x] = (int32_t)(lin / t);
    vj[x] = (int32_t)(lin % t);
    uint32_t src = perm[x];
    so[x] = st[src];
    eo[x] = en[src];
}

__global__ void pad_tail_kernel(unsigned long long *key, uint32_t *lin,
                                const unsigned long long *n, int cap) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < cap && (unsigned long long)x >= *n) {
        key[x] = ~0ull;
        if (lin) lin[x] = ~0u;
    }
}

__global__ void iota_kernel(uint32_t *p, int64_t n) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) p[x] = (uint32_t)x;
}

__global__ void gather_key_kernel(const unsigned long long *key, const uint32_t *perm,
                                  unsigned long long *out, const unsigned long long *n) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < (int64_t)*n) out[x] = key[perm[x]];
}

__global__ void gather_lin_kernel(const uint32_t *lin, const uint32_t *perm, uint32_t *out,
                                  const unsigned long long *n) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < (int64_t)*n) out[x] = lin[perm[x]];
}

struct TravLayout {
    size_t off_scratch, off_key, off_lin, off_st, off_en, off_n, off_perm0, off_perm1, off_keys2,
        off_lin2, off_cub, total;
    size_t cub_bytes;
    int64_t cap;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

TravLayout trav_layout(int64_t t, int64_t budget, int64_t total) {
    TravLayout L{};
    int64_t cap = budget < total ? budget : total;
    if (cap > t * t) cap = t * t;
    if (cap < 1) cap = 1;
    L.cap = cap;
    size_t o = 0;
    L.off_scratch = o;
    o += al(search_cta_scratch_bytes((int32_t)t, 0));
    L.off_key = o; o += al(cap * 8);
    L.off_lin = o; o += al(cap * 4);
    L.off_st = o; o += al(cap * 8);
    L.off_en = o; o += al(cap * 8);
    L.off_n = o; o += al(8);
    L.off_perm0 = o; o += al(cap * 4);
    L.off_perm1 = o; o += al(cap * 4);
    L.off_keys2 = o; o += al(cap * 8);
    L.off_lin2 = o; o += al(cap * 4);
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs<unsigned long long, uint32_t>(nullptr, a, nullptr, nullptr, nullptr, nullptr, (int)cap);
    cub::DeviceRadixSort::SortPairs<uint32_t, uint32_t>(nullptr, b, nullptr, nullptr, nullptr, nullptr, (int)cap);
    L.cub_bytes = a > b ? a : b;
    L.off_cub = o; o += al(L.cub_bytes);
    L.off_cub += 0;
    o += al(4);  // counter
    L.total = o;
    return L;
}

}  // namespace

size_t search_cta_scratch_bytes(int32_t T, int32_t D) {
    // row/column state, segments, four cell lists, rotated query displacements (HBPQ)
    return (((size_t)6 * T * 4 + 15) & ~(size_t)15) + (size_t)2 * T * sizeof(uint4) +
           (size_t)4 * kBandCap * sizeof(int4) + (size_t)kSearchThreads * D * 4;
}



int launch_search(const Index &ix, int engine, const float *queries, int64_t q0, int64_t nq,
                  int64_t budget, int32_t k, const SearchWorkspace &ws, float *out_dist,
                  uint32_t *out_ids, int32_t *out_count, int64_t *out_ncand,
                  int64_t *out_popped, cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    switch (engine) {
        case BPQ_ENGINE_BASELINE:
            return dispatch_m<BPQ_ENGINE_BASELINE>(ix, queries, q0, nq, budget, k, ws, out_dist, out_ids, out_count, out_ncand, out_popped, stream);
        case BPQ_ENGINE_FBPQ:
            return dispatch_m<BPQ_ENGINE_FBPQ>(ix, queries, q0, nq, budget, k, ws, out_dist, out_ids, out_count, out_ncand, out_popped, stream);
        case BPQ_ENGINE_HBPQ:
            return dispatch_m<BPQ_ENGINE_HBPQ>(ix, queries, q0, nq, budget, k, ws, out_dist, out_ids, out_count, out_ncand, out_popped, stream);
    }
    return fail(BPQ_ERR_INVALID, "unknown engine");
}

size_t traverse_stage_ws_bytes(int64_t t, int64_t budget, int64_t total) {
    return trav_layout(t, budget, total).total;
}

int launch_traverse_stage(const double *sr1, const double *sr2, const int32_t *o1,
                          const int32_t *o2, const int64_t *offsets, int64_t t, int64_t budget,
                          int64_t total, int32_t *vis_i, int32_t *vis_j, int64_t *starts,
                          int64_t *ends, int64_t *nvis_out, void *ws, size_t ws_bytes,
                          cudaStream_t stream) {
    TravLayout L = trav_layout(t, budget, total);
    BPQ_CHECK(ws_bytes >= L.total, BPQ_ERR_WORKSPACE, "traverse workspace too small");
    char *w = static_cast<char *>(ws);
    unsigned long long *dn = reinterpret_cast<unsigned long long *>(w + L.off_n);
    unsigned int *counter = reinterpret_cast<unsigned int *>(w + L.total - al(4));
    BPQ_CUDA_TRY(cudaMemsetAsync(dn, 0, 8, stream));
    BPQ_CUDA_TRY(cudaMemsetAsync(counter, 0, 4, stream));
    if (total == 0) {
        BPQ_CUDA_TRY(cudaMemsetAsync(nvis_out, 0, 8, stream));
        return BPQ_OK;
    }
    Args<double, int64_t> A{};
    A.tab_floats = 4 + kSortBytes / 4;  // the sort arrays live after the (unused) table
    A.sr_smem = t < kSrSmem ? (int)t : kSrSmem;
    A.tkcap = 0;
    A.tk_off = (int)tk_offset(A.tab_floats, A.sr_smem, sizeof(double));
    const size_t smem = dyn_smem_bytes(A.tab_floats, A.sr_smem, sizeof(double), 0);
    int n_cta = 0;
    int rc = configure<ENGINE_TRAVERSE, 2, double, int64_t>(smem, &n_cta);
    if (rc) return rc;
    A.T = (int)t;
    A.loff = offsets;
    A.goff = offsets;
    A.sharded = false;
    A.n_global = (unsigned long long)total;
    A.rho = (double)total / ((double)t * t);
    A.nq = 1;
    A.sr1 = sr1;
    A.sr2 = sr2;
    A.ord1 = o1;
    A.ord2 = o2;
    A.L = budget;
    A.k = 1;
    A.counter = counter;
    A.scratch = w + L.off_scratch;
    A.stride = 0;
    A.tv_key = reinterpret_cast<unsigned long long *>(w + L.off_key);
    A.tv_lin = reinterpret_cast<uint32_t *>(w + L.off_lin);
    A.tv_start = reinterpret_cast<int64_t *>(w + L.off_st);
    A.tv_end = reinterpret_cast<int64_t *>(w + L.off_en);
    A.tv_n = dn;
    search_kernel<ENGINE_TRAVERSE, 2, double, int64_t><<<1, NT, smem, stream>>>(A);
    BPQ_CUDA_TRY(cudaGetLastError());
    // visit order = sort by (key, oi*t+oj): stable sort by lin, then stable by key
    uint32_t *perm0 = reinterpret_cast<uint32_t *>(w + L.off_perm0);
    uint32_t *perm1 = reinterpret_cast<uint32_t *>(w + L.off_perm1);
    unsigned long long *keys2 = reinterpret_cast<unsigned long long *>(w + L.off_keys2);
    uint32_t *lin2 = reinterpret_cast<uint32_t *>(w + L.off_lin2);
    void *cubw = w + L.off_cub;
    size_t cb = L.cub_bytes;
    int cap = (int)L.cap;
    // the sorts run over the full capacity; unused slots are padded to sort last
    // (fill key/lin tails with max so they stay behind the real cells)
    int nb = (cap + 255) / 256;
    pad_tail_kernel<<<nb, 256, 0, stream>>>(A.tv_key, A.tv_lin, dn, cap);
    iota_kernel<<<nb, 256, 0, stream>>>(perm0, cap);
    BPQ_CUDA_TRY(cudaGetLastError());
    // pass 1: sort (lin -> perm) stable
    BPQ_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cubw, cb, A.tv_lin, lin2, perm0, perm1, cap, 0, 32, stream));
    // keys in lin order
    gather_key_kernel<<<nb, 256, 0, stream>>>(A.tv_key, perm1, keys2, dn);
    // pass 2: stable sort by key carrying perm1 -> perm0
    pad_tail_kernel<<<nb, 256, 0, stream>>>(keys2, nullptr, dn, cap);
    BPQ_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cubw, cb, keys2, A.tv_key, perm1, perm0, cap, 0, 64, stream));
    gather_lin_kernel<<<nb, 256, 0, stream>>>(A.tv_lin, perm0, lin2, dn);
    traverse_finish_kernel<<<nb, 256, 0, stream>>>(lin2, A.tv_start, A.tv_end, perm0, dn, t, vis_i, vis_j, starts, ends, nvis_out);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace bpq

// ------------------------------------------------------- C ABI: diagnostics
extern "C" int bpq_debug_set_phase_buffer(unsigned long long *dev_counters) {
    bpq::g_prof_buffer = dev_counters;
#ifdef BPQ_PHASE_PROF
    return 1;
#else
    return 0;
#endif
}

// --------------------------------------------------------------- C ABI: scans
using bpq::fail;

extern "C" int bpq_scan_tables(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                               const int64_t *cand_start, int64_t nvis, int64_t ncand,
                               const uint32_t *ids, const uint8_t *codes, int32_t m, int32_t k,
                               float q_norm, const float *qd1, const float *qd2, const float *cn1,
                               const float *cn2, const float *fold, const float *cross1,
                               const float *cross2, uint32_t *out_ids, float *out_d, void *stream) {
    if (ncand == 0) return BPQ_OK;
    int nb = (int)((ncand + 255) / 256);
    bpq::stage_scan_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(
        BPQ_ENGINE_FBPQ, vis_i, vis_j, starts, cand_start, nvis, ncand, ids, codes, m, k, 0, q_norm,
        qd1, qd2, cn1, cn2, fold, cross1, cross2, nullptr, nullptr, nullptr, out_ids, out_d);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

extern "C" int bpq_scan_global(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                               const int64_t *cand_start, int64_t nvis, int64_t ncand,
                               const uint32_t *ids, const uint8_t *codes, int32_t m, int32_t k,
                               int32_t ds, const float *e1, const float *e2, const float *books,
                               uint32_t *out_ids, float *out_d, void *stream) {
    if (ncand == 0) return BPQ_OK;
    int nb = (int)((ncand + 255) / 256);
    bpq::stage_scan_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(
        BPQ_ENGINE_BASELINE, vis_i, vis_j, starts, cand_start, nvis, ncand, ids, codes, m, k, ds,
        0.f, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, e1, e2, books, out_ids, out_d);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

extern "C" int bpq_scan_local(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                              const int64_t *cand_start, int64_t nvis, int64_t ncand,
                              const uint32_t *ids, const uint8_t *codes, int32_t m, int32_t k,
                              int32_t ds, const float *e1, const float *e2, const float *books1,
                              const float *books2, uint32_t *out_ids, float *out_d, void *stream) {
    if (ncand == 0) return BPQ_OK;
    int nb = (int)((ncand + 255) / 256);
    bpq::stage_scan_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(
        BPQ_ENGINE_HBPQ, vis_i, vis_j, starts, cand_start, nvis, ncand, ids, codes, m, k, ds, 0.f,
        nullptr, nullptr, nullptr, nullptr, nullptr, books1, books2, e1, e2, nullptr, out_ids, out_d);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}
