// C ABI: index lifecycle, batched search orchestration, traversal stage.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include <mutex>

#include "bpq_internal.cuh"

namespace bpq {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

namespace {

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct SearchLayout {
    int64_t chunk;
    size_t dots1, dots2, sr1, sr2, ord1, ord2, pos1, pos2, fold, ru1, ru2, retry, plen, qrot, counter, cta, cta_stride, total;
    size_t big, big_n, tk_n, tk_part, ncand_q, bigq;
    int64_t big_cap;  // 0: no large-cell stream
    int n_cta;
};

// large cells (>= lut_min entries) a query can visit: all but the cutoff cell lie inside the budget
// Side stream for the FBPQ fold (non-blocking, one per process and device; BPQ_FOLD_INLINE=1 keeps the fold
// on the caller's stream).  Work from concurrent searches serialises on it, ordered by per-call events.
cudaStream_t fold_side_stream() {
    static std::mutex mu;
    static cudaStream_t st = nullptr;
    static int st_dev = -1;
    static const bool inline_fold = getenv("BPQ_FOLD_INLINE") != nullptr;
    if (inline_fold) return nullptr;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lock(mu);
    if (st == nullptr) {
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            st = nullptr;
            return nullptr;
        }
        st_dev = dev;
    }
    return dev == st_dev ? st : nullptr;
}

int64_t big_cells_cap(const Index &ix, int64_t budget) {
    // the stream kernel moves codes by TMA bulk copies: 16-byte aligned code array
    if (!(ix.pterm != nullptr && ix.codes_rot != nullptr && (ix.M == 8 || ix.M == 16)) ||
        (reinterpret_cast<uintptr_t>(ix.codes_rot) & 15))
        return 0;
    return budget / std::max(effective_lut_min(), 1) + 2;
}

int64_t query_chunk(int64_t nq, int32_t T, int32_t M, int32_t K, int64_t big_cap, int32_t k) {
    // keep the per-chunk first-layer buffers (10 arrays of [chunk, T] x 4 B + fold), and the
    // deferred large-cell lists, near 8 GiB
    int64_t per_q = (int64_t)T * 40 + (int64_t)M * K * 4 + 4 + (big_cap ? big_cap * 16 + (int64_t)k * 8 + 32 : 0);
    int64_t c = ((int64_t)8 << 30) / per_q;
    c = std::max<int64_t>(c, 256);
    return std::max<int64_t>(1, std::min<int64_t>(nq, c));
}

bool layout_for(const Index &ix, int64_t nq, int64_t budget, int32_t k, SearchLayout *L) {
    SearchLayout s{};
    s.big_cap = big_cells_cap(ix, budget);
    s.chunk = query_chunk(nq, ix.T, ix.M, ix.K, s.big_cap, k);
    int n_cta = search_grid_ctas(BPQ_ENGINE_FBPQ, ix.M);
    if (n_cta <= 0) return false;
    s.n_cta = n_cta;
    size_t row = (size_t)s.chunk * ix.T * 4;
    size_t o = 0;
    s.dots1 = o; o += al(row);
    s.dots2 = o; o += al(row);
    s.sr1 = o; o += al(row);
    s.sr2 = o; o += al(row);
    s.ord1 = o; o += al(row);
    s.ord2 = o; o += al(row);
    s.pos1 = o; o += al(row);
    s.pos2 = o; o += al(row);
    s.fold = o; o += al((size_t)s.chunk * ix.M * ix.K * 4);
    s.ru1 = o; o += al(row);
    s.ru2 = o; o += al(row);
    s.retry = o; o += al((size_t)s.chunk * 4 + 4);
    s.plen = o; o += al((size_t)s.chunk * 8);
    s.qrot = o; o += ix.rot ? al((size_t)s.chunk * ix.D * 4) : 0;
    s.counter = o; o += al(4);
    if (s.big_cap) {
        s.big = o; o += al((size_t)s.chunk * s.big_cap * 16);
        s.big_n = o; o += al((size_t)s.chunk * 4);
        s.tk_n = o; o += al((size_t)s.chunk * 4);
        s.tk_part = o; o += al((size_t)s.chunk * k * 8);
        s.ncand_q = o; o += al((size_t)s.chunk * 8);
        s.bigq = o; o += al((size_t)s.chunk * 4 + 4);
    }
    s.cta_stride = al(search_cta_scratch_bytes(ix.T, ix.D));
    s.cta = o; o += s.cta_stride * n_cta;
    s.total = o;
    *L = s;
    return true;
}

template <typename T>
int copy_in(const T *host, size_t count, std::vector<void *> &owned, const T **dst) {
    if (host == nullptr) {
        *dst = nullptr;
        return BPQ_OK;
    }
    void *p = nullptr;
    BPQ_CUDA_TRY(cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 1)));
    owned.push_back(p);
    BPQ_CUDA_TRY(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
    *dst = static_cast<const T *>(p);
    return BPQ_OK;
}

}  // namespace
}  // namespace bpq

using namespace bpq;

extern "C" const char *bpq_last_error(void) { return g_last_error.c_str(); }

extern "C" int bpq_abi_version(void) { return BPQ_ABI_VERSION; }

extern "C" int bpq_index_create(const bpq_index_desc *d, int copy_from_host, bpq_index **out) {
    BPQ_CHECK(d != nullptr && out != nullptr, BPQ_ERR_INVALID, "null descriptor");
    // parameter rules of multi_index._check_fine_params (multi_index.py:199-207)
    BPQ_CHECK(d->num_parts >= 2 && d->num_parts % 2 == 0, BPQ_ERR_INVALID,
              "number of parts must be even and >= 2");
    BPQ_CHECK(d->num_parts <= 16, BPQ_ERR_INVALID, "number of parts must be <= 16");
    BPQ_CHECK(d->dim > 0 && d->dim % d->num_parts == 0 && d->dim % 2 == 0, BPQ_ERR_INVALID,
              "dimension is not divisible into parts");
    BPQ_CHECK(d->codebook_size >= 1 && d->codebook_size <= 256, BPQ_ERR_INVALID,
              "codebook size must be in [1, 256]");
    BPQ_CHECK(d->num_coarse >= 1 && d->num_coarse < 65536, BPQ_ERR_UNSUPPORTED,
              "num_coarse must be in [1, 65535]");
    BPQ_CHECK(d->num_coarse <= 16384, BPQ_ERR_UNSUPPORTED,
              "num_coarse > 16384 exceeds the row-sort kernel");
    BPQ_CHECK(d->dim <= kMaxDim, BPQ_ERR_UNSUPPORTED, "dim > 1024 exceeds the search kernel");
    BPQ_CHECK(d->num_entries >= 0 && d->num_entries <= 0xFFFFFFFFll, BPQ_ERR_UNSUPPORTED,
              "entries must fit uint32 offsets");
    BPQ_CHECK((d->row_ptr == nullptr) == (d->col_ptr == nullptr) &&
                  (d->row_ptr == nullptr) == (d->row_cols == nullptr) &&
                  (d->row_ptr == nullptr) == (d->col_rows == nullptr),
              BPQ_ERR_INVALID, "cell lists must be given all together or not at all");
    BPQ_CHECK(d->num_entries_global >= d->num_entries && d->num_entries_global <= 0xFFFFFFFFll,
              BPQ_ERR_INVALID, "global entry count must be >= local and fit uint32");
    BPQ_CHECK(d->coarse1 && d->coarse2 && d->coarse_norms1 && d->coarse_norms2 && d->cell_offsets &&
                  ((d->ids && d->codes) || d->num_entries == 0),
              BPQ_ERR_INVALID, "coarse books, norms, offsets, ids and codes are required");
    bpq_index *h = new bpq_index();
    Index &ix = h->ix;
    ix.D = d->dim;
    ix.T = d->num_coarse;
    ix.M = d->num_parts;
    ix.K = d->codebook_size;
    ix.dh = d->dim / 2;
    ix.ds = d->dim / d->num_parts;
    ix.N = d->num_entries;
    ix.N_global = d->num_entries_global;
    const size_t T = ix.T, D = ix.D, M = ix.M, K = ix.K, N = ix.N, dh = ix.dh, ds = ix.ds;
    if (!copy_from_host) {
        ix.c1 = d->coarse1;
        ix.c2 = d->coarse2;
        ix.cn1 = d->coarse_norms1;
        ix.cn2 = d->coarse_norms2;
        ix.loff = d->cell_offsets;
        ix.goff = d->global_offsets ? d->global_offsets : d->cell_offsets;
        ix.ids = d->ids;
        ix.codes = d->codes;
        ix.books = d->fine_books;
        ix.fine_norms = d->fine_norms;
        ix.cross1 = d->cross1;
        ix.cross2 = d->cross2;
        ix.bank1 = d->bank1;
        ix.bank2 = d->bank2;
        ix.rowptr = d->row_ptr;
        ix.populated = 0;
        if (d->row_ptr) {
            uint32_t pc = 0;
            if (cudaMemcpy(&pc, d->row_ptr + T, 4, cudaMemcpyDeviceToHost) == cudaSuccess) ix.populated = pc;
            else cudaGetLastError();
        }
        ix.rowcols = d->row_cols;
        ix.colptr = d->col_ptr;
        ix.colrows = d->col_rows;
        ix.rot = d->rotation;
        ix.rot1 = d->rot1;
        ix.rot2 = d->rot2;
    } else {
        int rc = 0;
        rc |= copy_in(d->coarse1, T * dh, ix.owned, &ix.c1);
        rc |= copy_in(d->coarse2, T * dh, ix.owned, &ix.c2);
        rc |= copy_in(d->coarse_norms1, T, ix.owned, &ix.cn1);
        rc |= copy_in(d->coarse_norms2, T, ix.owned, &ix.cn2);
        rc |= copy_in(d->cell_offsets, T * T + 1, ix.owned, &ix.loff);
        if (d->global_offsets)
            rc |= copy_in(d->global_offsets, T * T + 1, ix.owned, &ix.goff);
        else
            ix.goff = ix.loff;
        rc |= copy_in(d->ids, N, ix.owned, &ix.ids);
        rc |= copy_in(d->codes, N * M, ix.owned, &ix.codes);
        rc |= copy_in(d->fine_books, M * K * ds, ix.owned, &ix.books);
        rc |= copy_in(d->fine_norms, M * K, ix.owned, &ix.fine_norms);
        rc |= copy_in(d->cross1, T * (M / 2) * K, ix.owned, &ix.cross1);
        rc |= copy_in(d->cross2, T * (M / 2) * K, ix.owned, &ix.cross2);
        rc |= copy_in(d->bank1, T * (M / 2) * K * ds, ix.owned, &ix.bank1);
        rc |= copy_in(d->bank2, T * (M / 2) * K * ds, ix.owned, &ix.bank2);
        rc |= copy_in(d->rotation, D * D, ix.owned, &ix.rot);
        rc |= copy_in(d->rot1, dh * dh, ix.owned, &ix.rot1);
        rc |= copy_in(d->rot2, dh * dh, ix.owned, &ix.rot2);
        ix.rowptr = ix.colptr = nullptr;
        ix.rowcols = ix.colrows = nullptr;
        if (d->row_ptr && d->col_ptr && d->row_cols && d->col_rows) {
            // the lists describe the traversal table (global_offsets when
            // sharded): size them by its populated count, row_ptr[T]
            const size_t P = std::max<size_t>(d->row_ptr[T], 1);
            ix.populated = (int64_t)d->row_ptr[T];
            rc |= copy_in(d->row_ptr, T + 1, ix.owned, &ix.rowptr);
            rc |= copy_in(d->col_ptr, T + 1, ix.owned, &ix.colptr);
            rc |= copy_in(d->row_cols, P, ix.owned, &ix.rowcols);
            rc |= copy_in(d->col_rows, P, ix.owned, &ix.colrows);
        }
        if (rc) {
            std::string msg = g_last_error;
            bpq_index_destroy(h);
            return fail(BPQ_ERR_CUDA, msg);
        }
    }
    // tensor-core first layer (D = 128): pre-swizzled bf16 limbs of the coarse books
    ix.cimg1 = ix.cimg2 = nullptr;
    {
        const char *fl = getenv("BPQ_FIRST_LAYER");  // "ffma": A/B diagnostics (read per index)
        if (ix.dh == 64 && ix.T > 0 && !(fl && std::string(fl) == "ffma")) {
            const size_t nb = coarse_limb_image_bytes(ix.T);
            void *i1 = nullptr, *i2 = nullptr;
            int rc = BPQ_OK;
            if (cudaMalloc(&i1, nb) != cudaSuccess || cudaMalloc(&i2, nb) != cudaSuccess) {
                cudaGetLastError();
                rc = fail(BPQ_ERR_CUDA, "cannot allocate the coarse limb images");
            }
            if (i1) ix.owned.push_back(i1);
            if (i2) ix.owned.push_back(i2);
            if (rc == BPQ_OK && cudaDeviceSynchronize() != cudaSuccess)
                rc = fail(BPQ_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
            if (rc == BPQ_OK) rc = launch_coarse_limb_image(ix.c1, ix.T, static_cast<uint8_t *>(i1), 0);
            if (rc == BPQ_OK) rc = launch_coarse_limb_image(ix.c2, ix.T, static_cast<uint8_t *>(i2), 0);
            if (rc == BPQ_OK && cudaDeviceSynchronize() != cudaSuccess)
                rc = fail(BPQ_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
            if (rc) {
                std::string msg = g_last_error;
                bpq_index_destroy(h);
                return fail(BPQ_ERR_CUDA, msg);
            }
            ix.cimg1 = static_cast<uint8_t *>(i1);
            ix.cimg2 = static_cast<uint8_t *>(i2);
        }
    }
    ix.pterm = nullptr;
    ix.codes_rot = nullptr;
    ix.exact = d->fbpq_exact != 0;
    if (ix.cross1 && ix.cross2 && ix.codes && N > 0 && !d->fbpq_exact) {
        float *pt = nullptr;
        // kStreamPad entries of slack: the stream kernels read whole 32-aligned chunks (masked)
        if (cudaMalloc(&pt, (N + kStreamPad) * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            bpq_index_destroy(h);
            return fail(BPQ_ERR_CUDA, "cannot allocate the FBPQ point-term array");
        }
        ix.owned.push_back(pt);
        // device mode borrows caller buffers that may still be in flight on
        // any (possibly non-blocking) stream: drain the device first
        int rc = cudaDeviceSynchronize() == cudaSuccess
                     ? BPQ_OK
                     : fail(BPQ_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
        if (rc == BPQ_OK) rc = launch_point_term(ix.loff, ix.T, ix.M, ix.K, ix.codes, ix.cross1, ix.cross2, pt, 0);
        if (rc == BPQ_OK && cudaDeviceSynchronize() != cudaSuccess)
            rc = fail(BPQ_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
        if (rc) {
            std::string msg = g_last_error;
            bpq_index_destroy(h);
            return fail(BPQ_ERR_CUDA, msg);
        }
        ix.pterm = pt;
        if (ix.M == 8 || ix.M == 16) {
            // the point-term scans read the codes pre-rotated (cells.cu rotate_codes_kernel)
            void *cr = nullptr;
            if (cudaMalloc(&cr, (size_t)(N + kStreamPad) * M) != cudaSuccess) {
                cudaGetLastError();
                bpq_index_destroy(h);
                return fail(BPQ_ERR_CUDA, "cannot allocate the rotated code array");
            }
            ix.owned.push_back(cr);
            int rc = launch_rotate_codes(ix.codes, N, ix.M, static_cast<uint8_t *>(cr), 0);
            if (rc == BPQ_OK && cudaDeviceSynchronize() != cudaSuccess)
                rc = fail(BPQ_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
            if (rc) {
                std::string msg = g_last_error;
                bpq_index_destroy(h);
                return fail(BPQ_ERR_CUDA, msg);
            }
            ix.codes_rot = static_cast<uint8_t *>(cr);
        }
    }
    *out = h;
    return BPQ_OK;
}

extern "C" int bpq_index_destroy(bpq_index *index) {
    if (!index) return BPQ_OK;
    for (void *p : index->ix.owned) cudaFree(p);
    delete index;
    return BPQ_OK;
}

extern "C" size_t bpq_search_workspace_size(const bpq_index *index, int engine, int64_t nq,
                                            int64_t budget, int32_t k) {
    (void)engine;
    (void)budget;
    (void)k;
    if (!index) return 0;
    SearchLayout L;
    if (!layout_for(index->ix, std::max<int64_t>(nq, 1), std::max<int64_t>(budget, 1), std::max<int32_t>(k, 1), &L))
        return 0;
    return L.total;
}

extern "C" int bpq_search(const bpq_index *index, int engine, const float *queries, int64_t nq,
                          int64_t budget, int32_t k, float *out_dist, uint32_t *out_ids,
                          int32_t *out_count, int64_t *out_ncand, void *workspace,
                          size_t workspace_bytes, void *stream) {
    return bpq_search_ex(index, engine, queries, nq, budget, k, out_dist, out_ids, out_count,
                         out_ncand, nullptr, nullptr, workspace, workspace_bytes, stream);
}

namespace {
// The batched search; with rec != nullptr (query-split traversal) every visited non-empty cell is
// recorded into rec [nq][rec_cap] (counts rec_n) instead of scanned, and no top-k is produced.
int search_impl(const bpq_index *index, int engine, const float *queries, int64_t nq, int64_t budget, int32_t k,
                float *out_dist, uint32_t *out_ids, int32_t *out_count, int64_t *out_ncand, int64_t *out_popped,
                void *const *stage_events, void *workspace, size_t workspace_bytes, void *stream, int4 *rec,
                uint32_t *rec_n, int64_t rec_cap) {
    BPQ_CHECK(index != nullptr, BPQ_ERR_INVALID, "null index");
    const Index &ix = index->ix;
    // traverse() rejects budget < 1 (multi_index.py:308-309); search_* reject r < 1
    BPQ_CHECK(budget >= 1, BPQ_ERR_INVALID, "budget must be >= 1");
    BPQ_CHECK(k >= 1, BPQ_ERR_INVALID, "r must be >= 1");
    BPQ_CHECK(k <= kMaxK, BPQ_ERR_UNSUPPORTED, "k exceeds the engine's top-k buffer (1024)");
    BPQ_CHECK(nq >= 0, BPQ_ERR_INVALID, "nq must be >= 0");
    switch (engine) {
        case BPQ_ENGINE_BASELINE:
            BPQ_CHECK(ix.books, BPQ_ERR_INVALID, "engine baseline requires global fine codebooks");
            break;
        case BPQ_ENGINE_FBPQ:
            BPQ_CHECK(ix.books && ix.fine_norms && ix.cross1 && ix.cross2, BPQ_ERR_INVALID,
                      "engine fbpq requires fine codebooks and FBPQ tables");
            break;
        case BPQ_ENGINE_HBPQ:
            BPQ_CHECK(ix.bank1 && ix.bank2, BPQ_ERR_INVALID,
                      "engine hbpq requires an index built with local codebooks");
            break;
        default:
            return fail(BPQ_ERR_INVALID, "unknown engine");
    }
    if (nq == 0) return BPQ_OK;
    SearchLayout L;
    BPQ_CHECK(layout_for(ix, nq, budget, k, &L), BPQ_ERR_CUDA, "cannot size the search grid");
    BPQ_CHECK(workspace != nullptr && workspace_bytes >= L.total, BPQ_ERR_WORKSPACE,
              "search workspace too small (see bpq_search_workspace_size)");
    char *w = static_cast<char *>(workspace);
    SearchWorkspace ws{};
    ws.dots1 = reinterpret_cast<float *>(w + L.dots1);
    ws.dots2 = reinterpret_cast<float *>(w + L.dots2);
    ws.sr1 = reinterpret_cast<float *>(w + L.sr1);
    ws.sr2 = reinterpret_cast<float *>(w + L.sr2);
    ws.ord1 = reinterpret_cast<int32_t *>(w + L.ord1);
    ws.ord2 = reinterpret_cast<int32_t *>(w + L.ord2);
    ws.pos1 = reinterpret_cast<int32_t *>(w + L.pos1);
    ws.pos2 = reinterpret_cast<int32_t *>(w + L.pos2);
    ws.fold = reinterpret_cast<float *>(w + L.fold);
    ws.ru1 = reinterpret_cast<float *>(w + L.ru1);
    ws.ru2 = reinterpret_cast<float *>(w + L.ru2);
    ws.retry_count = reinterpret_cast<unsigned int *>(w + L.retry);
    ws.retry_list = ws.retry_count + 1;
    ws.plen = reinterpret_cast<int32_t *>(w + L.plen);
    ws.qrot = ix.rot ? reinterpret_cast<float *>(w + L.qrot) : nullptr;
    ws.qlist = nullptr;
    ws.qlist_count = nullptr;
    ws.counter = reinterpret_cast<unsigned int *>(w + L.counter);
    ws.big_cells = nullptr;
    ws.big_cap = 0;
    ws.big_start = nullptr;
    ws.record = nullptr;
    ws.record_n = nullptr;
    ws.record_cap = 0;
    if (L.big_cap && rec == nullptr) {
        ws.big_cells = reinterpret_cast<int4 *>(w + L.big);
        ws.big_cap = (int)L.big_cap;
        ws.big_n = reinterpret_cast<uint32_t *>(w + L.big_n);
        ws.tk_n = reinterpret_cast<uint32_t *>(w + L.tk_n);
        ws.tk_part = reinterpret_cast<unsigned long long *>(w + L.tk_part);
        ws.ncand_q = reinterpret_cast<unsigned long long *>(w + L.ncand_q);
        ws.bigq_count = reinterpret_cast<unsigned int *>(w + L.bigq);
        ws.bigq_list = ws.bigq_count + 1;
    }
    ws.cta_scratch = w + L.cta;
    ws.cta_stride = L.cta_stride;
    ws.n_cta = L.n_cta;
    cudaStream_t s = (cudaStream_t)stream;
    const bool ev = stage_events != nullptr && L.chunk >= nq;
    if (ev) BPQ_CUDA_TRY(cudaEventRecord((cudaEvent_t)stage_events[0], s));
    for (int64_t q0 = 0; q0 < nq; q0 += L.chunk) {
        int64_t n = std::min<int64_t>(L.chunk, nq - q0);
        if (rec != nullptr) {
            ws.record = rec + q0 * rec_cap;
            ws.record_n = rec_n + q0;
            ws.record_cap = (int)rec_cap;
        }
        const float *qc = queries + q0 * ix.D;
        if (ix.rot) {  // queries into the index's rotated space (CoarsePair.rotate_in)
            int rr = launch_rotate(qc, n, ix.D, ix.rot, ws.qrot, s);
            if (rr) return rr;
            qc = ws.qrot;
        }
        // The FBPQ fold depends on the queries only: it runs on a side stream under the first layer and
        // the row sort (the tensor-core first layer leaves most of every SM idle), ordered by two events:
        // after everything already queued on s (the last batch's readers of ws.fold), before the search.
        cudaEvent_t fold_done = nullptr;
        if (engine == BPQ_ENGINE_FBPQ) {
            cudaStream_t fs = fold_side_stream();
            cudaEvent_t q_ready = nullptr;
            if (fs != nullptr && cudaEventCreateWithFlags(&q_ready, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&fold_done, cudaEventDisableTiming) == cudaSuccess) {
                BPQ_CUDA_TRY(cudaEventRecord(q_ready, s));
                BPQ_CUDA_TRY(cudaStreamWaitEvent(fs, q_ready, 0));
                int rf = launch_fold(qc, n, ix.D, ix.M, ix.K, ix.books, ix.fine_norms, ws.fold, fs);
                if (rf) return rf;
                BPQ_CUDA_TRY(cudaEventRecord(fold_done, fs));
                cudaEventDestroy(q_ready);  // (released once the recorded work completes)
            } else {
                cudaGetLastError();
                if (q_ready) cudaEventDestroy(q_ready);
                fold_done = nullptr;
            }
        }
        int rc = ix.cimg1 ? launch_coarse_dots_tc(qc, n, ix.D, ix.cimg1, ix.cimg2, ix.T, ws.dots1, ws.dots2, s)
                          : launch_coarse_dots(qc, n, ix.D, ix.c1, ix.c2, ix.T, ws.dots1, ws.dots2, s);
        if (rc) return rc;
        if (ev) BPQ_CUDA_TRY(cudaEventRecord((cudaEvent_t)stage_events[1], s));
        // sparse tables only need the activated lines' sorted prefix: partial
        // sort first, full sort only for queries that outgrow it (retry pass)
        const bool sparse = ix.rowptr != nullptr;
        static const bool force_full = getenv("BPQ_FORCE_FULL_SORT") != nullptr;  // diagnostics
        const bool partial = sparse && ix.T > kTopP && out_popped == nullptr && !force_full;
        if (partial) {
            rc = launch_row_topk(qc, n, ix.D, ws.dots1, ws.dots2, ix.cn1, ix.cn2, ix.T, ws.sr1, ws.sr2,
                                 ws.ord1, ws.ord2, ws.ru1, ws.ru2, ws.plen, s);
        } else {
            rc = launch_row_sort(qc, n, ix.D, ws.dots1, ws.dots2, ix.cn1, ix.cn2, ix.T, ws.sr1, ws.sr2,
                                 ws.ord1, ws.ord2, ws.pos1, ws.pos2, sparse ? ws.ru1 : nullptr,
                                 sparse ? ws.ru2 : nullptr, nullptr, nullptr, s);
        }
        if (rc) return rc;
        ws.topP = partial ? kTopP : ix.T;
        BPQ_CUDA_TRY(cudaMemsetAsync(ws.retry_count, 0, 4, s));
        if (ws.big_cells) BPQ_CUDA_TRY(cudaMemsetAsync(ws.bigq_count, 0, 4, s));
        if (engine == BPQ_ENGINE_FBPQ) {
            if (fold_done != nullptr) {
                BPQ_CUDA_TRY(cudaStreamWaitEvent(s, fold_done, 0));
                cudaEventDestroy(fold_done);
            } else {
                rc = launch_fold(qc, n, ix.D, ix.M, ix.K, ix.books, ix.fine_norms, ws.fold, s);
                if (rc) return rc;
            }
        }
        if (ev) BPQ_CUDA_TRY(cudaEventRecord((cudaEvent_t)stage_events[2], s));
        rc = launch_search(ix, engine, qc, q0, n, budget, k, ws, out_dist, out_ids, out_count,
                           out_ncand, out_popped, s);
        if (rc) return rc;
        if (partial) {
            // retry pass: full sort + search for the queued queries (device-side list)
            rc = launch_row_sort(qc, n, ix.D, ws.dots1, ws.dots2, ix.cn1, ix.cn2, ix.T, ws.sr1, ws.sr2,
                                 ws.ord1, ws.ord2, ws.pos1, ws.pos2, ws.ru1, ws.ru2, ws.retry_list,
                                 ws.retry_count, s);
            if (rc) return rc;
            SearchWorkspace w2 = ws;
            w2.topP = ix.T;
            w2.qlist = ws.retry_list;
            w2.qlist_count = ws.retry_count;
            w2.retry_list = nullptr;
            w2.retry_count = nullptr;
            rc = launch_search(ix, engine, qc, q0, n, budget, k, w2, out_dist, out_ids, out_count,
                               out_ncand, out_popped, s);
            if (rc) return rc;
        }
        if (ev) BPQ_CUDA_TRY(cudaEventRecord((cudaEvent_t)stage_events[3], s));
        // the large cells of every query the traversal passes handed over
        rc = launch_big_scan(ix, engine, qc, q0, n, budget, k, ws, out_dist, out_ids, out_count, s);
        if (rc) return rc;
        if (ev) BPQ_CUDA_TRY(cudaEventRecord((cudaEvent_t)stage_events[4], s));
    }
    return BPQ_OK;
}
}  // namespace

extern "C" int bpq_search_ex(const bpq_index *index, int engine, const float *queries, int64_t nq,
                             int64_t budget, int32_t k, float *out_dist, uint32_t *out_ids,
                             int32_t *out_count, int64_t *out_ncand, int64_t *out_popped,
                             void *const *stage_events, void *workspace, size_t workspace_bytes,
                             void *stream) {
    return search_impl(index, engine, queries, nq, budget, k, out_dist, out_ids, out_count, out_ncand, out_popped,
                       stage_events, workspace, workspace_bytes, stream, nullptr, nullptr, 0);
}

extern "C" int64_t bpq_split_visit_cap(const bpq_index *index, int64_t budget) {
    if (!index || budget < 1) return 0;
    const Index &ix = index->ix;
    // every visited non-empty cell but the cutoff one lies inside the budget (>= 1 entry each)
    int64_t cap = budget;
    if (ix.populated > 0) cap = std::min<int64_t>(cap, ix.populated);
    cap = std::min<int64_t>(cap, (int64_t)ix.T * ix.T);
    return std::max<int64_t>(cap, 1);
}

extern "C" int bpq_search_split_traverse(const bpq_index *index, const float *queries, int64_t nq, int64_t budget,
                                         uint32_t *visit_count, void *visits, int64_t cap, int64_t *out_ncand,
                                         void *workspace, size_t workspace_bytes, void *stream) {
    BPQ_CHECK(index != nullptr && visits != nullptr && visit_count != nullptr, BPQ_ERR_INVALID, "null argument");
    BPQ_CHECK(cap >= bpq_split_visit_cap(index, budget), BPQ_ERR_INVALID, "visit capacity below bpq_split_visit_cap");
    // k only sizes buffers that record mode does not use
    return search_impl(index, BPQ_ENGINE_FBPQ, queries, nq, budget, 1, nullptr, nullptr, nullptr, out_ncand, nullptr,
                       nullptr, workspace, workspace_bytes, stream, static_cast<int4 *>(visits), visit_count, cap);
}

extern "C" size_t bpq_split_scan_workspace_size(const bpq_index *index, int64_t nq, int64_t total_visits) {
    if (!index || nq < 0 || total_visits < 0) return 0;
    const Index &ix = index->ix;
    size_t o = 0;
    o += al((size_t)std::max<int64_t>(nq, 1) * ix.M * ix.K * 4);       // fold
    o += al((size_t)std::max<int64_t>(total_visits, 1) * 16);          // local cells
    o += 3 * al((size_t)std::max<int64_t>(nq, 1) * 4);                 // cell_n, tk_n, qlist
    o += al((size_t)std::max<int64_t>(nq, 1) * 8);                     // ncand
    o += al(8);                                                         // qcount, counter
    o += ix.rot ? al((size_t)std::max<int64_t>(nq, 1) * ix.D * 4) : 0;  // rotated queries
    return o;
}

extern "C" int bpq_search_split_scan(const bpq_index *index, const float *queries, int64_t nq, int32_t k,
                                     const void *visits, const uint32_t *visit_start, int64_t total_visits,
                                     float *out_dist, uint32_t *out_ids, int32_t *out_count, void *workspace,
                                     size_t workspace_bytes, void *stream) {
    BPQ_CHECK(index != nullptr, BPQ_ERR_INVALID, "null index");
    const Index &ix = index->ix;
    BPQ_CHECK(k >= 1 && k <= kMaxK, BPQ_ERR_INVALID, "k must be in [1, 1024]");
    BPQ_CHECK(ix.pterm != nullptr && ix.codes_rot != nullptr && (ix.M == 8 || ix.M == 16), BPQ_ERR_UNSUPPORTED,
              "the split scan streams point-term FBPQ cells (M = 8 or 16, fbpq_exact = 0)");
    BPQ_CHECK(workspace_bytes >= bpq_split_scan_workspace_size(index, nq, total_visits), BPQ_ERR_WORKSPACE,
              "split-scan workspace too small (see bpq_split_scan_workspace_size)");
    if (nq == 0) return BPQ_OK;
    char *w = static_cast<char *>(workspace);
    size_t o = 0;
    float *fold = reinterpret_cast<float *>(w + o); o += al((size_t)nq * ix.M * ix.K * 4);
    int4 *cells = reinterpret_cast<int4 *>(w + o); o += al((size_t)std::max<int64_t>(total_visits, 1) * 16);
    uint32_t *cell_n = reinterpret_cast<uint32_t *>(w + o); o += al((size_t)nq * 4);
    uint32_t *tk_n = reinterpret_cast<uint32_t *>(w + o); o += al((size_t)nq * 4);
    unsigned int *qlist = reinterpret_cast<unsigned int *>(w + o); o += al((size_t)nq * 4);
    unsigned long long *ncand = reinterpret_cast<unsigned long long *>(w + o); o += al((size_t)nq * 8);
    unsigned int *qcount = reinterpret_cast<unsigned int *>(w + o);
    unsigned int *counter = qcount + 1; o += al(8);
    cudaStream_t s = (cudaStream_t)stream;
    const float *qc = queries;
    if (ix.rot) {
        float *qr = reinterpret_cast<float *>(w + o);
        int rr = launch_rotate(queries, nq, ix.D, ix.rot, qr, s);
        if (rr) return rr;
        qc = qr;
    }
    int rc = launch_fold(qc, nq, ix.D, ix.M, ix.K, ix.books, ix.fine_norms, fold, s);
    if (rc) return rc;
    rc = launch_visits_to_cells(static_cast<const int4 *>(visits), visit_start, nq, ix.loff, cells, cell_n, ncand,
                                tk_n, qlist, qcount, s);
    if (rc) return rc;
    SearchWorkspace ws{};
    ws.fold = fold;
    ws.big_cells = cells;
    ws.big_start = visit_start;
    ws.big_cap = 0;
    ws.big_n = cell_n;
    ws.tk_n = tk_n;
    ws.tk_part = nullptr;
    ws.ncand_q = ncand;
    ws.bigq_list = qlist;
    ws.bigq_count = qcount;
    ws.counter = counter;
    return launch_big_scan(ix, BPQ_ENGINE_FBPQ, qc, 0, nq, 1, k, ws, out_dist, out_ids, out_count, s);
}

extern "C" int bpq_coarse_dots(const bpq_index *index, const float *queries, int64_t nq, float *dots1, float *dots2,
                               void *stream) {
    BPQ_CHECK(index != nullptr, BPQ_ERR_INVALID, "null index");
    BPQ_CHECK(nq >= 0, BPQ_ERR_INVALID, "nq must be >= 0");
    const Index &ix = index->ix;
    cudaStream_t s = (cudaStream_t)stream;
    return ix.cimg1 ? launch_coarse_dots_tc(queries, nq, ix.D, ix.cimg1, ix.cimg2, ix.T, dots1, dots2, s)
                    : launch_coarse_dots(queries, nq, ix.D, ix.c1, ix.c2, ix.T, dots1, dots2, s);
}

extern "C" size_t bpq_traverse_workspace_size(int64_t t, int64_t budget, int64_t total_entries) {
    return traverse_stage_ws_bytes(t, budget, total_entries);
}

extern "C" int bpq_traverse_cells(const double *sorted_r1, const double *sorted_r2,
                                  const int32_t *order1, const int32_t *order2,
                                  const int64_t *offsets, int64_t t, int64_t budget,
                                  int64_t total_entries, int32_t *vis_i, int32_t *vis_j,
                                  int64_t *starts, int64_t *ends, int64_t *nvis_out,
                                  void *workspace, size_t workspace_bytes, void *stream) {
    BPQ_CHECK(budget >= 1, BPQ_ERR_INVALID, "budget must be >= 1");
    BPQ_CHECK(t >= 1 && t < 65536, BPQ_ERR_UNSUPPORTED, "t must be in [1, 65535]");
    BPQ_CHECK(total_entries >= 0 && total_entries <= 0xFFFFFFFFll, BPQ_ERR_UNSUPPORTED,
              "traversal stage handles < 2^32 entries");
    return launch_traverse_stage(sorted_r1, sorted_r2, order1, order2, offsets, t, budget,
                                 total_entries, vis_i, vis_j, starts, ends, nvis_out, workspace,
                                 workspace_bytes, (cudaStream_t)stream);
}
