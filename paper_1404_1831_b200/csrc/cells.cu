// Populated-cell lists of the multi-index cell table (CSR by row, CSC by
// column), built once per index.  The traversal uses them to enumerate a
// band segment in O(populated cells of the line) instead of O(cells), which
// is what makes sparse tables (BASELINE config 1: 9.5K populated of 16.8M
// cells) cheap to traverse.  Each list is ordered by ascending column/row.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "bpq_internal.cuh"

namespace bpq {
namespace {

constexpr int CT = 256;

__global__ void line_count_kernel(const uint32_t *__restrict__ off, int t, int by_col,
                                  uint32_t *__restrict__ cnt) {
    using Red = cub::BlockReduce<uint32_t, CT>;
    __shared__ typename Red::TempStorage tmp;
    const int line = blockIdx.x;
    uint32_t c = 0;
    for (int x = threadIdx.x; x < t; x += CT) {
        const int64_t lin = by_col ? (int64_t)x * t + line : (int64_t)line * t + x;
        c += off[lin + 1] > off[lin] ? 1u : 0u;
    }
    c = Red(tmp).Sum(c);
    if (threadIdx.x == 0) cnt[line] = c;
}

__global__ void line_fill_kernel(const uint32_t *__restrict__ off, int t, int by_col,
                                 const uint32_t *__restrict__ ptr, uint16_t *__restrict__ out) {
    using Scan = cub::BlockScan<uint32_t, CT>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t base;
    const int line = blockIdx.x;
    if (threadIdx.x == 0) base = ptr[line];
    __syncthreads();
    for (int x0 = 0; x0 < t; x0 += CT) {
        const int x = x0 + threadIdx.x;
        uint32_t f = 0;
        if (x < t) {
            const int64_t lin = by_col ? (int64_t)x * t + line : (int64_t)line * t + x;
            f = off[lin + 1] > off[lin] ? 1u : 0u;
        }
        uint32_t ex, tot;
        Scan(tmp).ExclusiveSum(f, ex, tot);
        if (f) out[base + ex] = (uint16_t)x;
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }


// FBPQ point term: pt[e] = sum_p 2 * cross_h[row][p][code_p] for every entry
// e of cell (i, j) (row = i for the first M/2 parts, j for the rest).  It is
// query independent, so the batched scan reads 4 B per entry instead of
// gathering M cross-table values (numba_backend.py:236-240 does the gathers
// per query).  Summed in f64 and rounded once.  One CTA per cell row i with
// cross1[i] staged in shared memory; the row's entries are contiguous and
// are spread over the CTA (a billion-point row holds ~60K entries), each
// thread finding its entry's column by binary search in the row's offsets.
__global__ void point_term_kernel(const uint32_t *__restrict__ off, int t, int m, int k,
                                  const uint8_t *__restrict__ codes, const float *__restrict__ cross1,
                                  const float *__restrict__ cross2, float *__restrict__ pt) {
    extern __shared__ float c1s[];
    const int i = blockIdx.x;
    const int m2 = m / 2;
    for (int x = threadIdx.x; x < m2 * k; x += CT) c1s[x] = cross1[(size_t)i * m2 * k + x];
    __syncthreads();
    const uint32_t *row = off + (size_t)i * t;
    const uint32_t e0 = row[0], e1 = row[t];
    for (uint32_t e = e0 + threadIdx.x; e < e1; e += CT) {
        int lo = 0, hi = t - 1;  // largest j with row[j] <= e (then row[j+1] > e)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(row + mid) <= e) lo = mid; else hi = mid - 1;
        }
        const float *c2 = cross2 + (size_t)lo * m2 * k;
        const uint8_t *c = codes + (size_t)e * m;
        double acc = 0.0;
        for (int p = 0; p < m2; p++) acc += 2.0 * (double)c1s[p * k + c[p]];
        for (int p = 0; p < m2; p++) acc += 2.0 * (double)__ldg(c2 + p * k + c[m2 + p]);
        pt[e] = (float)acc;
    }
}

}  // namespace
}  // namespace bpq

using bpq::fail;

extern "C" size_t bpq_cell_lists_workspace_size(int32_t t) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum<uint32_t *, uint32_t *>(nullptr, b, nullptr, nullptr, t + 1);
    return bpq::al((size_t)(t + 1) * 4) * 2 + bpq::al(b);
}

extern "C" int bpq_build_cell_lists(const uint32_t *offsets, int32_t t, uint32_t *row_ptr,
                                    uint16_t *row_cols, uint32_t *col_ptr, uint16_t *col_rows,
                                    void *workspace, size_t workspace_bytes, void *stream) {
    BPQ_CHECK(t >= 1 && t < 65536, BPQ_ERR_UNSUPPORTED, "num_coarse must be in [1, 65535]");
    BPQ_CHECK(workspace_bytes >= bpq_cell_lists_workspace_size(t), BPQ_ERR_WORKSPACE,
              "cell-list workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    char *w = static_cast<char *>(workspace);
    uint32_t *rc = reinterpret_cast<uint32_t *>(w);
    uint32_t *cc = reinterpret_cast<uint32_t *>(w + bpq::al((size_t)(t + 1) * 4));
    void *cub_tmp = w + 2 * bpq::al((size_t)(t + 1) * 4);
    size_t cb = workspace_bytes - 2 * bpq::al((size_t)(t + 1) * 4);
    BPQ_CUDA_TRY(cudaMemsetAsync(rc, 0, (size_t)(t + 1) * 4, s));
    BPQ_CUDA_TRY(cudaMemsetAsync(cc, 0, (size_t)(t + 1) * 4, s));
    bpq::line_count_kernel<<<t, bpq::CT, 0, s>>>(offsets, t, 0, rc);
    bpq::line_count_kernel<<<t, bpq::CT, 0, s>>>(offsets, t, 1, cc);
    BPQ_CUDA_TRY(cudaGetLastError());
    BPQ_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, rc, row_ptr, t + 1, s));
    BPQ_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, cc, col_ptr, t + 1, s));
    bpq::line_fill_kernel<<<t, bpq::CT, 0, s>>>(offsets, t, 0, row_ptr, row_cols);
    bpq::line_fill_kernel<<<t, bpq::CT, 0, s>>>(offsets, t, 1, col_ptr, col_rows);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

namespace bpq {
// codes_rot[e] = entry e's M code bytes rotated by e % M: byte i holds part
// (e % M + i) % M (the order the point-term scans read them in, search_impl.cuh
// LaneLut), so the scans skip the per-entry byte rotation
__global__ void rotate_codes_kernel(const uint8_t *__restrict__ codes, int64_t n, int m, uint8_t *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int x = (int)(e % m);
    const uint8_t *src = codes + e * m;
    uint8_t *dst = out + e * m;
    for (int i = 0; i < m; i++) dst[i] = src[(x + i) % m];
}

int launch_rotate_codes(const uint8_t *codes, int64_t n, int32_t m, uint8_t *out, cudaStream_t s) {
    if (n <= 0) return BPQ_OK;
    rotate_codes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(codes, n, m, out);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

// Query-split sharding: the visited cells of every query (all ranks'
// traversals, packed by query) -> this shard's non-empty local cells
// (start, count, cell_base) at the same packed positions, per-query counts
// and local candidate counts, and the query list of the stream kernel.
// One warp per query.
__global__ void visits_to_cells_kernel(const int4 *__restrict__ visits, const uint32_t *__restrict__ vstart,
                                       int64_t nq, const uint32_t *__restrict__ loff, int4 *__restrict__ cells,
                                       uint32_t *__restrict__ cell_n, unsigned long long *__restrict__ ncand,
                                       uint32_t *__restrict__ tk_n, unsigned int *__restrict__ qlist,
                                       unsigned int *__restrict__ qcount) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    const uint32_t s = vstart[q], e = vstart[q + 1];
    uint32_t n = 0;
    unsigned long long cand = 0;
    for (uint32_t i0 = s; i0 < e; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool ok = false;
        uint32_t l0 = 0, l1 = 0;
        int4 v = make_int4(0, 0, 0, 0);
        if (i < e) {
            v = visits[i];
            const uint32_t lin = (uint32_t)v.x;
            l0 = __ldg(loff + lin);
            l1 = __ldg(loff + lin + 1);
            ok = l1 > l0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            cells[s + n + __popc(bal & ((1u << lane) - 1u))] = make_int4((int)l0, (int)(l1 - l0), v.z, 0);
            cand += l1 - l0;
        }
        n += __popc(bal);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
    if (lane == 0) {
        cell_n[q] = n;
        ncand[q] = cand;
        tk_n[q] = 0;
        qlist[q] = (unsigned int)q;
        if (q == 0) *qcount = (unsigned int)nq;
    }
}

int launch_visits_to_cells(const int4 *visits, const uint32_t *visit_start, int64_t nq, const uint32_t *loff,
                           int4 *cells, uint32_t *cell_n, unsigned long long *ncand, uint32_t *tk_n,
                           unsigned int *qlist, unsigned int *qcount, cudaStream_t st) {
    if (nq <= 0) return BPQ_OK;
    const int64_t threads = nq * 32;
    visits_to_cells_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(visits, visit_start, nq, loff, cells,
                                                                             cell_n, ncand, tk_n, qlist, qcount);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

int launch_point_term(const uint32_t *offsets, int32_t t, int32_t m, int32_t k, const uint8_t *codes,
                      const float *cross1, const float *cross2, float *pt, cudaStream_t s) {
    const size_t smem = (size_t)(m / 2) * k * sizeof(float);
    point_term_kernel<<<t, CT, smem, s>>>(offsets, t, m, k, codes, cross1, cross2, pt);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}
}  // namespace bpq
