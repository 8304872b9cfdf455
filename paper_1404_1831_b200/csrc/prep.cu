// First-layer query preparation: query-to-half-codeword distances and the
// per-query stable sort of each half's distances.
//
// Replaces, per query, coarse_scan (multi_index.py:270-293) and the two
// stable argsorts of traverse (multi_index.py:319-322).
//
// Distances are an FFMA (fp32) tiled contraction, not tensor cores: the
// traversal keys r = (|c|^2 - 2 q.c) + |q|^2 cancel heavily (|c|^2, |q|^2 ~
// 2e5 against r ~ 6e4 at config 0), and TF32/BF16 products would reorder
// cells well outside the parity contract.  The work is
// 2*T*D flop per query -- 10.5 GFLOP per 10k-query batch at config 1 --
// under 1% of the batch time even at FFMA rate.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "bpq_internal.cuh"

namespace bpq {

namespace {

constexpr int BQ = 64, BT = 64, BK = 16;

// dots_h[q, t] = sum_x Q[q, h*dh + x] * C_h[t, x]   (h = blockIdx.z)
__global__ void __launch_bounds__(256) coarse_dots_kernel(const float *__restrict__ Q, int64_t nq,
                                                          int D, const float *__restrict__ C1,
                                                          const float *__restrict__ C2, int T,
                                                          float *__restrict__ dots1,
                                                          float *__restrict__ dots2) {
    __shared__ __align__(16) float Qs[BK][BQ + 4];
    __shared__ __align__(16) float Cs[BK][BT + 4];
    const int h = blockIdx.z;
    const int dh = D / 2;
    const float *C = h ? C2 : C1;
    float *out = h ? dots2 : dots1;
    const int64_t q0 = (int64_t)blockIdx.y * BQ;
    const int t0 = blockIdx.x * BT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.f;

    // loader mapping: 256 threads x 4 elements = 64 rows x 16 k
    const int lr = threadIdx.x >> 2;        // row within tile 0..63
    const int lk = (threadIdx.x & 3) * 4;   // k offset 0,4,8,12
    for (int k0 = 0; k0 < dh; k0 += BK) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            int kk = k0 + lk + u;
            int64_t q = q0 + lr;
            int t = t0 + lr;
            Qs[lk + u][lr] = (q < nq && kk < dh) ? __ldg(Q + q * D + h * dh + kk) : 0.f;
            Cs[lk + u][lr] = (t < T && kk < dh) ? __ldg(C + (int64_t)t * dh + kk) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float4 a = *reinterpret_cast<const float4 *>(&Qs[kk][ty * 4]);
            float4 b = *reinterpret_cast<const float4 *>(&Cs[kk][tx * 4]);
            float av[4] = {a.x, a.y, a.z, a.w};
            float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        int64_t q = q0 + ty * 4 + i;
        if (q >= nq) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int t = t0 + tx * 4 + j;
            if (t < T) out[q * T + t] = acc[i][j];
        }
    }
}

// FBPQ query tables for a batch (fbpq.py:140-144): for every query, part p
// and codeword c, fold[q][p][c] = fine_norms[p][c] - 2 * (books[p][c] . q_p).
// One CTA per (32-query tile, part): the part's codebook (K x ds) and the
// query slices are staged in shared memory; thread c owns codeword c.
constexpr int FQ = 32;

__global__ void __launch_bounds__(256) fold_kernel(const float *__restrict__ Q, int64_t nq, int D, int M,
                                                   int K, const float *__restrict__ books,
                                                   const float *__restrict__ fine_norms,
                                                   float *__restrict__ fold) {
    extern __shared__ __align__(16) float fs[];
    const int p = blockIdx.y;
    const int ds = D / M;
    const int64_t q0 = (int64_t)blockIdx.x * FQ;
    float *bk = fs;              // [K][ds+1] (padded: conflict-free column reads)
    float *qs = fs + K * (ds + 1);  // [FQ][ds]
    for (int x = threadIdx.x; x < K * ds; x += blockDim.x) {
        const int c = x / ds, u = x - c * ds;
        bk[c * (ds + 1) + u] = __ldg(books + ((size_t)p * K) * ds + x);
    }
    for (int x = threadIdx.x; x < FQ * ds; x += blockDim.x) {
        const int qq = x / ds, u = x - qq * ds;
        const int64_t q = q0 + qq;
        qs[x] = q < nq ? __ldg(Q + q * D + p * ds + u) : 0.f;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < K; c += blockDim.x) {
        const float fn = __ldg(fine_norms + p * K + c);
        const float *b = bk + c * (ds + 1);
        for (int qq = 0; qq < FQ; qq++) {
            const int64_t q = q0 + qq;
            if (q >= nq) break;
            const float *qv = qs + qq * ds;
            float dot = 0.f;
            for (int u = 0; u < ds; u++) dot = fmaf(b[u], qv[u], dot);
            fold[(q * M + p) * K + c] = __fsub_rn(fn, __fmul_rn(2.f, dot));
        }
    }
}

constexpr int kSortThreads = 512;

// One CTA per (query, half): r = max((cn - 2*dot) + |q_h|^2, 0) then a
// stable LSD radix sort of (bits(r), index) -- equal keys keep ascending
// original index exactly as np.argsort(kind="stable").
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads) row_sort_kernel(
    const float *__restrict__ Q, int D, const float *__restrict__ dots1,
    const float *__restrict__ dots2, const float *__restrict__ cn1,
    const float *__restrict__ cn2, int T, float *__restrict__ sr1, float *__restrict__ sr2,
    int32_t *__restrict__ ord1, int32_t *__restrict__ ord2, int32_t *__restrict__ pos1,
    int32_t *__restrict__ pos2, float *__restrict__ ru1, float *__restrict__ ru2,
    const unsigned int *__restrict__ qlist, const unsigned int *__restrict__ qcount) {
    using Sort = cub::BlockRadixSort<unsigned int, kSortThreads, ITEMS, int>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto &temp = *reinterpret_cast<typename Sort::TempStorage *>(smem_raw);
    __shared__ float s_part[kSortThreads / 32];
    __shared__ float s_qn;

    if (qlist != nullptr && blockIdx.x >= *qcount) return;
    const int64_t q = qlist != nullptr ? (int64_t)qlist[blockIdx.x] : (int64_t)blockIdx.x;
    const int h = blockIdx.y;
    const int dh = D / 2;
    const float *qv = Q + q * D + h * dh;
    // |q_h|^2 (q1 @ q1 in coarse_scan, multi_index.py:287-288)
    float part = 0.f;
    for (int x = threadIdx.x; x < dh; x += kSortThreads) {
        float v = qv[x];
        part = fmaf(v, v, part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int w = 0; w < kSortThreads / 32; w++) s += s_part[w];
        s_qn = s;
    }
    __syncthreads();
    const float qn = s_qn;
    const float *dots = (h ? dots2 : dots1) + q * T;
    const float *cn = h ? cn2 : cn1;

    unsigned int keys[ITEMS];
    int vals[ITEMS];
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        int idx = threadIdx.x * ITEMS + s;  // blocked arrangement = original order
        if (idx < T) {
            float r = __fadd_rn(__fsub_rn(__ldg(cn + idx), __fmul_rn(2.f, __ldg(dots + idx))), qn);
            if (!(r > 0.f)) r = 0.f;  // np.maximum(r, 0) (multi_index.py:291-292)
            keys[s] = __float_as_uint(r);
            if (ru1 != nullptr) (h ? ru2 : ru1)[q * T + idx] = r;
        } else {
            keys[s] = 0xFFFFFFFFu;
        }
        vals[s] = idx;
    }
    Sort(temp).SortBlockedToStriped(keys, vals, 0, 32);
    float *sr = (h ? sr2 : sr1) + q * T;
    int32_t *ord = (h ? ord2 : ord1) + q * T;
    int32_t *pos = (h ? pos2 : pos1) + q * T;  // inverse permutation
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        int rank = s * kSortThreads + threadIdx.x;
        if (rank < T) {
            sr[rank] = __uint_as_float(keys[s]);
            ord[rank] = vals[s];
            pos[vals[s]] = rank;
        }
    }
}

// Partial variant for sparse tables: only the P smallest (r, index) of each
// half in sorted order (plus the unsorted r).  A 4-pass MSB radix select
// finds the P-th smallest r; elements below it, and the first of its ties in
// index order, are compacted (index order preserved) and block-sorted.
template <int ITEMS, int P>
__global__ void __launch_bounds__(kSortThreads) row_topk_kernel(
    const float *__restrict__ Q, int D, const float *__restrict__ dots1,
    const float *__restrict__ dots2, const float *__restrict__ cn1,
    const float *__restrict__ cn2, int T, float *__restrict__ sr1, float *__restrict__ sr2,
    int32_t *__restrict__ ord1, int32_t *__restrict__ ord2, float *__restrict__ ru1,
    float *__restrict__ ru2) {
    constexpr int PI = P / kSortThreads;
    using Sort = cub::BlockRadixSort<unsigned int, kSortThreads, PI, int>;
    using Scan = cub::BlockScan<unsigned int, kSortThreads>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ unsigned int hist[256];
    __shared__ unsigned int skeys[P];
    __shared__ int svals[P];
    __shared__ float s_part[kSortThreads / 32];
    __shared__ float s_qn;
    __shared__ unsigned int s_digit, s_below;

    const int64_t q = blockIdx.x;
    const int h = blockIdx.y;
    const int dh = D / 2;
    const float *qv = Q + q * D + h * dh;
    float part = 0.f;
    for (int x = threadIdx.x; x < dh; x += kSortThreads) {
        float v = qv[x];
        part = fmaf(v, v, part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        float sum = 0.f;
        for (int w = 0; w < kSortThreads / 32; w++) sum += s_part[w];
        s_qn = sum;
    }
    __syncthreads();
    const float qn = s_qn;
    const float *dots = (h ? dots2 : dots1) + q * T;
    const float *cn = h ? cn2 : cn1;
    float *ru = (h ? ru2 : ru1) + q * T;
    unsigned int keys[ITEMS];
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        const int idx = threadIdx.x * ITEMS + s;
        if (idx < T) {
            float r = __fadd_rn(__fsub_rn(__ldg(cn + idx), __fmul_rn(2.f, __ldg(dots + idx))), qn);
            if (!(r > 0.f)) r = 0.f;
            keys[s] = __float_as_uint(r);
            ru[idx] = r;
        } else {
            keys[s] = 0xFFFFFFFFu;
        }
    }
    // radix select: value bits of the P-th smallest
    unsigned int prefix = 0, mask = 0, rank = P;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += kSortThreads) hist[i] = 0;
        __syncthreads();
#pragma unroll
        for (int s = 0; s < ITEMS; s++)
            if (threadIdx.x * ITEMS + s < T && (keys[s] & mask) == prefix) atomicAdd(&hist[(keys[s] >> shift) & 0xFF], 1u);
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned int loc[8], sum = 0;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                loc[x] = hist[lane * 8 + x];
                sum += loc[x];
            }
            unsigned int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            unsigned int run = incl - sum;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                if (run < rank && run + loc[x] >= rank) {
                    s_digit = lane * 8 + x;
                    s_below = run;
                }
                run += loc[x];
            }
        }
        __syncthreads();
        rank -= s_below;
        prefix |= s_digit << shift;
        mask |= 0xFFu << shift;
        __syncthreads();
    }
    const unsigned int theta = prefix;  // rank = how many of the ties to take
    unsigned int neq = 0;
#pragma unroll
    for (int s = 0; s < ITEMS; s++) neq += (threadIdx.x * ITEMS + s < T && keys[s] == theta) ? 1u : 0u;
    unsigned int eq_before;
    Scan(tmp.scan).ExclusiveSum(neq, eq_before);
    __syncthreads();
    unsigned int take = 0;
    bool tk[ITEMS];
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        const bool valid = threadIdx.x * ITEMS + s < T;
        bool t = valid && keys[s] < theta;
        if (valid && keys[s] == theta) {
            t = eq_before < rank;
            eq_before++;
        }
        tk[s] = t;
        take += t ? 1u : 0u;
    }
    unsigned int pos;
    Scan(tmp.scan).ExclusiveSum(take, pos);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        if (tk[s]) {
            skeys[pos] = keys[s];
            svals[pos] = threadIdx.x * ITEMS + s;
            pos++;
        }
    }
    __syncthreads();
    unsigned int k2[PI];
    int v2[PI];
#pragma unroll
    for (int s = 0; s < PI; s++) {
        k2[s] = skeys[threadIdx.x * PI + s];
        v2[s] = svals[threadIdx.x * PI + s];
    }
    __syncthreads();
    Sort(tmp.sort).SortBlockedToStriped(k2, v2, 0, 32);
    float *sr = (h ? sr2 : sr1) + q * T;
    int32_t *ord = (h ? ord2 : ord1) + q * T;
#pragma unroll
    for (int s = 0; s < PI; s++) {
        const int rank_out = s * kSortThreads + threadIdx.x;
        sr[rank_out] = __uint_as_float(k2[s]);
        ord[rank_out] = v2[s];
    }
}

template <int ITEMS>
int launch_row_topk_t(const float *Q, int64_t nq, int32_t D, const float *dots1, const float *dots2,
                      const float *cn1, const float *cn2, int32_t T, float *sr1, float *sr2, int32_t *ord1,
                      int32_t *ord2, float *ru1, float *ru2, cudaStream_t stream) {
    dim3 grid((unsigned)nq, 2);
    row_topk_kernel<ITEMS, kTopP><<<grid, kSortThreads, 0, stream>>>(Q, D, dots1, dots2, cn1, cn2, T, sr1, sr2,
                                                                   ord1, ord2, ru1, ru2);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

template <int ITEMS>
int launch_row_sort_t(const float *Q, int64_t nq, int32_t D, const float *dots1,
                      const float *dots2, const float *cn1, const float *cn2, int32_t T,
                      float *sr1, float *sr2, int32_t *ord1, int32_t *ord2, int32_t *pos1,
                      int32_t *pos2, float *ru1, float *ru2, const unsigned int *qlist,
                      const unsigned int *qcount, cudaStream_t stream) {
    using Sort = cub::BlockRadixSort<unsigned int, kSortThreads, ITEMS, int>;
    size_t smem = sizeof(typename Sort::TempStorage);
    static bool configured = false;
    if (!configured) {
        BPQ_CUDA_TRY(cudaFuncSetAttribute(row_sort_kernel<ITEMS>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    dim3 grid((unsigned)nq, 2);
    row_sort_kernel<ITEMS><<<grid, kSortThreads, smem, stream>>>(Q, D, dots1, dots2, cn1, cn2, T,
                                                                 sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2,
                                                                 qlist, qcount);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace

int launch_fold(const float *queries, int64_t nq, int32_t D, int32_t M, int32_t K, const float *books,
                const float *fine_norms, float *fold, cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    const int ds = D / M;
    const size_t smem = ((size_t)K * (ds + 1) + (size_t)FQ * ds) * sizeof(float);
    static bool configured = false;
    if (!configured) {
        BPQ_CUDA_TRY(cudaFuncSetAttribute(fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    dim3 grid((unsigned)((nq + FQ - 1) / FQ), (unsigned)M);
    fold_kernel<<<grid, 256, smem, stream>>>(queries, nq, D, M, K, books, fine_norms, fold);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

int launch_coarse_dots(const float *queries, int64_t nq, int32_t D, const float *c1,
                       const float *c2, int32_t T, float *dots1, float *dots2,
                       cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    dim3 grid((T + BT - 1) / BT, (unsigned)((nq + BQ - 1) / BQ), 2);
    coarse_dots_kernel<<<grid, 256, 0, stream>>>(queries, nq, D, c1, c2, T, dots1, dots2);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

int launch_row_sort(const float *queries, int64_t nq, int32_t D, const float *dots1,
                    const float *dots2, const float *cn1, const float *cn2, int32_t T,
                    float *sr1, float *sr2, int32_t *ord1, int32_t *ord2, int32_t *pos1,
                    int32_t *pos2, float *ru1, float *ru2, const unsigned int *qlist,
                    const unsigned int *qcount, cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    if (T <= kSortThreads * 1)
        return launch_row_sort_t<1>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2, qlist, qcount, stream);
    if (T <= kSortThreads * 4)
        return launch_row_sort_t<4>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2, qlist, qcount, stream);
    if (T <= kSortThreads * 8)
        return launch_row_sort_t<8>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2, qlist, qcount, stream);
    if (T <= kSortThreads * 16)
        return launch_row_sort_t<16>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2, qlist, qcount, stream);
    if (T <= kSortThreads * 32)
        return launch_row_sort_t<32>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, pos1, pos2, ru1, ru2, qlist, qcount, stream);
    return fail(BPQ_ERR_UNSUPPORTED, "num_coarse > 16384 is outside the row-sort kernel range");
}

int launch_row_topk(const float *queries, int64_t nq, int32_t D, const float *dots1,
                    const float *dots2, const float *cn1, const float *cn2, int32_t T, float *sr1,
                    float *sr2, int32_t *ord1, int32_t *ord2, float *ru1, float *ru2, cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    if (T <= kSortThreads * 4)
        return launch_row_topk_t<4>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, stream);
    if (T <= kSortThreads * 8)
        return launch_row_topk_t<8>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, stream);
    if (T <= kSortThreads * 16)
        return launch_row_topk_t<16>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, stream);
    if (T <= kSortThreads * 32)
        return launch_row_topk_t<32>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, stream);
    return fail(BPQ_ERR_UNSUPPORTED, "num_coarse > 16384 is outside the row-sort kernel range");
}

}  // namespace bpq
