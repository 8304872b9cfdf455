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
#include <algorithm>
#include <cstdlib>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "bpq_internal.cuh"

namespace bpq {

int launch_row_cut(const float *queries, int64_t nq, int32_t D, const float *dots1, const float *dots2,
                   const float *cn1, const float *cn2, int32_t T, float *sr1, float *sr2, int32_t *ord1,
                   int32_t *ord2, float *ru1, float *ru2, int32_t *plen, cudaStream_t stream);

namespace {

constexpr int BQ = 128, BT = 128, BKC = 32;  // tile 128 x 128, k staged 32 at a time

// dots_h[q, t] = sum_x Q[q, h*dh + x] * C_h[t, x]   (h = blockIdx.z)
// 128x128 output tile per CTA, 8x8 per thread; each k chunk of 32 is loaded
// with 16-byte loads into k-major shared tiles (one barrier pair per chunk).
__global__ void __launch_bounds__(256) coarse_dots_kernel(const float *__restrict__ Q, int64_t nq,
                                                          int D, const float *__restrict__ C1,
                                                          const float *__restrict__ C2, int T,
                                                          float *__restrict__ dots1,
                                                          float *__restrict__ dots2) {
    __shared__ __align__(16) float Qs[BKC][BQ + 4];
    __shared__ __align__(16) float Cs[BKC][BT + 4];
    const int h = blockIdx.z;
    const int dh = D / 2;
    const float *C = h ? C2 : C1;
    float *out = h ? dots2 : dots1;
    const int64_t q0 = (int64_t)blockIdx.y * BQ;
    const int t0 = blockIdx.x * BT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
    const bool vec = (dh & 3) == 0 && (D & 3) == 0;
    for (int k0 = 0; k0 < dh; k0 += BKC) {
        // 128 rows x 32 k per operand = 1024 float4; 256 threads x 4
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int f = threadIdx.x + u * 256;  // float4 index
            const int row = f >> 3, kq = (f & 7) * 4;
            const int kk = k0 + kq;
            const int64_t q = q0 + row;
            const int t = t0 + row;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
            if (vec) {
                if (q < nq && kk < dh) a = __ldg(reinterpret_cast<const float4 *>(Q + q * D + h * dh + kk));
                if (t < T && kk < dh) b = __ldg(reinterpret_cast<const float4 *>(C + (int64_t)t * dh + kk));
            } else {
                float av[4], bv[4];
#pragma unroll
                for (int z = 0; z < 4; z++) {
                    av[z] = (q < nq && kk + z < dh) ? __ldg(Q + q * D + h * dh + kk + z) : 0.f;
                    bv[z] = (t < T && kk + z < dh) ? __ldg(C + (int64_t)t * dh + kk + z) : 0.f;
                }
                a = make_float4(av[0], av[1], av[2], av[3]);
                b = make_float4(bv[0], bv[1], bv[2], bv[3]);
            }
            Qs[kq + 0][row] = a.x; Qs[kq + 1][row] = a.y; Qs[kq + 2][row] = a.z; Qs[kq + 3][row] = a.w;
            Cs[kq + 0][row] = b.x; Cs[kq + 1][row] = b.y; Cs[kq + 2][row] = b.z; Cs[kq + 3][row] = b.w;
        }
        __syncthreads();
        const int kn = min(BKC, dh - k0);
#pragma unroll 8
        for (int kk = 0; kk < kn; kk++) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&Qs[kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&Qs[kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Cs[kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Cs[kk][64 + tx * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int64_t q = q0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (q >= nq) continue;
        float *orow = out + q * T;
        const int tA = t0 + tx * 4, tB = t0 + 64 + tx * 4;
        if ((T & 3) == 0 && tA + 3 < T) {
            *reinterpret_cast<float4 *>(orow + tA) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        } else {
            for (int j = 0; j < 4; j++) if (tA + j < T) orow[tA + j] = acc[i][j];
        }
        if ((T & 3) == 0 && tB + 3 < T) {
            *reinterpret_cast<float4 *>(orow + tB) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        } else {
            for (int j = 0; j < 4; j++) if (tB + j < T) orow[tB + j] = acc[i][4 + j];
        }
    }
}

// FBPQ query tables for a batch (fbpq.py:140-144): for every query, part p
// and codeword c, fold[q][p][c] = fine_norms[p][c] - 2 * (books[p][c] . q_p).
// One CTA per (64-query tile, part): the part's codebook (K x ds, padded to
// ds + 1 so the strided codeword reads are conflict-free) and the query
// slices are staged in shared memory.  Each thread owns 4 codewords (c = cg +
// 64 i) x 16 queries in registers; every dot is the same ascending-u fmaf
// chain from 0 as a scalar loop, so the values do not depend on the tiling.
constexpr int FQ = 64;

__global__ void __launch_bounds__(256, 3) fold_kernel(const float *__restrict__ Q, int64_t nq, int D, int M,
                                                   int K, const float *__restrict__ books,
                                                   const float *__restrict__ fine_norms,
                                                   float *__restrict__ fold) {
    extern __shared__ __align__(16) float fs[];
    const int p = blockIdx.y;
    const int ds = D / M;
    const int64_t q0 = (int64_t)blockIdx.x * FQ;
    float *bk = fs;                 // [K][ds+1]
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
    const int cg = threadIdx.x & 63, qg = threadIdx.x >> 6;
    float acc[4][16];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 16; j++) acc[i][j] = 0.f;
    for (int u = 0; u < ds; u++) {
        float b[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int c = cg + 64 * i;
            b[i] = c < K ? bk[c * (ds + 1) + u] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const float qv = qs[(qg * 16 + j) * ds + u];
#pragma unroll
            for (int i = 0; i < 4; i++) acc[i][j] = fmaf(b[i], qv, acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int c = cg + 64 * i;
        if (c >= K) continue;
        const float fn = __ldg(fine_norms + p * K + c);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int64_t q = q0 + qg * 16 + j;
            if (q < nq) fold[(q * M + p) * K + c] = __fsub_rn(fn, __fmul_rn(2.f, acc[i][j]));
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

    // queue mode (the retry pass): a few hundred CTAs walk the device-side list -- a grid of nq CTAs that
    // almost all exit at once cost 35 us per batch in launch overhead alone
    for (unsigned int row = blockIdx.x;; row += gridDim.x) {
    if (qlist != nullptr && row >= *qcount) return;
    const int64_t q = qlist != nullptr ? (int64_t)qlist[row] : (int64_t)row;
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
    if (qlist == nullptr) return;
    __syncthreads();  // the sort's shared storage is reused by the next row
    }
}

// Partial variant for sparse tables: only the smallest P' (256 <= P' <=
// kTopP when the value spread allows) (r, index) of each half in sorted
// order, plus the unsorted r.  One 1024-bucket histogram over the block's
// [min, max] key range (a second, finer one only when the bucket holding
// rank 256 is overfull) gives a cut value that never splits equal keys;
// the keys below it are compacted in index order and block-sorted.  P' per
// (query, half) goes to plen; the traversal queues a query for the
// full-sort retry pass if it needs a sorted position beyond P'.
constexpr int kCutMin = 256;
constexpr int kBuckets = 1024;

// SMEM_KEYS (large T): each thread's keys live in dynamic shared memory at
// the positions it loaded (no barrier needed, a thread only reads its own),
// which frees the registers that capped these rows at one CTA per SM.
template <int ITEMS, int P, bool SMEM_KEYS>
__global__ void __launch_bounds__(kSortThreads, SMEM_KEYS ? 2 : (ITEMS <= 8 ? 4 : 1)) row_topk_kernel(
    const float *__restrict__ Q, int D, const float *__restrict__ dots1,
    const float *__restrict__ dots2, const float *__restrict__ cn1,
    const float *__restrict__ cn2, int T, float *__restrict__ sr1, float *__restrict__ sr2,
    int32_t *__restrict__ ord1, int32_t *__restrict__ ord2, float *__restrict__ ru1,
    float *__restrict__ ru2, int32_t *__restrict__ plen) {
    using Scan = cub::BlockScan<unsigned int, kSortThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ unsigned int hist[kBuckets];
    __shared__ float s_part[kSortThreads / 32];
    __shared__ unsigned int s_min[kSortThreads / 32], s_max[kSortThreads / 32];
    __shared__ float s_qn;
    __shared__ unsigned int s_lo, s_cut, s_cnt, s_shift;
    __shared__ unsigned int s_wsum[kSortThreads / 32];
    __shared__ unsigned long long sk64[P];

    const int64_t q = blockIdx.x;
    const int h = blockIdx.y;
    const int dh = D / 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *qv = Q + q * D + h * dh;
    float part = 0.f;
    for (int x = threadIdx.x; x < dh; x += kSortThreads) {
        float v = qv[x];
        part = fmaf(v, v, part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_part[warp] = part;
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
    // striped float4 arrangement (coalesced 16-byte loads/stores); the
    // order of keys across threads is irrelevant to the (value, index) sort
    auto ix = [](int s) { return ((s >> 2) * kSortThreads + (int)threadIdx.x) * 4 + (s & 3); };
    unsigned int kreg[SMEM_KEYS ? 1 : ITEMS];
    extern __shared__ unsigned int skeys[];
    auto KEY = [&](int s) -> unsigned int & {
        if constexpr (SMEM_KEYS) return skeys[ix(s)];
        else return kreg[s];
    };
    unsigned int kmin = 0xFFFFFFFFu, kmax = 0u;
    auto rval = [&](float c, float d) {
        float r = __fadd_rn(__fsub_rn(c, __fmul_rn(2.f, d)), qn);
        return r > 0.f ? r : 0.f;  // np.maximum(r, 0) (multi_index.py:291-292)
    };
    if ((T & 3) == 0) {
#pragma unroll
        for (int j = 0; j < ITEMS / 4; j++) {
            const int b = ix(j * 4);
            if (b < T) {
                const float4 dv = __ldg(reinterpret_cast<const float4 *>(dots + b));
                const float4 cv = __ldg(reinterpret_cast<const float4 *>(cn + b));
                const float4 rv = make_float4(rval(cv.x, dv.x), rval(cv.y, dv.y), rval(cv.z, dv.z), rval(cv.w, dv.w));
                *reinterpret_cast<float4 *>(ru + b) = rv;
                KEY(j * 4 + 0) = __float_as_uint(rv.x);
                KEY(j * 4 + 1) = __float_as_uint(rv.y);
                KEY(j * 4 + 2) = __float_as_uint(rv.z);
                KEY(j * 4 + 3) = __float_as_uint(rv.w);
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    kmin = min(kmin, KEY(j * 4 + e));
                    kmax = max(kmax, KEY(j * 4 + e));
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; e++) KEY(j * 4 + e) = 0xFFFFFFFFu;
            }
        }
    } else {
#pragma unroll
        for (int s = 0; s < ITEMS; s++) {
            const int idx = ix(s);
            if (idx < T) {
                const float r = rval(__ldg(cn + idx), __ldg(dots + idx));
                KEY(s) = __float_as_uint(r);
                ru[idx] = r;
                kmin = min(kmin, KEY(s));
                kmax = max(kmax, KEY(s));
            } else {
                KEY(s) = 0xFFFFFFFFu;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
        s_min[warp] = kmin;
        s_max[warp] = kmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int a = 0xFFFFFFFFu, b = 0u;
        for (int w = 0; w < kSortThreads / 32; w++) {
            a = min(a, s_min[w]);
            b = max(b, s_max[w]);
        }
        const unsigned int range = b - a;
        const int bits = range ? 32 - __clz(range) : 0;
        s_lo = a;
        s_shift = bits > 10 ? bits - 10 : 0;
        s_cut = 0;
        s_cnt = 0;
    }
    __syncthreads();
    const unsigned int gmin = s_lo;
    // up to two histogram refinements of [lo, lo + 1024 << shift)
    unsigned int below = 0;  // keys already known to be under the window
    for (int pass = 0; pass < 2; pass++) {
        const unsigned int lo = s_lo, shift = s_shift;
        for (int i = threadIdx.x; i < kBuckets; i += kSortThreads) hist[i] = 0;
        __syncthreads();
#pragma unroll
        for (int s = 0; s < ITEMS; s++) {
            if (ix(s) < T && KEY(s) >= lo) {
                const unsigned int bkt = (KEY(s) - lo) >> shift;
                if (bkt < (unsigned int)kBuckets) atomicAdd(&hist[bkt], 1u);
            }
        }
        __syncthreads();
        {
            // all warps: warp w scans bins [64 w, 64 w + 64), 2 per lane
            constexpr int BPW = kBuckets / (kSortThreads / 32);
            const int b0 = warp * BPW + lane * 2;
            const unsigned int c0 = hist[b0], c1 = hist[b0 + 1];
            unsigned int incl = c0 + c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            unsigned int base = below;
            for (int w = 0; w < warp; w++) base += s_wsum[w];
            unsigned int run = base + incl - (c0 + c1);
            for (int x = 0; x < 2; x++) {
                const int bkt = b0 + x;
                const unsigned int c = x ? c1 : c0;
                if (run < (unsigned int)kCutMin && run + c >= (unsigned int)kCutMin) {
                    // bucket holding rank kCutMin: cut after it if it fits, else before it
                    if (run + c <= (unsigned int)P) {
                        s_cut = lo + ((unsigned int)(bkt + 1) << shift);
                        s_cnt = run + c;
                        s_shift = 0xFFFFFFFFu;  // done
                    } else {
                        s_cut = lo + ((unsigned int)bkt << shift);
                        s_cnt = run;
                        s_lo = lo + ((unsigned int)bkt << shift);  // refine inside this bucket
                        s_shift = shift > 10 ? shift - 10 : 0;
                        if (shift == 0) s_shift = 0xFFFFFFFFu;  // single key value: cannot split
                    }
                }
                run += c;
            }
        }
        __syncthreads();
        if (s_shift == 0xFFFFFFFFu) break;
        below = s_cnt;
    }
    // (if both passes ended inside an overfull bucket, s_cut / s_cnt hold
    // the last clean cut below it; a short prefix just retries sooner)
    const unsigned int cut = s_cut;
    // Counting sort of the keys below the cut: 1024 linear buckets over
    // [gmin, cut) (monotone in the key), scatter, then each bucket -- almost
    // always 0-3 keys -- is insertion-sorted on (value, index) by one thread,
    // so equal values keep ascending index (stable, as np.argsort).  A bucket
    // fuller than kBucketSortMax (massive ties) falls back to a bitonic sort.
    constexpr unsigned int kBucketSortMax = 24;
    const unsigned int span = cut - gmin;
    const int sbits = span ? 32 - __clz(span) : 0;
    const unsigned int sshift = sbits > 10 ? sbits - 10 : 0;
    for (int i = threadIdx.x; i < kBuckets; i += kSortThreads) hist[i] = 0;
    __syncthreads();
#pragma unroll
    for (int s = 0; s < ITEMS; s++)
        if (ix(s) < T && KEY(s) < cut) atomicAdd(&hist[(KEY(s) - gmin) >> sshift], 1u);
    __syncthreads();
    unsigned int total;
    {
        const int b0 = threadIdx.x * 2;
        const unsigned int c0 = hist[b0], c1 = hist[b0 + 1];
        unsigned int base;
        Scan(tmp.scan).ExclusiveSum(c0 + c1, base, total);
        unsigned int m = max(c0, c1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) s_wsum[warp] = m;
        __syncthreads();  // all reads of hist done before it becomes the cursor array
        hist[b0] = base;
        hist[b0 + 1] = base + c0;
    }
    __syncthreads();
    unsigned int maxb = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; w++) maxb = max(maxb, s_wsum[w]);
#pragma unroll
    for (int s = 0; s < ITEMS; s++) {
        if (ix(s) < T && KEY(s) < cut) {
            const unsigned int at = atomicAdd(&hist[(KEY(s) - gmin) >> sshift], 1u);
            sk64[at] = ((unsigned long long)KEY(s) << 32) | (unsigned int)ix(s);
        }
    }
    __syncthreads();
    if (maxb <= kBucketSortMax) {
        if (maxb > 1) {
            // hist[b] is now the end of bucket b (= start of bucket b + 1)
            for (int b = threadIdx.x; b < kBuckets; b += kSortThreads) {
                const int e = (int)hist[b], st = b ? (int)hist[b - 1] : 0;
                for (int i = st + 1; i < e; i++) {
                    const unsigned long long v = sk64[i];
                    int j = i - 1;
                    while (j >= st && sk64[j] > v) {
                        sk64[j + 1] = sk64[j];
                        j--;
                    }
                    sk64[j + 1] = v;
                }
            }
            __syncthreads();
        }
    } else {
        int P2 = 1;
        while (P2 < (int)total) P2 <<= 1;
        for (int x = total + threadIdx.x; x < P2; x += kSortThreads) sk64[x] = ~0ull;
        __syncthreads();
        for (int k = 2; k <= P2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P2; i += kSortThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const bool up = (i & k) == 0;
                        const unsigned long long x = sk64[i], y = sk64[ixj];
                        if ((x > y) == up) {
                            sk64[i] = y;
                            sk64[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    float *sr = (h ? sr2 : sr1) + q * T;
    int32_t *ord = (h ? ord2 : ord1) + q * T;
    for (int x = threadIdx.x; x < (int)total; x += kSortThreads) {
        const unsigned long long kv = sk64[x];
        sr[x] = __uint_as_float((unsigned int)(kv >> 32));
        ord[x] = (int32_t)(kv & 0xFFFFFFFFu);
    }
    if (threadIdx.x == 0) plen[q * 2 + h] = (int32_t)total;
}

template <int ITEMS>
int launch_row_topk_t(const float *Q, int64_t nq, int32_t D, const float *dots1, const float *dots2,
                      const float *cn1, const float *cn2, int32_t T, float *sr1, float *sr2, int32_t *ord1,
                      int32_t *ord2, float *ru1, float *ru2, int32_t *plen, cudaStream_t stream) {
    dim3 grid((unsigned)nq, 2);
    constexpr bool kSmem = ITEMS > 8;
    const size_t smem = kSmem ? (size_t)ITEMS * kSortThreads * 4 : 0;
    if (kSmem) {
        static bool configured = false;
        if (!configured) {
            BPQ_CUDA_TRY(cudaFuncSetAttribute(row_topk_kernel<ITEMS, kTopP, kSmem>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured = true;
        }
    }
    row_topk_kernel<ITEMS, kTopP, kSmem><<<grid, kSortThreads, smem, stream>>>(Q, D, dots1, dots2, cn1, cn2, T, sr1,
                                                                            sr2, ord1, ord2, ru1, ru2, plen);
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
    dim3 grid((unsigned)(qlist != nullptr ? std::min<int64_t>(nq, 296) : nq), 2);
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
                    float *sr2, int32_t *ord1, int32_t *ord2, float *ru1, float *ru2, int32_t *plen,
                    cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    // BPQ_ROW_CUT=1: the TMA-staged, sample-cut kernel (rowcut.cu).  Measured on B200 against the
    // histogram kernel below: config 4 (T = 16384) 1.29 vs 1.40 ms, config 1 (T = 4096) 0.73 vs 0.44 ms
    // (two persistent CTAs per SM against four one-row CTAs), so it is off for those shapes
    // ... except for T > 8192 (32 keys per thread), where it is the faster one and the default;
    // BPQ_ROW_CUT=0 / 1 forces either
    const char *rc_env = getenv("BPQ_ROW_CUT");
    const bool row_cut = rc_env != nullptr ? atoi(rc_env) != 0 : T > kSortThreads * 16;
    if ((T & 3) == 0 && row_cut)
        return launch_row_cut(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kSortThreads * 4)
        return launch_row_topk_t<4>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kSortThreads * 8)
        return launch_row_topk_t<8>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kSortThreads * 16)
        return launch_row_topk_t<16>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kSortThreads * 32)
        return launch_row_topk_t<32>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    return fail(BPQ_ERR_UNSUPPORTED, "num_coarse > 16384 is outside the row-sort kernel range");
}

namespace {
// out[q][x] = sum_y X[q][y] * R[y][x]: 64x64 tiles, 4x4 per thread (FFMA).
__global__ void __launch_bounds__(256) rotate_kernel(const float *__restrict__ X, int64_t n, int d,
                                                     const float *__restrict__ R, float *__restrict__ out) {
    __shared__ float Xs[16][64 + 4];
    __shared__ float Rs[16][64 + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t q0 = (int64_t)blockIdx.y * 64;
    const int x0 = blockIdx.x * 64;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < d; k0 += 16) {
        for (int f = threadIdx.x; f < 64 * 16; f += 256) {
            const int r = f >> 4, kk = f & 15;      // X tile: row r, k kk
            const int64_t q = q0 + r;
            Xs[kk][r] = (q < n && k0 + kk < d) ? __ldg(X + q * d + k0 + kk) : 0.f;
            const int kr = f >> 6, c = f & 63;      // R tile: k kr, column c
            Rs[kr][c] = (k0 + kr < d && x0 + c < d) ? __ldg(R + (int64_t)(k0 + kr) * d + x0 + c) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; kk++) {
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(Xs[kk][ty * 4 + i], Rs[kk][tx * 4 + j], acc[i][j]);
        }
        __syncthreads();
    }
    for (int i = 0; i < 4; i++) {
        const int64_t q = q0 + ty * 4 + i;
        if (q >= n) continue;
        for (int j = 0; j < 4; j++) {
            const int x = x0 + tx * 4 + j;
            if (x < d) out[q * d + x] = acc[i][j];
        }
    }
}
}  // namespace

int launch_rotate(const float *x, int64_t n, int32_t d, const float *R, float *out, cudaStream_t stream) {
    if (n == 0) return BPQ_OK;
    dim3 grid((d + 63) / 64, (unsigned)((n + 63) / 64));
    rotate_kernel<<<grid, 256, 0, stream>>>(x, n, d, R, out);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace bpq

extern "C" int bpq_rotate(const float *x, int64_t n, int32_t d, const float *R, float *out, void *stream) {
    BPQ_CHECK(n >= 0 && d >= 1 && x && R && out, BPQ_ERR_INVALID, "bad rotate arguments");
    return bpq::launch_rotate(x, n, d, R, out, (cudaStream_t)stream);
}
