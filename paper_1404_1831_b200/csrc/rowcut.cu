// Partial row sort for sparse tables, second generation (`row_cut_kernel`).
//
// Same contract as row_topk_kernel (prep.cu): for each (query, half) the
// unsorted r = max((cn - 2*dot) + |q_h|^2, 0) of every codeword (ru) and the
// smallest P' keys (bits(r), index) in stable sorted order (sr / ord, P' to
// plen), where the cut never splits equal keys.  P' is wherever the cut
// falls (0 .. P); the traversal extends a prefix in place, or queues the
// query for the full-sort pass, when it needs more
// (multi_index.py:319-322 is the reference's full stable argsort).
//
// What changed:
//   * persistent CTAs; the NEXT row's dots (T floats, contiguous) are
//     fetched by one TMA bulk copy into shared memory while the current row
//     is selected and sorted, so no phase waits on HBM;
//   * keys live in registers (T / 512 per thread);
//   * the cut comes from a sample instead of two 1024-bucket histogram
//     passes over all T keys: every warp takes the j-th smallest of 32
//     sampled keys (j ~ 32 * 384 / T), three order statistics of the 16 warp
//     values are candidate cuts, one counting pass over the registers picks
//     the candidate whose prefix lands in [192, P].
#include <cub/block/block_scan.cuh>

#include "bpq_internal.cuh"

namespace bpq {

namespace {

constexpr int kRowThreads = 512;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kRowBuckets = 1024;
constexpr unsigned int kRowTarget = 384;  // aimed prefix length
constexpr unsigned int kRowMinOk = 192;   // a shorter prefix tries the next larger candidate (the first batch probes up to 130)

__device__ __forceinline__ uint32_t rc_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void rc_mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(rc_smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void rc_bulk_row(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // earlier generic reads of dst
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(rc_smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     rc_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(rc_smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void rc_mbar_wait(unsigned long long *bar, unsigned parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(rc_smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

// rank of v among the n lane values of the warp's first n lanes (ties by lane)
__device__ __forceinline__ int warp_rank(unsigned int v, int lane, int n) {
    int rank = 0;
#pragma unroll
    for (int l = 0; l < 32; l++) {
        const unsigned int o = __shfl_sync(0xffffffffu, v, l);
        rank += (l < n && (o < v || (o == v && l < lane))) ? 1 : 0;
    }
    return rank;
}

template <int ITEMS, int P>
__global__ void __launch_bounds__(kRowThreads, 2) row_cut_kernel(
    const float *__restrict__ Q, int D, const float *__restrict__ dots1, const float *__restrict__ dots2,
    const float *__restrict__ cn1, const float *__restrict__ cn2, int T, float *__restrict__ sr1,
    float *__restrict__ sr2, int32_t *__restrict__ ord1, int32_t *__restrict__ ord2, float *__restrict__ ru1,
    float *__restrict__ ru2, int32_t *__restrict__ plen, int64_t nq) {
    using Scan = cub::BlockScan<unsigned int, kRowThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned int hist[kRowBuckets];
    __shared__ float s_part[kRowWarps];
    __shared__ unsigned int s_wstat[kRowWarps];
    __shared__ unsigned int s_wcnt[kRowWarps][4];  // counts under the three candidates, min key
    __shared__ unsigned int s_cand[3];
    __shared__ unsigned int s_wsum[kRowWarps];
    __shared__ float s_qn;
    __shared__ unsigned int s_cut, s_gmin;
    __shared__ unsigned long long sk64[P];
    __shared__ unsigned long long mbar;
    extern __shared__ __align__(16) float stage[];  // [T]: the row's dots, written by TMA

    const int h = blockIdx.x & 1;  // a CTA stays on one half: its codeword norms stay cached
    const int64_t qstep = gridDim.x >> 1;
    const int dh = D / 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *dots_h = h ? dots2 : dots1;
    const float *cn = h ? cn2 : cn1;
    const unsigned int row_bytes = (unsigned int)T * 4u;
    // striped float4 arrangement as row_topk_kernel: the order of keys across threads is irrelevant
    auto ix = [](int s) { return ((s >> 2) * kRowThreads + (int)threadIdx.x) * 4 + (s & 3); };

    int64_t q = blockIdx.x >> 1;
    if (threadIdx.x == 0) {
        rc_mbar_init(&mbar, 1);
        if (q < nq) rc_bulk_row(stage, dots_h + q * T, row_bytes, &mbar);
    }
    __syncthreads();
    unsigned int parity = 0;
    for (; q < nq; q += qstep) {
        // |q_h|^2 in row_topk_kernel's order (same bits in r)
        const float *qv = Q + q * D + h * dh;
        float part = 0.f;
        for (int x = threadIdx.x; x < dh; x += kRowThreads) {
            float v = qv[x];
            part = fmaf(v, v, part);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) s_part[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            float sum = 0.f;
            for (int w = 0; w < kRowWarps; w++) sum += s_part[w];
            s_qn = sum;
        }
        __syncthreads();
        const float qn = s_qn;
        float *ru = (h ? ru2 : ru1) + q * T;
        auto rval = [&](float c, float d) {
            float r = __fadd_rn(__fsub_rn(c, __fmul_rn(2.f, d)), qn);
            return r > 0.f ? r : 0.f;  // np.maximum(r, 0) (multi_index.py:291-292)
        };
        rc_mbar_wait(&mbar, parity);
        parity ^= 1u;
        unsigned int kreg[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS / 4; j++) {
            const int b = ix(j * 4);
            if (b < T) {
                const float4 dv = *reinterpret_cast<const float4 *>(stage + b);
                const float4 cv = __ldg(reinterpret_cast<const float4 *>(cn + b));
                const float4 rv = make_float4(rval(cv.x, dv.x), rval(cv.y, dv.y), rval(cv.z, dv.z), rval(cv.w, dv.w));
                *reinterpret_cast<float4 *>(ru + b) = rv;
                kreg[j * 4 + 0] = __float_as_uint(rv.x);
                kreg[j * 4 + 1] = __float_as_uint(rv.y);
                kreg[j * 4 + 2] = __float_as_uint(rv.z);
                kreg[j * 4 + 3] = __float_as_uint(rv.w);
            } else {
#pragma unroll
                for (int e = 0; e < 4; e++) kreg[j * 4 + e] = 0xFFFFFFFFu;
            }
        }
        __syncthreads();  // the stage has been read: refill it with the next row under the selection
        if (threadIdx.x == 0 && q + qstep < nq) rc_bulk_row(stage, dots_h + (q + qstep) * T, row_bytes, &mbar);

        // ---- cut from a sample: per warp the j-th smallest of 32 keys, then 3 order statistics of 16
        {
            const int sel = (int)(threadIdx.x % ITEMS);
            unsigned int smp = kreg[0];
#pragma unroll
            for (int s = 1; s < ITEMS; s++) smp = s == sel ? kreg[s] : smp;
            int j0 = (int)((32u * kRowTarget + (unsigned int)T / 2u) / (unsigned int)T);
            j0 = min(max(j0, 1), 16) - 1;
            if (warp_rank(smp, lane, 32) == j0) s_wstat[warp] = smp;
        }
        __syncthreads();
        if (warp == 0) {
            const unsigned int v = lane < kRowWarps ? s_wstat[lane] : 0xFFFFFFFFu;
            const int rk = warp_rank(v, lane, kRowWarps);
            if (lane < kRowWarps) {
                if (rk == 4) s_cand[0] = v;
                if (rk == 8) s_cand[1] = v;
                if (rk == 12) s_cand[2] = v;
            }
        }
        __syncthreads();
        {
            const unsigned int ca = s_cand[0], cb = s_cand[1], cc = s_cand[2];
            unsigned int na = 0, nb = 0, nc = 0, kmin = 0xFFFFFFFFu;
#pragma unroll
            for (int s = 0; s < ITEMS; s++) {
                const unsigned int key = kreg[s];
                na += key < ca ? 1u : 0u;
                nb += key < cb ? 1u : 0u;
                nc += key < cc ? 1u : 0u;
                kmin = min(kmin, key);
            }
            na = __reduce_add_sync(0xffffffffu, na);
            nb = __reduce_add_sync(0xffffffffu, nb);
            nc = __reduce_add_sync(0xffffffffu, nc);
            kmin = __reduce_min_sync(0xffffffffu, kmin);
            if (lane == 0) {
                s_wcnt[warp][0] = na;
                s_wcnt[warp][1] = nb;
                s_wcnt[warp][2] = nc;
                s_wcnt[warp][3] = kmin;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int na = 0, nb = 0, nc = 0, kmin = 0xFFFFFFFFu;
            for (int w = 0; w < kRowWarps; w++) {
                na += s_wcnt[w][0];
                nb += s_wcnt[w][1];
                nc += s_wcnt[w][2];
                kmin = min(kmin, s_wcnt[w][3]);
            }
            // the middle candidate when its prefix fits; a smaller one when it is too long, a larger one
            // when it is too short; no prefix at all (the traversal extends from nothing) if none fits
            unsigned int cut = kmin;
            if (nb <= (unsigned int)P && (nb >= kRowMinOk || nc > (unsigned int)P)) cut = s_cand[1];
            else if (nb > (unsigned int)P) cut = na <= (unsigned int)P ? s_cand[0] : kmin;
            else cut = s_cand[2];  // nb < kRowMinOk and nc fits
            s_cut = cut;
            s_gmin = kmin;
        }
        for (int i = threadIdx.x; i < kRowBuckets; i += kRowThreads) hist[i] = 0;
        __syncthreads();
        const unsigned int cut = s_cut, gmin = s_gmin;
        // ---- counting sort of the keys below the cut (row_topk_kernel's): 1024 linear buckets over
        // [gmin, cut), scatter, insertion sort inside each bucket on (value, index) -- stable
        constexpr unsigned int kBucketSortMax = 24;
        const unsigned int span = cut - gmin;
        const int sbits = span ? 32 - __clz(span) : 0;
        const unsigned int sshift = sbits > 10 ? sbits - 10 : 0;
#pragma unroll
        for (int s = 0; s < ITEMS; s++)
            if (kreg[s] < cut) atomicAdd(&hist[(kreg[s] - gmin) >> sshift], 1u);
        __syncthreads();
        unsigned int total;
        {
            const int b0 = threadIdx.x * 2;
            const unsigned int c0 = hist[b0], c1 = hist[b0 + 1];
            unsigned int base;
            Scan(scan_tmp).ExclusiveSum(c0 + c1, base, total);
            unsigned int m = max(c0, c1);
            m = __reduce_max_sync(0xffffffffu, m);
            if (lane == 0) s_wsum[warp] = m;
            __syncthreads();  // all reads of hist done before it becomes the cursor array
            hist[b0] = base;
            hist[b0 + 1] = base + c0;
        }
        __syncthreads();
        unsigned int maxb = 0;
#pragma unroll
        for (int w = 0; w < kRowWarps; w++) maxb = max(maxb, s_wsum[w]);
#pragma unroll
        for (int s = 0; s < ITEMS; s++) {
            if (kreg[s] < cut) {
                const unsigned int at = atomicAdd(&hist[(kreg[s] - gmin) >> sshift], 1u);
                sk64[at] = ((unsigned long long)kreg[s] << 32) | (unsigned int)ix(s);
            }
        }
        __syncthreads();
        if (maxb <= kBucketSortMax) {
            if (maxb > 1) {
                // hist[b] is now the end of bucket b (= start of bucket b + 1)
                for (int b = threadIdx.x; b < kRowBuckets; b += kRowThreads) {
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
            for (int x = total + threadIdx.x; x < P2; x += kRowThreads) sk64[x] = ~0ull;
            __syncthreads();
            for (int k = 2; k <= P2; k <<= 1) {
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = threadIdx.x; i < P2; i += kRowThreads) {
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
        for (int x = threadIdx.x; x < (int)total; x += kRowThreads) {
            const unsigned long long kv = sk64[x];
            sr[x] = __uint_as_float((unsigned int)(kv >> 32));
            ord[x] = (int32_t)(kv & 0xFFFFFFFFu);
        }
        if (threadIdx.x == 0) plen[q * 2 + h] = (int32_t)total;
        __syncthreads();  // sk64 / hist / s_* are reused by the next row
    }
}

template <int ITEMS>
int launch_row_cut_t(const float *Q, int64_t nq, int32_t D, const float *dots1, const float *dots2, const float *cn1,
                     const float *cn2, int32_t T, float *sr1, float *sr2, int32_t *ord1, int32_t *ord2, float *ru1,
                     float *ru2, int32_t *plen, cudaStream_t stream) {
    const size_t smem = (size_t)T * 4;
    auto kfn = row_cut_kernel<ITEMS, kTopP>;
    static bool configured = false;
    static int ctas = 0;
    if (!configured) {
        BPQ_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        configured = true;
    }
    if (ctas == 0) {
        int dev = 0, sms = 0;
        BPQ_CUDA_TRY(cudaGetDevice(&dev));
        BPQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ctas = sms;
    }
    int occ = 0;
    BPQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kRowThreads, smem));
    if (occ < 1) return fail(BPQ_ERR_UNSUPPORTED, "row-cut kernel shared memory does not fit on an SM");
    int64_t grid = (int64_t)occ * ctas;  // even: 148 SMs x occ
    grid &= ~(int64_t)1;
    if (grid > 2 * nq) grid = 2 * nq;
    kfn<<<(unsigned)grid, kRowThreads, smem, stream>>>(Q, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2,
                                                      plen, nq);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace

// TMA-staged, sample-cut partial row sort; T a multiple of 4 in (1024, 16384]
int launch_row_cut(const float *queries, int64_t nq, int32_t D, const float *dots1, const float *dots2,
                   const float *cn1, const float *cn2, int32_t T, float *sr1, float *sr2, int32_t *ord1,
                   int32_t *ord2, float *ru1, float *ru2, int32_t *plen, cudaStream_t stream) {
    if (nq == 0) return BPQ_OK;
    if (T <= kRowThreads * 4)
        return launch_row_cut_t<4>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kRowThreads * 8)
        return launch_row_cut_t<8>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kRowThreads * 16)
        return launch_row_cut_t<16>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    if (T <= kRowThreads * 32)
        return launch_row_cut_t<32>(queries, nq, D, dots1, dots2, cn1, cn2, T, sr1, sr2, ord1, ord2, ru1, ru2, plen, stream);
    return fail(BPQ_ERR_UNSUPPORTED, "num_coarse > 16384 is outside the row-sort kernel range");
}

}  // namespace bpq
