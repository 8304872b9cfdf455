// Large-cell stream kernels (point-term FBPQ, M = 8 / 16) and their launch:
// cell_flow_kernel (register-pipelined, the default) and the TMA-ring
// kernels big_scan_kernel / big_stream_kernel kept for A/B runs
// (BPQ_STREAM_TMA=1).  Included by stream_inst.cu only, after
// search_impl.cuh (Args, top-k compaction, block utilities), so editing this
// file does not rebuild the fused search instantiations.
#pragma once
#include "search_impl.cuh"

namespace bpq {
namespace {

// ------------------------------------------------------------------------
// Large-cell stream (point-term FBPQ, M = 8 / 16).  For every query the
// traversal kernel handed over (its small cells' top-k plus the list of its
// large cells), stream the cells' contiguous code / point-term ranges
// through a ring of kRingS shared-memory stages filled by TMA bulk copies
// (cp.async.bulk, one elected thread, mbarrier completion), kRingCh entries
// per stage, kRingS - 1 stages in flight.  Chunks start at a 32-entry
// boundary, so lane l always scores entries with index % 32 == l and its
// replicated-table offsets (LaneLut) are per-lane constants; leading entries
// outside the cell are skipped, and entries past the 4-aligned end of the
// arrays are read directly.  The fold table is the conflict-free replicated
// layout (fold_index).  2 CTAs per SM.
template <int MT>
__host__ __device__ constexpr int ring_chunk() { return MT == 16 ? 512 : 1024; }
#ifndef BPQ_RING_S
#define BPQ_RING_S 4
#endif
constexpr int kRingS = BPQ_RING_S;
template <int MT>
__host__ __device__ constexpr int ring_bytes() { return kRingS * ring_chunk<MT>() * (MT + 4); }

// shared state of big_scan_kernel with BT threads
template <int BT>
struct __align__(16) ScanSmem {
    unsigned long long mbar[kRingS];
    uint32_t hist_c[256];
    unsigned long long red[BT / 32];
    unsigned long long tor[BT / 32];
    unsigned long long thr;
    uint32_t ntk;
    int tsel_v;
    uint32_t tcnt;
    unsigned long long tsel_below;
    unsigned long long tkey;
    uint32_t nholes;
    uint16_t holes[kMaxK];
    int64_t qidx;
    int prof_ph;
    long long prof_t;
};

template <int MT, int BT, typename KT, typename OffT>
__global__ void __launch_bounds__(BT, 2) big_scan_kernel(Args<KT, OffT> A) {
    static_assert(MT == 8 || MT == 16, "large-cell stream needs M = 8 or 16");
    constexpr int kCh = ring_chunk<MT>();
    constexpr int kPer = kCh / BT;
    constexpr int R = 32 / MT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmem<BT> &S = *reinterpret_cast<ScanSmem<BT> *>(smem_raw);
    float *tab = reinterpret_cast<float *>(smem_raw + ((sizeof(ScanSmem<BT>) + 15) & ~(size_t)15));  // replicated fold
    unsigned long long *tk = reinterpret_cast<unsigned long long *>(smem_raw + A.tk_off);
    uint8_t *stc = smem_raw + A.tk_off + (size_t)A.tkcap * 8;      // [kRingS][kCh][MT] codes
    float *stp = reinterpret_cast<float *>(stc + (size_t)kRingS * kCh * MT);  // [kRingS][kCh] point terms
    const int K = A.K, k = A.k;
    const uint32_t nal = A.n_local & ~3u;  // 4-aligned end of the arrays
    // this lane's rotation and replica slots (chunks start at a 32-entry boundary: lane l scores
    // entries with index % 32 == l); byte offsets into the replicated table
    const char *tabb = reinterpret_cast<const char *>(tab);
    int offb[MT];
    {
        const LaneLut<MT> L((int)(threadIdx.x & 31));
#pragma unroll
        for (int i = 0; i < MT; i++) offb[i] = L.off[i] * 4;
    }
    if (threadIdx.x == 0) {
        for (int st = 0; st < kRingS; st++) mbar_init(&S.mbar[st], 1);
        mbar_fence_init();
#ifdef BPQ_PHASE_PROF
        S.prof_ph = PH_IDLE;
        S.prof_t = clock64();
#endif
    }
    uint32_t ph = 0;  // stage mbarrier parities (block-uniform)
    for (;;) {
        PROF(PH_BPRO);
        if (threadIdx.x == 0) {
            const unsigned int c = atomicAdd(A.counter, 1u);
            S.qidx = c < *A.bigq_count ? (int64_t)A.bigq_list[c] : (int64_t)-1;
        }
        __syncthreads();
        const int64_t qi = S.qidx;
        if (qi < 0) {
            PROF(PH_IDLE);
            return;
        }
        // replicated fold table and the small cells' top-k
        const float *fq = A.fold + (size_t)qi * MT * K;
        for (int x = threadIdx.x; x < MT * K; x += BT) {
            const int p = x / K, c = x - p * K;
            const float v = __ldg(fq + x);
#pragma unroll
            for (int r = 0; r < R; r++) tab[fold_index<MT>(p, c, K) + r] = v;
        }
        const uint32_t n0 = A.tk_n[qi];
        unsigned long long mx = 0;
        for (uint32_t x = threadIdx.x; x < n0; x += BT) {
            const unsigned long long key = A.tk_part[(size_t)qi * k + x];
            tk[x] = key;
            mx = key > mx ? key : mx;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = y > mx ? y : mx;
        }
        if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m = 0;
            for (int w = 0; w < BT / 32; w++) m = S.red[w] > m ? S.red[w] : m;
            S.ntk = n0;
            // k keys held: the k-th smallest (their max) is the admission bound
            S.thr = n0 >= (uint32_t)k ? m : ~0ull;
        }
        __syncthreads();
        // stream the large cells
        const int4 *cells = A.big_cells + (A.big_start ? (size_t)A.big_start[qi] : (size_t)qi * A.big_cap);
        const uint32_t nb = A.big_n[qi];
        uint32_t x_i = 0, c_i = 0, x_c = 0, c_c = 0;  // issue / score cursors: cell, chunk start
        if (nb) c_i = c_c = (uint32_t)__ldg(&cells[0].x) & ~31u;
        if (threadIdx.x == 0) fence_proxy_async();  // the ring's previous readers were generic loads
        auto issue = [&](int slot) {
            if (x_i >= nb) return;
            const int4 cl = __ldg(&cells[x_i]);
            const uint32_t end = (uint32_t)cl.x + (uint32_t)cl.y;
            if (threadIdx.x == 0) {
                const uint32_t b1 = min(min(c_i + (uint32_t)kCh, (end + 3u) & ~3u), nal);
                const uint32_t n = b1 > c_i ? b1 - c_i : 0u;
                unsigned long long *bar = &S.mbar[slot];
                mbar_arrive_tx(bar, n * (MT + 4));
                if (n) {
                    bulk_g2s(stc + (size_t)slot * kCh * MT, A.codes_rot + (size_t)c_i * MT, n * MT, bar);
                    bulk_g2s(stp + (size_t)slot * kCh, A.pterm + c_i, n * 4, bar);
                }
            }
            c_i += kCh;
            if (c_i >= end) {
                x_i++;
                if (x_i < nb) c_i = (uint32_t)__ldg(&cells[x_i].x) & ~31u;
            }
        };
#pragma unroll
        for (int r = 0; r < kRingS - 1; r++) issue(r);
        for (int r = 0; x_c < nb; r++) {
            issue((r + kRingS - 1) % kRingS);
            const int slot = r % kRingS;
            PROF(PH_BWAIT);
            mbar_wait(&S.mbar[slot], (ph >> slot) & 1u);
            ph ^= 1u << slot;
            PROF(PH_BSCORE);
            const int4 cl = __ldg(&cells[x_c]);
            const uint32_t lst = (uint32_t)cl.x, end = lst + (uint32_t)cl.y;
            const float cb = __int_as_float(cl.z);
            const uint32_t b1 = min(min(c_c + (uint32_t)kCh, (end + 3u) & ~3u), nal);
            const uint32_t thr_hi = (uint32_t)(S.thr >> 32);
            // straight-line over the thread's kPer entries (independent chains): codes and point
            // terms from the stage (stale slots past the copied range are masked below), the rare
            // entries past the arrays' aligned end from global memory
            uint32_t w[kPer][4];
            float ptv[kPer], acc[kPer];
#pragma unroll
            for (int u = 0; u < kPer; u++) {
                const int j = u * BT + threadIdx.x;
                if constexpr (MT == 16) {
                    const uint4 v = *reinterpret_cast<const uint4 *>(stc + ((size_t)slot * kCh + j) * MT);
                    w[u][0] = v.x; w[u][1] = v.y; w[u][2] = v.z; w[u][3] = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2 *>(stc + ((size_t)slot * kCh + j) * MT);
                    w[u][0] = v.x; w[u][1] = v.y; w[u][2] = 0; w[u][3] = 0;
                }
                ptv[u] = stp[slot * kCh + j];
            }
            if (c_c + (uint32_t)kCh > b1 && end > b1) {
#pragma unroll
                for (int u = 0; u < kPer; u++) {
                    const uint32_t e = c_c + u * BT + threadIdx.x;
                    if (e >= b1 && e < end) {
                        load_code<MT>(A.codes_rot + (size_t)e * MT, w[u], MT);
                        ptv[u] = __ldg(A.pterm + e);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kPer; u++) acc[u] = dist_pt_rep<MT>(tabb, offb, cb, ptv[u], w[u]);
            // admission: the distance bits first; the id reads of all admitted entries go out
            // together (one exposed load latency per chunk, not one per entry)
            uint32_t dbv[kPer], idv[kPer];
            bool ok[kPer];
#pragma unroll
            for (int u = 0; u < kPer; u++) {
                const uint32_t e = c_c + u * BT + threadIdx.x;
                dbv[u] = canon_bits(acc[u]);
                ok[u] = e >= lst && e < end && dbv[u] <= thr_hi;
                idv[u] = ok[u] ? __ldg(A.ids + e) : 0u;
            }
            const unsigned long long thr = S.thr;
#pragma unroll
            for (int u = 0; u < kPer; u++) {
                const unsigned long long kk = ((unsigned long long)dbv[u] << 32) | idv[u];
                if (ok[u] && kk < thr) tk[atomicAdd(&S.ntk, 1u)] = kk;
            }
            c_c += kCh;
            if (c_c >= end) {
                x_c++;
                if (x_c < nb) c_c = (uint32_t)__ldg(&cells[x_c].x) & ~31u;
            }
            __syncthreads();
            if (S.ntk > (uint32_t)(A.tkcap - kCh)) {
                PROF(PH_BCOMPACT);
                topk_compact<BT>(S, tk, k);
            }
        }
        PROF(PH_BFIN);
        topk_compact<BT>(S, tk, k);
        const int64_t qo = A.q0 + qi;
        write_topk<BT>(S, tk, k, A.ncand_q[qi], A.out_d + qo * k, A.out_ids + qo * k, A.out_count + qo);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// Warp-independent large-cell stream (k <= kStreamMaxK).  Same ring and
// lane mapping as big_scan_kernel, but no CTA barrier per chunk: each warp
// scores its own 1/8 of every chunk and keeps its own top-k candidates in
// a private shared-memory region (warp ballots append, a warp-level radix
// select compacts), and the LAST warp to finish a chunk refills its stage
// (an arrival counter per stage), so warps drift up to the ring depth apart
// instead of waiting for the slowest at every chunk.  The tightest per-warp
// k-th key is published (atomicMin) as a bound every warp admits against.
// The warps' lists and the traversal kernel's list are merged once per
// query by the CTA top-k.
constexpr int kStreamMaxK = 256;
constexpr int kCapW = 384;   // per-warp top-k region (keys)
constexpr int kPlan = 512;   // cells whose chunk plan is staged at a time

struct __align__(16) StreamSmem {
    unsigned long long mbar[kRingS];
    uint32_t done[kRingS];
    uint32_t plan[kPlan + 1];  // chunk prefix over the batch's cells
    unsigned long long gthr;   // admission bound: min over warps of their k-th key
    uint32_t wcnt[NW];
    uint32_t wscan[NW];
    int64_t qidx;
    // CTA top-k (topk_compact / write_topk)
    uint32_t hist_c[256];
    unsigned long long red[NW];
    unsigned long long tor[NW];
    unsigned long long thr;
    uint32_t ntk;
    int tsel_v;
    uint32_t tcnt;
    unsigned long long tsel_below;
    unsigned long long tkey;
    uint32_t nholes;
    uint16_t holes[kMaxK];
    int prof_ph;
    long long prof_t;
};

// k-th smallest of a warp's n (> k) unique keys in tkw[0, n), n <= kCapW:
// MSB-first bit construction with warp-wide counts, then the k survivors
// are packed to tkw[0, k).  Returns the k-th key (the warp's admission bound).
__device__ unsigned long long warp_topk(unsigned long long *tkw, uint32_t n, int k) {
    constexpr int PER = kCapW / 32;
    const int lane = threadIdx.x & 31;
    unsigned long long key[PER];
    unsigned long long ka = ~0ull, ko = 0ull;
#pragma unroll
    for (int i = 0; i < PER; i++) {
        const uint32_t idx = lane + 32 * i;
        key[i] = idx < n ? tkw[idx] : ~0ull;
        if (idx < n) {
            ka &= key[i];
            ko |= key[i];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ka &= __shfl_xor_sync(0xffffffffu, ka, o);
        ko |= __shfl_xor_sync(0xffffffffu, ko, o);
    }
    const int hb = 63 - __clzll((long long)(ka ^ ko));  // keys unique: ka != ko
    unsigned long long v = hb >= 63 ? 0ull : (ka & ~((2ull << hb) - 1));
    for (int b = hb; b >= 0; b--) {
        const unsigned long long cand = v | ((1ull << b) - 1);
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < PER; i++) c += key[i] <= cand ? 1u : 0u;
        c = __reduce_add_sync(0xffffffffu, c);
        if (c < (uint32_t)k) v |= 1ull << b;
    }
    __syncwarp();
    uint32_t pos = 0;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < PER; i++) {
        const bool keep = key[i] <= v;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) tkw[pos + __popc(bal & lt)] = key[i];
        pos += __popc(bal);
    }
    __syncwarp();
    return v;
}

template <int MT, typename KT, typename OffT>
__global__ void __launch_bounds__(NT, 2) big_stream_kernel(Args<KT, OffT> A) {
    static_assert(MT == 8 || MT == 16, "large-cell stream needs M = 8 or 16");
    constexpr int kCh = ring_chunk<MT>();
    constexpr int kPerW = kCh / NW;  // entries per warp per chunk
    constexpr int kPer = kPerW / 32;  // per lane
    constexpr int R = 32 / MT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    StreamSmem &S = *reinterpret_cast<StreamSmem *>(smem_raw);
    float *tab = reinterpret_cast<float *>(smem_raw + ((sizeof(StreamSmem) + 15) & ~(size_t)15));
    unsigned long long *tkall = reinterpret_cast<unsigned long long *>(smem_raw + A.tk_off);  // [NW][kCapW]
    uint8_t *stc = reinterpret_cast<uint8_t *>(tkall + NW * kCapW);                       // [kRingS][kCh][MT]
    float *stp = reinterpret_cast<float *>(stc + (size_t)kRingS * kCh * MT);               // [kRingS][kCh]
    const int K = A.K, k = A.k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t nal = A.n_local & ~3u;
    unsigned long long *tkw = tkall + warp * kCapW;
    const char *tabb = reinterpret_cast<const char *>(tab);
    int offb[MT];
    {
        const LaneLut<MT> L(lane);
#pragma unroll
        for (int i = 0; i < MT; i++) offb[i] = L.off[i] * 4;
    }
    if (threadIdx.x == 0) {
        for (int st = 0; st < kRingS; st++) {
            mbar_init(&S.mbar[st], 1);
            S.done[st] = 0;
        }
        mbar_fence_init();
#ifdef BPQ_PHASE_PROF
        S.prof_ph = PH_IDLE;
        S.prof_t = clock64();
#endif
    }
    uint32_t base = 0;  // chunks streamed so far by this CTA (stage = base % kRingS, parity = base / kRingS)
    for (;;) {
        PROF(PH_BPRO);
        if (threadIdx.x == 0) {
            const unsigned int c = atomicAdd(A.counter, 1u);
            S.qidx = c < *A.bigq_count ? (int64_t)A.bigq_list[c] : (int64_t)-1;
        }
        __syncthreads();
        const int64_t qi = S.qidx;
        if (qi < 0) {
            PROF(PH_IDLE);
            return;
        }
        const float *fq = A.fold + (size_t)qi * MT * K;
        for (int x = threadIdx.x; x < MT * K; x += NT) {
            const int p = x / K, c = x - p * K;
            const float v = __ldg(fq + x);
#pragma unroll
            for (int r = 0; r < R; r++) tab[fold_index<MT>(p, c, K) + r] = v;
        }
        // the traversal kernel's k-th key (if it holds k) bounds admission from the start
        const uint32_t n0 = A.tk_n[qi];
        unsigned long long mx = 0;
        for (uint32_t x = threadIdx.x; x < n0; x += NT) {
            const unsigned long long key = A.tk_part[(size_t)qi * k + x];
            mx = key > mx ? key : mx;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = y > mx ? y : mx;
        }
        if (lane == 0) S.red[warp] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m = 0;
            for (int w = 0; w < NW; w++) m = S.red[w] > m ? S.red[w] : m;
            S.gthr = n0 >= (uint32_t)k ? m : ~0ull;
        }
        __syncthreads();
        uint32_t wcnt = 0;
        unsigned long long wthr = ~0ull;
        const int4 *cells = A.big_cells + (size_t)qi * A.big_cap;
        const uint32_t nb = A.big_n[qi];
        for (uint32_t xb = 0; xb < nb; xb += kPlan) {
            const uint32_t nbb = min((uint32_t)kPlan, nb - xb);
            // chunk plan: prefix of each cell's chunk count (chunks start at a 32-entry boundary)
            {
                constexpr int PT = (kPlan + NT - 1) / NT;
                uint32_t cnt[PT], sum = 0;
#pragma unroll
                for (int i = 0; i < PT; i++) {
                    const uint32_t x = threadIdx.x * PT + i;
                    cnt[i] = 0;
                    if (x < nbb) {
                        const int4 cl = __ldg(&cells[xb + x]);
                        const uint32_t c0 = (uint32_t)cl.x & ~31u, end = (uint32_t)cl.x + (uint32_t)cl.y;
                        cnt[i] = (end - c0 + kCh - 1) / kCh;
                    }
                    sum += cnt[i];
                }
                uint32_t tot;
                uint32_t ex = block_excl_scan(S, sum, &tot);
#pragma unroll
                for (int i = 0; i < PT; i++) {
                    const uint32_t x = threadIdx.x * PT + i;
                    if (x < nbb) S.plan[x] = ex;
                    ex += cnt[i];
                }
                if (threadIdx.x == 0) S.plan[nbb] = tot;
            }
            __syncthreads();
            const uint32_t C = S.plan[nbb];
            // chunk c of the batch -> stage (base + c) % kRingS, by whichever thread issues it
            auto issue = [&](uint32_t c) {
                int lo = 0, hi = (int)nbb;  // largest x with plan[x] <= c
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (S.plan[mid] <= c) lo = mid; else hi = mid;
                }
                const int4 cl = __ldg(&cells[xb + lo]);
                const uint32_t end = (uint32_t)cl.x + (uint32_t)cl.y;
                const uint32_t c0 = ((uint32_t)cl.x & ~31u) + (c - S.plan[lo]) * (uint32_t)kCh;
                const uint32_t b1 = min(min(c0 + (uint32_t)kCh, (end + 3u) & ~3u), nal);
                const uint32_t n = b1 > c0 ? b1 - c0 : 0u;
                const int slot = (int)((base + c) % kRingS);
                unsigned long long *bar = &S.mbar[slot];
                fence_proxy_async();
                mbar_arrive_tx(bar, n * (MT + 4));
                if (n) {
                    bulk_g2s(stc + (size_t)slot * kCh * MT, A.codes_rot + (size_t)c0 * MT, n * MT, bar);
                    bulk_g2s(stp + (size_t)slot * kCh, A.pterm + c0, n * 4, bar);
                }
            };
            if (threadIdx.x == 0)
                for (uint32_t c = 0; c < C && c < (uint32_t)kRingS; c++) issue(c);
            uint32_t x = 0;  // this warp's cell cursor
            for (uint32_t c = 0; c < C; c++) {
                const uint32_t gc = base + c;
                const int slot = (int)(gc % kRingS);
                PROF(PH_BWAIT);
                mbar_wait(&S.mbar[slot], (gc / kRingS) & 1u);
                PROF(PH_BSCORE);
                while (S.plan[x + 1] <= c) x++;
                const int4 cl = __ldg(&cells[xb + x]);
                const uint32_t lst = (uint32_t)cl.x, end = lst + (uint32_t)cl.y;
                const float cb = __int_as_float(cl.z);
                const uint32_t c0 = (lst & ~31u) + (c - S.plan[x]) * (uint32_t)kCh;
                const uint32_t b1 = min(min(c0 + (uint32_t)kCh, (end + 3u) & ~3u), nal);
                uint32_t w[kPer][4];
                float ptv[kPer], acc[kPer];
#pragma unroll
                for (int u = 0; u < kPer; u++) {
                    const int j = warp * kPerW + u * 32 + lane;
                    if constexpr (MT == 16) {
                        const uint4 v = *reinterpret_cast<const uint4 *>(stc + ((size_t)slot * kCh + j) * MT);
                        w[u][0] = v.x; w[u][1] = v.y; w[u][2] = v.z; w[u][3] = v.w;
                    } else {
                        const uint2 v = *reinterpret_cast<const uint2 *>(stc + ((size_t)slot * kCh + j) * MT);
                        w[u][0] = v.x; w[u][1] = v.y; w[u][2] = 0; w[u][3] = 0;
                    }
                    ptv[u] = stp[slot * kCh + j];
                }
                if (c0 + (uint32_t)kCh > b1 && end > b1) {
#pragma unroll
                    for (int u = 0; u < kPer; u++) {
                        const uint32_t e = c0 + warp * kPerW + u * 32 + lane;
                        if (e >= b1 && e < end) {
                            load_code<MT>(A.codes_rot + (size_t)e * MT, w[u], MT);
                            ptv[u] = __ldg(A.pterm + e);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kPer; u++) acc[u] = dist_pt_rep<MT>(tabb, offb, cb, ptv[u], w[u]);
                // admission against min(own k-th key, published bound); ids only for candidates
                const unsigned long long g = S.gthr;
                const unsigned long long bound = wthr < g ? wthr : g;
                const uint32_t bhi = (uint32_t)(bound >> 32);
#pragma unroll
                for (int u = 0; u < kPer; u++) {
                    const uint32_t e = c0 + warp * kPerW + u * 32 + lane;
                    const uint32_t db = canon_bits(acc[u]);
                    bool pass = e >= lst && e < end && db <= bhi;
                    unsigned long long kk = 0;
                    if (pass) {
                        kk = ((unsigned long long)db << 32) | __ldg(A.ids + e);
                        pass = kk < bound;
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, pass);
                    if (pass) tkw[wcnt + __popc(bal & lt)] = kk;
                    wcnt += __popc(bal);
                }
                __syncwarp();
                // release the stage; the last warp through refills it
                if (lane == 0) {
                    __threadfence_block();
                    const uint32_t old = atomicAdd(&S.done[slot], 1u);
                    if (old == NW - 1) {
                        __threadfence_block();
                        S.done[slot] = 0;
                        if (c + kRingS < C) issue(c + kRingS);
                    }
                }
                if (wcnt > (uint32_t)(kCapW - kPerW)) {
                    PROF(PH_BCOMPACT);
                    wthr = warp_topk(tkw, wcnt, k);
                    wcnt = (uint32_t)k;
                    if (lane == 0) atomicMin(&S.gthr, wthr);
                }
            }
            base += C;
            __syncthreads();  // batch done: every stage drained
        }
        // merge: each warp's list (<= k after a final select) and the traversal kernel's list
        PROF(PH_BFIN);
        if (wcnt > (uint32_t)k) {
            warp_topk(tkw, wcnt, k);
            wcnt = (uint32_t)k;
        }
        if (lane == 0) S.wcnt[warp] = wcnt;
        __syncthreads();
        unsigned long long *m = reinterpret_cast<unsigned long long *>(stc);  // the drained ring
        uint32_t off = 0;
        for (int w2 = 0; w2 < NW; w2++) {
            const uint32_t cw = S.wcnt[w2];
            for (uint32_t i = threadIdx.x; i < cw; i += NT) m[off + i] = tkall[w2 * kCapW + i];
            off += cw;
        }
        for (uint32_t i = threadIdx.x; i < n0; i += NT) m[off + i] = A.tk_part[(size_t)qi * k + i];
        off += n0;
        if (threadIdx.x == 0) {
            S.ntk = off;
            S.thr = ~0ull;
        }
        __syncthreads();
        topk_compact(S, m, k);
        const int64_t qo = A.q0 + qi;
        write_topk(S, m, k, A.ncand_q[qi], A.out_d + qo * k, A.out_ids + qo * k, A.out_count + qo);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// Register-pipelined large-cell stream (`cell_flow_kernel`, the default).
//
// A large cell's codes and point terms are read exactly once by exactly one
// lane, so they go from global memory straight into registers (16-/8-byte
// and 4-byte coalesced no-allocate loads, the next chunk's loads issued
// before the current chunk is scored) -- no shared-memory stage, no
// mbarrier, no barrier per chunk.  Every warp walks its own interleaved
// chunks (32 * U consecutive entries starting at a 32-entry boundary, so
// lane l scores entries with index % 32 == l and an entry's summation order
// is the one dist_pt_plain / dist_pt_rep use).
//
// Fold table: `fold[p][c]` is stored at float index c * 64 + (p + d * M) * R
// + g for both d = 0, 1 and every replica g < R = 32 / M (256 bytes per
// codeword).  Lane (x = l % M, g = l / M) reads step i at byte offset
// (c << 8) + (x * R + g) * 4 + i * R * 4: the per-lane part is one constant
// below 128 that a single PRMT merges with the code byte (byte 0 = lane
// constant, byte 1 = code), the per-step part is an immediate -- one PRMT
// and one LDS per lookup, 32 distinct banks per warp-wide lookup.
//
// Admission is a float compare against the distance of the k-th key so far;
// only warps holding a passing lane enter the append path (one ballot per
// entry slot, ONE shared-memory atomicAdd per warp, keys stored raw as
// (canonical distance bits, entry index) -- no id load, no dependent global
// latency).  The ids of the appended entries are gathered by the whole CTA
// once per segment (`convert_raw`), before the radix compaction that orders
// keys by (distance, id).  The stream is cut into segments: a SAFE segment is
// short enough that the buffer could not overflow even if every candidate
// passed (used until a k-th key exists, and to redo a failed segment); an
// OPTIMISTIC segment is sized so its expected admissions (k / seen per
// candidate on unordered data) fill a third of the free space, and at most
// quadruples the entries seen so the bound keeps tightening.  An append past
// the buffer raises `overflow`: the segment's appends are rolled back and
// its head is redone as a safe segment, so any input order is answered
// exactly.  The buffer is radix-compacted to k between segments.
// Checked build (-DBPQ_CHECKED, csrc/build_checked.sh): every index the stream kernel forms is tested
// against its array's bound; a violation counts into counter 19 of the diagnostics buffer
// (bpq_debug_set_phase_buffer) instead of touching memory out of range where that is possible.
// compute-sanitizer is closed on the build pool; tests/test_gpu_parity.py runs the small cases of
// tools/sanitize_case.py under this build and requires the counter to stay 0.
constexpr int PROF_CHECK_FAIL = PH_N + 2;
#ifdef BPQ_CHECKED
#define FLOW_CHECK(cond)                                                        \
    do {                                                                        \
        if (!(cond) && A.prof != nullptr) atomicAdd(A.prof + PROF_CHECK_FAIL, 1ull); \
    } while (0)
#else
#define FLOW_CHECK(cond) \
    do {                 \
    } while (0)
#endif

constexpr int kFlowBT = 512;
constexpr int kFlowNWMax = kFlowBT / 32;
constexpr int kFlowSlack = 4096;  // free keys above roundup(k, 256)
#ifndef BPQ_FLOW_AHEAD
#define BPQ_FLOW_AHEAD 0
#endif
constexpr uint32_t kAhead = BPQ_FLOW_AHEAD;  // chunks (per warp) prefetched into L2 beyond the register pipeline
#ifndef BPQ_FLOW_U8
#define BPQ_FLOW_U8 4
#endif
template <int MT>
__host__ __device__ constexpr int flow_u() { return MT == 16 ? 2 : BPQ_FLOW_U8; }  // entries per lane per half chunk

struct __align__(16) FlowSmem {
    uint32_t hist_c[256];
    unsigned long long red[kFlowNWMax];
    unsigned long long tor[kFlowNWMax];
    unsigned long long thr;
    uint32_t ntk;
    int tsel_v;
    uint32_t tcnt;
    unsigned long long tsel_below;
    unsigned long long tkey;
    uint32_t nholes;
    uint32_t overflow;
    uint32_t save[kFlowNWMax][3];  // per-warp cursor at the segment's start
    float per_chunk;               // appends per chunk measured on the last bounded segment (< 0: none yet)
    uint16_t holes[kMaxK];
    int64_t qidx;
    int prof_ph;
    long long prof_t;
};

__device__ __forceinline__ uint2 ldg_stream_u2(const void *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldg_stream_u4(const void *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, bytes a multiple of 16): no
// destination, no completion to wait for -- memory-level depth that costs no registers
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ float ldg_stream_f(const void *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];\n" : "=f"(v) : "l"(p));
    return v;
}
// half a chunk in registers: U entries per lane (codes + point terms)
template <int MT>
struct FlowHalf {
    static constexpr int U = flow_u<MT>();
    uint32_t w[U][MT / 4];
    float pt[U];
};
// the chunk's owning cell and this lane's first entry in the chunk
struct FlowMeta {
    uint32_t e0, lst, cnt;
    float cb;
};

// BT = 512: two CTAs per SM, kFlowSlack free keys.  BT = 320 (BPQ_FLOW_CTAS=3): three CTAs per SM with a
// 512-key slack -- more, shorter segments, a third CTA to cover the per-query serial phases.
template <int MT, int BT, typename KT, typename OffT>
__global__ void __launch_bounds__(BT, BT == 512 ? 2 : 3) cell_flow_kernel(Args<KT, OffT> A) {
    static_assert(MT == 8 || MT == 16, "large-cell stream needs M = 8 or 16");
    constexpr int kFlowNW = BT / 32;
    constexpr int U = flow_u<MT>();
    constexpr int kH = 32 * U;    // entries per half chunk
    constexpr int kCh = 2 * kH;   // entries per chunk
    constexpr int R = 32 / MT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FlowSmem &S = *reinterpret_cast<FlowSmem *>(smem_raw);
    float *tab = reinterpret_cast<float *>(smem_raw + ((sizeof(FlowSmem) + 15) & ~(size_t)15));  // [K][64]
    unsigned long long *tk = reinterpret_cast<unsigned long long *>(smem_raw + A.tk_off);
    const int K = A.K, k = A.k;
    const uint32_t cap = (uint32_t)A.tkcap;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the lane's constant part of every table offset (< 128), merged under the code byte by PRMT
    const uint32_t lane_b = (uint32_t)(((lane % MT) * R + (lane / MT) % R) * 4);
    const char *tabb = reinterpret_cast<const char *>(tab);
    bool first = true;
    unsigned int qnext = 0;  // thread 0: the next query ticket
#ifdef BPQ_PHASE_PROF
    if (threadIdx.x == 0) {
        S.prof_ph = PH_IDLE;
        S.prof_t = clock64();
    }
#endif
    for (;;) {
        PROF(PH_BPRO);
        __syncthreads();  // the previous query's table / buffer readers are done
        if (threadIdx.x == 0) {
            // (the ticket for the query after this one was drawn while the last one streamed)
            const unsigned int c = first ? atomicAdd(A.counter, 1u) : qnext;
            S.qidx = c < *A.bigq_count ? (int64_t)A.bigq_list[c] : (int64_t)-1;
        }
        first = false;
        __syncthreads();
        const int64_t qi = S.qidx;
        if (qi < 0) {
            PROF(PH_IDLE);
            return;
        }
        // every independent read of the query goes out first (one global round trip instead of four):
        // its fold row, the seed count and first seed keys, the cell count and first cells
        const float *fq = A.fold + (size_t)qi * MT * K;
        constexpr int FV = (MT * 256 + BT - 1) / BT;  // fold values per thread (K <= 256)
        float fv[FV];
#pragma unroll
        for (int i = 0; i < FV; i++) {
            const int x = threadIdx.x + i * BT;  // thread -> (p fastest, c)
            fv[i] = x < MT * K ? __ldg(fq + (x % MT) * K + x / MT) : 0.f;
        }
        const uint32_t n0 = A.tk_n[qi];
        const uint32_t nb = A.big_n[qi];
        const unsigned long long *seeds = A.tk_part + (size_t)qi * k;
        // (speculative: the row is [k]; the split scan has no seeds and passes a null tk_part with n0 = 0)
        const unsigned long long key0 = A.tk_part != nullptr && (int)threadIdx.x < k ? seeds[threadIdx.x] : 0ull;
        const bool packed = A.big_start != nullptr;
        const int4 *cells = A.big_cells + (packed ? (size_t)A.big_start[qi] : (size_t)qi * A.big_cap);
        int4 cl0 = make_int4(0, 0, 0, 0);
        if (!packed && (int)threadIdx.x < A.big_cap) cl0 = __ldg(&cells[threadIdx.x]);  // speculative: row is [big_cap]
        // fold table, doubled and replicated: each quarter warp writes one 128-byte row segment
#pragma unroll
        for (int i = 0; i < FV; i++) {
            const int x = threadIdx.x + i * BT;
            if (x < MT * K) {
                const int p = x % MT, c = x / MT;
                const float v = fv[i];
                float *d0 = tab + c * 64 + p * R;
                FLOW_CHECK(c * 64 + p * R + MT * R + R <= K * 64);
                if constexpr (R == 4) {
                    const float4 vv = make_float4(v, v, v, v);
                    *reinterpret_cast<float4 *>(d0) = vv;
                    *reinterpret_cast<float4 *>(d0 + MT * R) = vv;
                } else {
                    const float2 vv = make_float2(v, v);
                    *reinterpret_cast<float2 *>(d0) = vv;
                    *reinterpret_cast<float2 *>(d0 + MT * R) = vv;
                }
            }
        }
        // the small cells' top-k seeds the buffer; holding k keys, their largest bounds admission
        unsigned long long mx = 0;
        for (uint32_t x = threadIdx.x; x < n0; x += BT) {
            const unsigned long long key = x < (uint32_t)BT ? key0 : seeds[x];
            tk[x] = key;
            mx = key > mx ? key : mx;
        }
        uint32_t csum = 0;  // chunks of this query
        unsigned long long esum = 0;
        for (uint32_t x = threadIdx.x; x < nb; x += BT) {
            const int4 cl = (!packed && x < (uint32_t)BT) ? cl0 : __ldg(&cells[x]);
            csum += ((uint32_t)cl.x + (uint32_t)cl.y - ((uint32_t)cl.x & ~31u) + kCh - 1) / kCh;
            esum += (uint32_t)cl.y;
        }
        if (A.prof != nullptr && esum) atomicAdd(A.prof + PROF_STREAM_CAND, esum);  // diagnostics only
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = y > mx ? y : mx;
            csum += __shfl_xor_sync(0xffffffffu, csum, o);
        }
        if (lane == 0) {
            S.red[warp] = mx;
            S.tor[warp] = csum;
        }
        __syncthreads();
        uint32_t C = 0;
        {
            unsigned long long m = 0;
#pragma unroll
            for (int w2 = 0; w2 < kFlowNW; w2++) {
                m = S.red[w2] > m ? S.red[w2] : m;
                C += (uint32_t)S.tor[w2];
            }
            if (threadIdx.x == 0) {
                S.ntk = n0;
                S.thr = n0 >= (uint32_t)k ? m : ~0ull;
                S.overflow = 0;
                S.per_chunk = -1.f;
            }
        }
        __syncthreads();

        // the warp's position in the cell list: cell cx covers chunks [cpre, cend)
        uint32_t cx = 0xFFFFFFFFu, cpre = 0, cend = 0;
        FlowMeta mn{};  // the located chunk
        auto locate = [&](uint32_t c) {  // c < C, non-decreasing between rewinds
            while (c >= cend) {
                cx++;
                FLOW_CHECK(cx < nb);
                const int4 cl = __ldg(&cells[cx]);
                mn.lst = (uint32_t)cl.x;
                mn.cnt = (uint32_t)cl.y;
                mn.cb = __int_as_float(cl.z);
                cpre = cend;
                cend += (mn.lst + mn.cnt - (mn.lst & ~31u) + kCh - 1) / kCh;
            }
            mn.e0 = (mn.lst & ~31u) + (c - cpre) * (uint32_t)kCh + (uint32_t)lane;
        };
        // optional lookahead cursor (BPQ_FLOW_AHEAD > 0): the chunk kAhead steps after the one being
        // fetched is bulk-prefetched into L2 by TMA.  Measured on B200 at config 4: L2 hit rate 1 % ->
        // 27 %, kernel time unchanged (2.15 ms) -- the stream is not latency-bound -- so it ships off
        uint32_t px = 0xFFFFFFFFu, ppre = 0, pend = 0, plst = 0;
        auto prefetch_chunk = [&](uint32_t c) {  // c < C, non-decreasing between rewinds
            while (c >= pend) {
                px++;
                const int4 cl = __ldg(&cells[px]);
                plst = (uint32_t)cl.x;
                ppre = pend;
                pend += (plst + (uint32_t)cl.y - (plst & ~31u) + kCh - 1) / kCh;
            }
            if (lane == 0) {
                const uint32_t e = (plst & ~31u) + (c - ppre) * (uint32_t)kCh;
                bulk_prefetch_l2(A.codes_rot + (size_t)e * MT, kCh * MT);
                bulk_prefetch_l2(A.pterm + e, kCh * 4);
            }
        };
        auto fetch = [&](FlowHalf<MT> &h, uint32_t e) {
            const uint8_t *pc = A.codes_rot + (size_t)e * MT;
            const float *pp = A.pterm + e;
            FLOW_CHECK((unsigned long long)e + (U - 1) * 32 < (unsigned long long)A.n_local + kStreamPad);
#pragma unroll
            for (int u = 0; u < U; u++) {
                if constexpr (MT == 16) {
                    const uint4 v = ldg_stream_u4(pc + (size_t)u * 32 * MT);
                    h.w[u][0] = v.x; h.w[u][1] = v.y; h.w[u][2] = v.z; h.w[u][3] = v.w;
                } else {
                    const uint2 v = ldg_stream_u2(pc + (size_t)u * 32 * MT);
                    h.w[u][0] = v.x; h.w[u][1] = v.y;
                }
                h.pt[u] = ldg_stream_f(pp + u * 32);
            }
        };
        // score half a chunk: entries e + 32 u of cell (lst, cnt, cb).  Candidates at or under the
        // bound's distance are appended RAW, as (distance bits, entry index): no id load and no
        // dependent latency here; convert_raw() swaps in the ids once per segment
        auto score = [&](const FlowHalf<MT> &h, uint32_t e, uint32_t lst, uint32_t cnt, float cb, float thrf,
                         bool bounded) {
            float acc[U];
            bool pass[U], any = false;
#pragma unroll
            for (int u = 0; u < U; u++) {
                float v[MT];
#pragma unroll
                for (int i = 0; i < MT; i++) {
                    // byte 0 = lane constant, byte 1 = code byte i, bytes 2-3 = 0
                    const uint32_t off = __byte_perm(h.w[u][i >> 2], lane_b, 0x6504u | ((uint32_t)(i & 3) << 4));
                    FLOW_CHECK(off + i * R * 4 + 4 <= (uint32_t)K * 256u);
                    v[i] = *reinterpret_cast<const float *>(tabb + off + i * R * 4);
                }
                acc[u] = __fadd_rn(__fadd_rn(tree_sum<MT>(v), h.pt[u]), cb);
                pass[u] = (e + u * 32 - lst) < cnt && acc[u] <= thrf;  // negative sums clamp to 0 below
                any |= pass[u];
            }
            if (bounded) {
                // a k-th key exists: passes are rare (about k / seen per entry), so each passing lane
                // appends on its own -- a not-taken branch per slot is all the common case pays
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (pass[u]) {
                        const uint32_t idx = atomicAdd(&S.ntk, 1u);
                        const float a = acc[u] < 0.f ? 0.f : acc[u];
                        if (idx < cap) tk[idx] = ((unsigned long long)canon_bits(a) << 32) | (e + u * 32);
                        else S.overflow = 1u;
                    }
                }
            } else if (__any_sync(0xffffffffu, any)) {
                // no bound yet: every valid entry passes; one atomicAdd per warp
                const unsigned lt = (1u << lane) - 1u;
                unsigned bal[U];
                uint32_t tot = 0;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    bal[u] = __ballot_sync(0xffffffffu, pass[u]);
                    tot += __popc(bal[u]);
                }
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&S.ntk, tot);
                base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (pass[u]) {
                        const uint32_t idx = base + __popc(bal[u] & lt);
                        const float a = acc[u] < 0.f ? 0.f : acc[u];
                        if (idx < cap) tk[idx] = ((unsigned long long)canon_bits(a) << 32) | (e + u * 32);
                        else S.overflow = 1u;
                    }
                    base += __popc(bal[u]);
                }
            }
        };
        // raw keys [from, ntk) -> (distance bits, id): one parallel gather per segment
        auto convert_raw = [&](uint32_t from) {
            const uint32_t to = min(S.ntk, cap);
            for (uint32_t x = from + threadIdx.x; x < to; x += BT) {
                const unsigned long long kk = tk[x];
                FLOW_CHECK((uint32_t)kk < A.n_local);
                tk[x] = (kk & 0xFFFFFFFF00000000ull) | __ldg(A.ids + (uint32_t)kk);
            }
            __syncthreads();
        };
        // the warp's chunks of [sb, se): sb + warp, + kFlowNW, ...; the next chunk's halves are
        // fetched while the current chunk's other half is scored
        auto run_segment = [&](uint32_t sb, uint32_t se) {
            const uint32_t thi = (uint32_t)(S.thr >> 32);  // the bound's distance; equal distances pass
            const bool bounded = thi < 0x7F800000u;
            const float thrf = bounded ? __uint_as_float(thi) : INFINITY;
            uint32_t c = sb + (uint32_t)warp;
            if (c >= se) return;
            FlowHalf<MT> ha, hb;
            locate(c);
            FlowMeta mc = mn;
            fetch(ha, mc.e0);
            fetch(hb, mc.e0 + kH);
            for (;;) {
                const uint32_t cn = c + kFlowNW;
                const bool more = cn < se;
                if (kAhead > 0 && cn + kAhead * kFlowNW < C) prefetch_chunk(cn + kAhead * kFlowNW);  // may run past se
                score(ha, mc.e0, mc.lst, mc.cnt, mc.cb, thrf, bounded);
                if (more) {
                    locate(cn);
                    fetch(ha, mn.e0);
                }
                score(hb, mc.e0 + kH, mc.lst, mc.cnt, mc.cb, thrf, bounded);
                if (!more) break;
                fetch(hb, mn.e0 + kH);
                mc = mn;
                c = cn;
            }
        };

        if (threadIdx.x == 0) qnext = atomicAdd(A.counter, 1u);  // latency hidden under the stream
        uint32_t pos = 0;
        while (pos < C) {
            PROF(PH_BSCORE);
            const uint32_t n_start = S.ntk;  // <= k (compacted) or the seed keys
            const uint32_t free_keys = cap - n_start;
            const uint32_t safe = free_keys / (uint32_t)kCh;
            uint32_t len = safe;
            const bool bounded = S.thr != ~0ull;
            if (bounded) {
                // Optimistic length: fill about half the free space at the append rate the last bounded
                // segment MEASURED (the bound only tightens, but cell lists are not exchangeable: later
                // cells can be better); before any measurement, k / seen per entry on unordered data.
                // A segment boundary costs a barrier pair, a compaction and a cold pipeline, so segments
                // also grow by at most flow_growth x the chunks seen.
                unsigned long long opt;
                const float per_chunk = S.per_chunk;  // (kept in shared memory: nothing extra lives across the stream loop)
                if (per_chunk >= 0.f) opt = (unsigned long long)(0.5f * (float)free_keys / fmaxf(per_chunk, 1e-3f));
                else opt = (unsigned long long)pos * free_keys / (3ull * (uint32_t)k);
                if (A.flow_growth > 0 && pos > 0 && opt > (unsigned long long)A.flow_growth * pos)
                    opt = (unsigned long long)A.flow_growth * pos;
                if (opt > len) len = opt > (unsigned long long)(C - pos) ? C - pos : (uint32_t)opt;
            }
            if (len > C - pos) len = C - pos;
            if (lane == 0) {  // the cursor at the segment's start, for a roll-back
                S.save[warp][0] = cx;
                S.save[warp][1] = cpre;
                S.save[warp][2] = cend;
            }
            __syncthreads();  // everyone has read ntk / thr / overflow state
            run_segment(pos, pos + len);
            __syncthreads();
            if (S.overflow) {
                // more admissions than the buffer holds: roll the segment back, redo its head safely
                const float seen_rate = (float)free_keys / (float)len;  // at least this many per chunk
                __syncthreads();
                if (threadIdx.x == 0) {
                    S.ntk = n_start;
                    S.overflow = 0;
                    if (A.prof != nullptr) atomicAdd(A.prof + PROF_CHECK_FAIL + 1, 1ull);  // roll-backs (diagnostics)
                }
                cx = S.save[warp][0];
                cpre = S.save[warp][1];
                cend = S.save[warp][2];
                if (cx != 0xFFFFFFFFu) {  // the cell under the cursor again
                    const int4 cl = __ldg(&cells[cx]);
                    mn.lst = (uint32_t)cl.x;
                    mn.cnt = (uint32_t)cl.y;
                    mn.cb = __int_as_float(cl.z);
                }
                px = 0xFFFFFFFFu;
                ppre = pend = 0;
                len = min(safe, len);
                __syncthreads();
                run_segment(pos, pos + len);
                __syncthreads();
                if (threadIdx.x == 0)
                    S.per_chunk = fmaxf(seen_rate, (float)(min(S.ntk, cap) - n_start) / (float)len);
            } else if (bounded) {
                if (threadIdx.x == 0) S.per_chunk = (float)(S.ntk - n_start) / (float)len;
            }
            convert_raw(n_start);  // (ends in a barrier: per_chunk is visible to the next segment's sizing)
            pos += len;
            if (pos < C) {
                PROF(PH_BCOMPACT);
                topk_compact<BT>(S, tk, k);
            }
        }
        PROF(PH_BFIN);
        topk_compact<BT>(S, tk, k);
        const int64_t qo = A.q0 + qi;
        write_topk<BT>(S, tk, k, A.ncand_q[qi], A.out_d + qo * k, A.out_ids + qo * k, A.out_count + qo);
    }
}

// the large-cell stream over the queries the traversal passes handed over
template <int MT>
int launch_big_one(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget, int32_t k,
                   const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids, int32_t *out_count,
                   cudaStream_t stream) {
    if constexpr (!rep_fold<MT>()) {
        return BPQ_OK;
    } else {
        Args<float, uint32_t> A{};
        fill_args<BPQ_ENGINE_FBPQ, MT>(A, ix, queries, q0, nq, budget, k, ws, out_dist, out_ids, out_count,
                                       nullptr, nullptr);
        if (A.big_cells == nullptr) return BPQ_OK;
        // default: the register-pipelined stream (cell_flow_kernel); BPQ_STREAM_TMA=1 selects the
        // TMA-ring kernels below for A/B runs
        if (getenv("BPQ_STREAM_TMA") == nullptr) {
            A.flow_growth = getenv("BPQ_FLOW_GROWTH") ? atoi(getenv("BPQ_FLOW_GROWTH")) : 3;  // env: A/B experiments
            // Three 320-thread CTAs per SM (512-key slack) for mid budgets and k <= 256: the third CTA
            // covers the per-query serial phases (config 4: 2.08 -> 1.97 ms, with M = 16 2.89 -> 2.79, at
            // k = 10 1.85 -> 1.66; configs 1 and 3 unchanged within 2 %).  Long cell lists roll the small
            // buffer back too often (config 1 at L = 100,000: 3.1 -> 6.4 ms) and short queries have too few
            // chunks per segment (L = 1,000: 0.47 -> 0.51 ms): those keep two 512-thread CTAs and the
            // 4096-key slack.  BPQ_FLOW_CTAS=2 / 3 forces either.
            const char *force = getenv("BPQ_FLOW_CTAS");
            const bool three = force != nullptr ? atoi(force) == 3 : (budget >= 4096 && budget <= 32768 && k <= 256);
            const int bt = three ? 320 : kFlowBT;
            A.tkcap = ((k + 255) & ~255) + (three ? 512 : kFlowSlack);
            A.tk_off = (int)((((sizeof(FlowSmem) + 15) & ~(size_t)15) + (size_t)64 * ix.K * 4 + 15) & ~(size_t)15);
            const size_t smem = (size_t)A.tk_off + (size_t)A.tkcap * 8;
            auto kfn = three ? cell_flow_kernel<MT, 320, float, uint32_t> : cell_flow_kernel<MT, kFlowBT, float, uint32_t>;
            static bool fattr = false;
            if (!fattr) {
                int dev = 0, optin = 0;
                BPQ_CUDA_TRY(cudaGetDevice(&dev));
                BPQ_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
                BPQ_CUDA_TRY(cudaFuncSetAttribute(cell_flow_kernel<MT, 320, float, uint32_t>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
                BPQ_CUDA_TRY(cudaFuncSetAttribute(cell_flow_kernel<MT, kFlowBT, float, uint32_t>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
                fattr = true;
            }
            int occ = 0;
            BPQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, bt, smem));
            if (occ < 1) return fail(BPQ_ERR_UNSUPPORTED, "large-cell stream shared memory does not fit on an SM");
            BPQ_CUDA_TRY(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned int), stream));
            kfn<<<occ * num_sms(), bt, smem, stream>>>(A);
            BPQ_CUDA_TRY(cudaGetLastError());
            return BPQ_OK;
        }
        // the warp-independent variant measured slower (per-warp compactions, looser
        // admission); it stays available for A/B runs
        constexpr int BT = 512;
        const bool warp_mode = k <= kStreamMaxK && getenv("BPQ_STREAM_WARP") != nullptr;
        size_t smem;
        if (warp_mode) {
            A.tkcap = kCapW;
            A.tk_off = (int)((((sizeof(StreamSmem) + 15) & ~(size_t)15) + (size_t)32 * ix.K * 4 + 15) & ~(size_t)15);
            smem = (size_t)A.tk_off + (size_t)NW * kCapW * 8 + ring_bytes<MT>();
        } else {
            A.tkcap = ((k + 255) & ~255) + 2 * ring_chunk<MT>();  // compaction once per >= one chunk of offers
            A.tk_off = (int)((((sizeof(ScanSmem<BT>) + 15) & ~(size_t)15) + (size_t)32 * ix.K * 4 + 15) & ~(size_t)15);
            smem = (size_t)A.tk_off + (size_t)A.tkcap * 8 + ring_bytes<MT>();
        }
        auto kfn = warp_mode ? big_stream_kernel<MT, float, uint32_t> : big_scan_kernel<MT, BT, float, uint32_t>;
        const int threads = warp_mode ? NT : BT;
        static bool attr = false;
        if (!attr) {
            int dev = 0, optin = 0;
            BPQ_CUDA_TRY(cudaGetDevice(&dev));
            BPQ_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            BPQ_CUDA_TRY(cudaFuncSetAttribute(big_stream_kernel<MT, float, uint32_t>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
            BPQ_CUDA_TRY(cudaFuncSetAttribute(big_scan_kernel<MT, BT, float, uint32_t>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
            attr = true;
        }
        int occ = 0;
        BPQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem));
        if (occ < 1) return fail(BPQ_ERR_UNSUPPORTED, "large-cell stream shared memory does not fit on an SM");
        BPQ_CUDA_TRY(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned int), stream));
        kfn<<<occ * num_sms(), threads, smem, stream>>>(A);
        BPQ_CUDA_TRY(cudaGetLastError());
        return BPQ_OK;
    }
}

}  // namespace
}  // namespace bpq
