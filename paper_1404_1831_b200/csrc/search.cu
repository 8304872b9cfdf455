// Fused multi-sequence traversal + PQ-code scan + top-k, one CTA per query.
//
// Replaces the per-query chain traverse -> kernels.traverse_cells ->
// kernels.scan_{global,tables,local} -> select_top of the reference
// (multi_index.py:302-339, kernels/numba_backend.py:11-246).
//
// Traversal.  The reference pops cells one at a time from a min-heap keyed
// (key = f64(sr1[a]) + f64(sr2[b]), oi, oj) and stops after the first
// non-empty cell that brings the collected entry count to >= L.  Because
// that total order is a linear extension of the grid dominance order, the
// visited set is exactly "all cells whose (key, oi, oj) precedes the cutoff
// cell".  We find it with parallel "bands" instead of a
// sequential heap:
//   * pick a key threshold tau (bisection on the staircase cell count
//     C(tau) = sum_a #{b : key(a,b) <= tau}, one binary search per row);
//   * enumerate the band of cells with tauLo < key <= tau (flattened over
//     the 256 threads) and read their entry counts from the cell table;
//   * if the band keeps the running total < L, every band cell is visited:
//     scan it and continue; otherwise the cutoff lies inside the band and a
//     weighted radix select over the 96-bit key (f64 key bits, oi*T+oj),
//     finished by a shared-memory bitonic sort, finds the exact cutoff.
// The per-row staircase state (rowB) replaces the reference's T*T popped
// bitmap (numba_backend.py:25).
//
// Scan.  Visited cells are scanned from a list in chunks of 256 cells; the
// chunk's entries are flattened over the CTA so a thread handles one
// candidate (code + id loads, per-part table lookups).  Arithmetic follows
// the reference's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction), so a candidate's distance is bit-exact
// given the same per-query tables.
//
// Top-k.  Candidates below the current k-th best key ((dist bits << 32) |
// id, i.e. (dist asc, id asc) as select_top, multi_index.py:326-339) are
// appended to a shared-memory buffer that is bitonic-compacted to k when
// full.
#include <cub/device/device_radix_sort.cuh>

#include <cfloat>
#include <cmath>

#include "bpq_internal.cuh"

namespace bpq {
namespace {

constexpr int NT = kSearchThreads;
constexpr int NW = NT / 32;
constexpr int ENGINE_TRAVERSE = 3;
constexpr int kTabFloats = 4096;  // >= 16 parts * 256 codewords, >= kMaxDim

struct __align__(16) Smem {
    unsigned long long tk[kTopkBuf];
    float tab[kTabFloats];
    uint32_t cpre[NT + 1];
    int32_t coi[NT];
    int32_t coj[NT];
    uint32_t cstart[NT];
    float cbase[NT];
    unsigned long long skey[kSortCap];
    uint32_t slin[kSortCap];
    uint16_t sidx[kSortCap];
    uint32_t hist_w[256];
    uint32_t hist_c[256];
    unsigned long long red[NW];
    uint32_t wscan[NW];
    unsigned long long thr;
    uint32_t ntk;
    uint32_t nlist;
    int64_t qidx;
    float qnorm;
    int sel_v;
    unsigned long long sel_below;
    int arows;
    int err;
    unsigned long long cut_key;
};

template <typename KT, typename OffT>
struct Args {
    int T, D, dh, ds, K;
    const float *c1, *c2, *cn1, *cn2;
    const OffT *loff, *goff;
    bool sharded;
    const uint32_t *ids;
    const uint8_t *codes;
    const float *books, *fine_norms, *cross1, *cross2, *bank1, *bank2;
    double rho;
    unsigned long long n_global;
    const float *queries;
    int64_t q0, nq;
    const float *dots1, *dots2;
    const KT *sr1, *sr2;
    const int32_t *ord1, *ord2;
    long long L;
    int k;
    float *out_d;
    uint32_t *out_ids;
    int32_t *out_count;
    int64_t *out_ncand;
    int64_t *out_popped;
    unsigned int *counter;
    char *scratch;
    size_t stride;
    // traversal-only outputs (stage API)
    unsigned long long *tv_key;
    uint32_t *tv_lin;
    int64_t *tv_start, *tv_end;
    unsigned long long *tv_n;
};

// ---------------------------------------------------------------- block utils
__device__ __forceinline__ unsigned long long block_sum_u64(Smem &S, unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long s = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) s += S.red[w];
    return s;
}

__device__ __forceinline__ float block_sum_f32_ordered(Smem &S, float v) {
    // deterministic: warp tree then warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = __float_as_uint(v);
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; w++) s += __uint_as_float((uint32_t)S.red[w]);
    return s;
}

// exclusive scan of one u32 per thread; returns exclusive prefix, *total = sum
__device__ __forceinline__ uint32_t block_excl_scan(Smem &S, uint32_t v, uint32_t *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) S.wscan[w] = x;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        uint32_t s = S.wscan[i];
        if (i < w) off += s;
        tot += s;
    }
    *total = tot;
    return off + x - v;
}

__device__ __forceinline__ void bitonic_sort_u64(unsigned long long *a, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool up = (i & k) == 0;
                    unsigned long long x = a[i], y = a[ixj];
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// sort (skey, slin) ascending carrying sidx; n power of two
__device__ __forceinline__ void bitonic_sort_cells(Smem &S, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool up = (i & k) == 0;
                    unsigned long long ka = S.skey[i], kb = S.skey[ixj];
                    uint32_t la = S.slin[i], lb = S.slin[ixj];
                    bool gt = (ka > kb) || (ka == kb && la > lb);
                    if (gt == up) {
                        S.skey[i] = kb;
                        S.skey[ixj] = ka;
                        S.slin[i] = lb;
                        S.slin[ixj] = la;
                        uint16_t t = S.sidx[i];
                        S.sidx[i] = S.sidx[ixj];
                        S.sidx[ixj] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t canon_bits(float d) {
    uint32_t b = __float_as_uint(d);
    return b == 0x80000000u ? 0u : b;  // -0.0 ties +0.0 as in numpy's lexsort
}

template <typename KT>
__device__ __forceinline__ double kd(const KT *p, int i) {
    return (double)__ldg(p + i);
}

// ------------------------------------------------------------ code loading
template <int M>
__device__ __forceinline__ void load_code(const uint8_t *p, uint32_t (&w)[4]) {
    if constexpr (M == 16) {
        uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else if constexpr (M == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = v.x; w[1] = v.y;
    } else if constexpr (M % 4 == 0) {
#pragma unroll
        for (int i = 0; i < M / 4; i++) w[i] = __ldg(reinterpret_cast<const uint32_t *>(p) + i);
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) w[i] = 0;
#pragma unroll
        for (int i = 0; i < M / 2; i++) {
            uint32_t h = __ldg(reinterpret_cast<const uint16_t *>(p) + i);
            w[i >> 1] |= h << ((i & 1) * 16);
        }
    }
}

__device__ __forceinline__ int code_at(const uint32_t (&w)[4], int p) {
    return (w[p >> 2] >> ((p & 3) * 8)) & 0xFF;
}

// --------------------------------------------------- per-candidate distances
template <int M, typename KT, typename OffT>
__device__ __forceinline__ float dist_fbpq(const Args<KT, OffT> &A, const Smem &S, int oi, int oj,
                                           float cbase, const uint32_t (&w)[4]) {
    constexpr int M2 = M / 2;
    const int K = A.K;
    float acc = cbase;
#pragma unroll
    for (int p = 0; p < M2; p++) {
        int c = code_at(w, p);
        float x = __ldg(A.cross1 + ((size_t)oi * M2 + p) * K + c);
        acc = __fadd_rn(acc, __fadd_rn(S.tab[p * K + c], __fmul_rn(2.f, x)));
    }
#pragma unroll
    for (int p = M2; p < M; p++) {
        int c = code_at(w, p);
        float x = __ldg(A.cross2 + ((size_t)oj * M2 + (p - M2)) * K + c);
        acc = __fadd_rn(acc, __fadd_rn(S.tab[p * K + c], __fmul_rn(2.f, x)));
    }
    if (acc < 0.f) acc = 0.f;  // numba_backend.py:241-242
    return acc;
}

// Multi-D-ADC explicit reconstruction (ENGINE 0) and HBPQ local books
// (ENGINE 2): e = q_h - c_h[row] (one rounding, multi_index.py:345-346),
// d = e - book, acc += d*d sequentially (numba_backend.py:165-176, 198-210).
template <int ENGINE, int M, typename KT, typename OffT>
__device__ __forceinline__ float dist_recon(const Args<KT, OffT> &A, const Smem &S, int oi, int oj,
                                            const uint32_t (&w)[4]) {
    constexpr int M2 = M / 2;
    const int K = A.K, ds = A.ds, dh = A.dh;
    float acc = 0.f;
#pragma unroll
    for (int p = 0; p < M; p++) {
        const int hp = p < M2 ? p : p - M2;
        const int row = p < M2 ? oi : oj;
        const float *cr = (p < M2 ? A.c1 : A.c2) + (size_t)row * dh + hp * ds;
        const float *qv = S.tab + (p < M2 ? 0 : dh) + hp * ds;
        const int c = code_at(w, p);
        const float *bk;
        if constexpr (ENGINE == BPQ_ENGINE_HBPQ)
            bk = (p < M2 ? A.bank1 : A.bank2) + (((size_t)row * M2 + hp) * K + c) * ds;
        else
            bk = A.books + ((size_t)p * K + c) * ds;
        for (int u = 0; u < ds; u++) {
            float e = __fsub_rn(qv[u], __ldg(cr + u));
            float d = __fsub_rn(e, __ldg(bk + u));
            acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
    }
    return acc;
}

// ------------------------------------------------------------ top-k buffer
__device__ __forceinline__ void topk_compact(Smem &S, int k) {
    uint32_t n = S.ntk;
    for (int i = threadIdx.x; i < kTopkBuf; i += NT)
        if (i >= (int)n) S.tk[i] = ~0ull;
    __syncthreads();
    bitonic_sort_u64(S.tk, kTopkBuf);
    if (threadIdx.x == 0) {
        if ((int)n > k) {
            S.ntk = k;
            S.thr = S.tk[k - 1];
        }
    }
    __syncthreads();
}

// ------------------------------------------------------- per-query context
template <int ENGINE, int M, typename KT, typename OffT>
struct Query {
    const Args<KT, OffT> &A;
    Smem &S;
    int64_t qi;
    const KT *sr1, *sr2;
    const int32_t *o1, *o2;
    const float *d1, *d2;
    int T;
    unsigned long long ncand;  // uniform across the CTA
    unsigned long long popped;

    __device__ Query(const Args<KT, OffT> &a, Smem &s, int64_t q) : A(a), S(s), qi(q) {
        T = A.T;
        sr1 = A.sr1 + q * T;
        sr2 = A.sr2 + q * T;
        o1 = A.ord1 + q * T;
        o2 = A.ord2 + q * T;
        d1 = A.dots1 ? A.dots1 + q * T : nullptr;
        d2 = A.dots2 ? A.dots2 + q * T : nullptr;
        ncand = 0;
        popped = 0;
    }

    __device__ __forceinline__ double key(int a, int b) const { return kd(sr1, a) + kd(sr2, b); }

    __device__ __forceinline__ unsigned long long lin_of(int a, int b) const {
        return (unsigned long long)__ldg(o1 + a) * (unsigned long long)T + (unsigned)__ldg(o2 + b);
    }

    // 12-byte composite sort key digit d (0 = most significant)
    __device__ __forceinline__ int digit(int d, int4 e) const {
        int a = (unsigned)e.x >> 16, b = e.x & 0xFFFF;
        if (d < 8) {
            unsigned long long kb = (unsigned long long)__double_as_longlong(key(a, b));
            return (int)((kb >> (56 - 8 * d)) & 0xFF);
        }
        unsigned long long lin = lin_of(a, b);
        return (int)((lin >> (24 - 8 * (d - 8))) & 0xFF);
    }

    // Visit a list of cells: scan their entries (search) or record them
    // (traversal stage).  filt_d < 0: all cells; else only cells whose digit
    // filt_d is < filt_v.
    __device__ void emit(const int4 *list, int n, int filt_d, int filt_v) {
        for (int base = 0; base < n; base += NT) {
            int c = base + threadIdx.x;
            uint32_t lc = 0;
            int oi = 0, oj = 0;
            uint32_t lst = 0;
            float cb = 0.f;
            int a = 0, b = 0;
            if (c < n) {
                int4 e = list[c];
                bool pass = filt_d < 0 || digit(filt_d, e) < filt_v;
                if (pass) {
                    a = (unsigned)e.x >> 16;
                    b = e.x & 0xFFFF;
                    oi = __ldg(o1 + a);
                    oj = __ldg(o2 + b);
                    lst = (uint32_t)e.z;
                    lc = (uint32_t)e.w;
                    if constexpr (ENGINE == ENGINE_TRAVERSE) {
                        unsigned long long pos = atomicAdd(A.tv_n, 1ull);
                        A.tv_key[pos] = (unsigned long long)__double_as_longlong(key(a, b));
                        A.tv_lin[pos] = (uint32_t)oi * (uint32_t)T + (uint32_t)oj;
                        A.tv_start[pos] = (int64_t)lst;
                        A.tv_end[pos] = (int64_t)lst + lc;
                    }
                    if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                        // cell_base, numba_backend.py:232
                        float s = __fadd_rn(__ldg(d1 + oi), __ldg(d2 + oj));
                        float t0 = __fsub_rn(S.qnorm, __fmul_rn(2.f, s));
                        cb = __fadd_rn(__fadd_rn(t0, __ldg(A.cn1 + oi)), __ldg(A.cn2 + oj));
                    }
                }
            }
            if constexpr (ENGINE == ENGINE_TRAVERSE) {
                continue;
            } else {
                uint32_t E;
                uint32_t ex = block_excl_scan(S, lc, &E);
                S.cpre[threadIdx.x] = ex;
                S.coi[threadIdx.x] = oi;
                S.coj[threadIdx.x] = oj;
                S.cstart[threadIdx.x] = lst;
                S.cbase[threadIdx.x] = cb;
                __syncthreads();
                ncand += E;
                for (uint32_t e0 = 0; e0 < E; e0 += NT) {
                    uint32_t e = e0 + threadIdx.x;
                    if (e < E) {
                        int lo = 0, hi = NT;
                        while (hi - lo > 1) {
                            int mid = (lo + hi) >> 1;
                            if (S.cpre[mid] <= e) lo = mid; else hi = mid;
                        }
                        uint32_t entry = S.cstart[lo] + (e - S.cpre[lo]);
                        uint32_t w[4];
                        load_code<M>(A.codes + (size_t)entry * M, w);
                        float dist;
                        if constexpr (ENGINE == BPQ_ENGINE_FBPQ)
                            dist = dist_fbpq<M>(A, S, S.coi[lo], S.coj[lo], S.cbase[lo], w);
                        else
                            dist = dist_recon<ENGINE, M>(A, S, S.coi[lo], S.coj[lo], w);
                        uint32_t id = __ldg(A.ids + entry);
                        unsigned long long kk = ((unsigned long long)canon_bits(dist) << 32) | id;
                        if (kk < S.thr) {
                            uint32_t pos = atomicAdd(&S.ntk, 1u);
                            S.tk[pos] = kk;
                        }
                    }
                    __syncthreads();
                    if (S.ntk > (uint32_t)(kTopkBuf - NT)) topk_compact(S, A.k);
                }
                __syncthreads();
            }
        }
        if constexpr (ENGINE == ENGINE_TRAVERSE) __syncthreads();
    }

    // count of cells with key <= tau; optionally records the per-row bound
    __device__ unsigned long long count_le(double tau, const int32_t *rowB, int32_t *rowNew) {
        unsigned long long cnt = 0;
        const double k0 = kd(sr2, 0);
        for (int a = threadIdx.x; a < T; a += NT) {
            double ka = kd(sr1, a);
            if (!(ka + k0 <= tau)) break;
            int lo = rowB[a], hi = T;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (ka + kd(sr2, mid) <= tau) lo = mid + 1; else hi = mid;
            }
            cnt += lo;
            if (rowNew) rowNew[a] = lo;
        }
        return block_sum_u64(S, cnt);
    }

    // exact cutoff inside the final band (weighted select, then smem sort)
    __device__ void final_select(int4 *cur, int4 *other, int n, unsigned long long need) {
        for (int d = 0;; d++) {
            if (n <= kSortCap) {
                int P = 1;
                while (P < n) P <<= 1;
                for (int c = threadIdx.x; c < P; c += NT) {
                    if (c < n) {
                        int4 e = cur[c];
                        int a = (unsigned)e.x >> 16, b = e.x & 0xFFFF;
                        S.skey[c] = (unsigned long long)__double_as_longlong(key(a, b));
                        S.slin[c] = (uint32_t)lin_of(a, b);
                    } else {
                        S.skey[c] = ~0ull;
                        S.slin[c] = ~0u;
                    }
                    S.sidx[c] = (uint16_t)c;
                }
                __syncthreads();
                bitonic_sort_cells(S, P);
                // first sorted position where the running count reaches need
                if (threadIdx.x == 0) S.nlist = 0xFFFFFFFFu;
                unsigned long long run = 0;
                for (int base = 0; base < n; base += NT) {
                    int pidx = base + threadIdx.x;
                    uint32_t g = pidx < n ? (uint32_t)cur[S.sidx[pidx]].y : 0u;
                    uint32_t tot;
                    uint32_t ex = block_excl_scan(S, g, &tot);
                    if (pidx < n && run + ex < need && run + ex + g >= need) S.nlist = pidx;
                    run += tot;
                    __syncthreads();
                    if (S.nlist != 0xFFFFFFFFu) break;
                }
                __syncthreads();
                int cut = (int)S.nlist;  // always found: total >= need
                if (cut == -1) cut = n - 1;
                if (threadIdx.x == 0) S.cut_key = S.skey[cut];
                for (int c = threadIdx.x; c <= cut; c += NT) other[c] = cur[S.sidx[c]];
                __syncthreads();
                emit(other, cut + 1, -1, 0);
                return;
            }
            for (int i = threadIdx.x; i < 256; i += NT) {
                S.hist_w[i] = 0;
                S.hist_c[i] = 0;
            }
            __syncthreads();
            for (int c = threadIdx.x; c < n; c += NT) {
                int4 e = cur[c];
                int dg = digit(d, e);
                atomicAdd(&S.hist_w[dg], (uint32_t)e.y);
                atomicAdd(&S.hist_c[dg], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long run = 0;
                int v = 255;
                for (int i = 0; i < 256; i++) {
                    if (run + S.hist_w[i] >= need) {
                        v = i;
                        break;
                    }
                    run += S.hist_w[i];
                }
                S.sel_v = v;
                S.sel_below = run;
                S.nlist = 0;
            }
            __syncthreads();
            const int v = S.sel_v;
            const unsigned long long below = S.sel_below;
            if (below > 0 || v > 0) emit(cur, n, d, v);
            need -= below;
            for (int c = threadIdx.x; c < n; c += NT) {
                int4 e = cur[c];
                if (digit(d, e) == v) other[atomicAdd(&S.nlist, 1u)] = e;
            }
            __syncthreads();
            n = (int)S.nlist;
            int4 *t = cur;
            cur = other;
            other = t;
            __syncthreads();
        }
    }

    __device__ void run() {
        char *scr = A.scratch + (size_t)blockIdx.x * A.stride;
        int32_t *rowB = reinterpret_cast<int32_t *>(scr);
        int32_t *rowNew = rowB + T;
        uint32_t *rowPre = reinterpret_cast<uint32_t *>(rowNew + T);
        int4 *listA = reinterpret_cast<int4 *>(scr + (((size_t)3 * T * 4 + 15) & ~(size_t)15));
        int4 *listB = listA + kBandCap;

        for (int a = threadIdx.x; a < T; a += NT) rowB[a] = 0;
        if (threadIdx.x == 0) {
            S.ntk = 0;
            S.thr = ~0ull;
            S.err = 0;
        }
        __syncthreads();
        if (A.n_global == 0) return;

        const unsigned long long Tall = (unsigned long long)T * T;
        const unsigned long long L = (unsigned long long)A.L;
        unsigned long long W = 0, Cprev = 0;
        double tauLo = -1.0;
        const double maxKey = key(T - 1, T - 1);
        double target = (double)L / A.rho * 0.5;
        for (int it_band = 0;; it_band++) {
            if (target < 256.0) target = 256.0;
            if (target > (double)kBandCap) target = (double)kBandCap;
            double tauHi;
            unsigned long long cHi;
            if ((double)(Tall - Cprev) <= target) {
                tauHi = INFINITY;
                cHi = Tall;
            } else {
                double lo = tauLo, hi = maxKey;
                unsigned long long clo = Cprev, chi = Tall;
                bool accepted = false;
                tauHi = hi;
                cHi = chi;
                const double want = (double)Cprev + target;
                const double k00 = key(0, 0);
                for (int it = 0; it < 200; it++) {
                    const double xlo = fmax(lo - k00, 0.0), xhi = hi - k00;
                    if (!(xhi > 0.0)) break;
                    double mid;
                    if ((it & 1) == 0 && clo > 0 && xlo > 0.0) {
                        // secant on log C(tau) against log(tau - key00)
                        double ylo = log((double)clo), yhi = log((double)chi), yw = log(want);
                        double f = (yw - ylo) / fmax(yhi - ylo, 1e-30);
                        f = fmin(fmax(f, 0.02), 0.98);
                        mid = k00 + exp(log(xlo) + (log(xhi) - log(xlo)) * f);
                    } else {
                        // geometric bisection of (tau - key00)
                        double xl = xlo > 0.0 ? xlo : xhi * 1e-6;
                        mid = k00 + sqrt(xl * xhi);
                    }
                    if (!(mid > lo && mid < hi)) {
                        mid = lo + 0.5 * (hi - lo);
                        if (!(mid > lo && mid < hi)) break;
                    }
                    unsigned long long cm = count_le(mid, rowB, nullptr);
                    double band = (double)(cm - Cprev);
                    if (band > target) {
                        hi = mid;
                        chi = cm;
                    } else if (band < 0.5 * target) {
                        lo = mid;
                        clo = cm;
                    } else {
                        tauHi = mid;
                        cHi = cm;
                        accepted = true;
                        break;
                    }
                }
                if (!accepted) {
                    if (clo > Cprev) {
                        tauHi = lo;
                        cHi = clo;
                    } else {
                        tauHi = hi;
                        cHi = chi;
                    }
                }
                if (cHi - Cprev > (unsigned long long)kBandCap) {
                    // a single key value shared by more than kBandCap cells
                    if (threadIdx.x == 0) S.err = 1;
                    __syncthreads();
                    return;
                }
            }
            // rows touched by this band and their new bounds
            unsigned long long chk = count_le(tauHi, rowB, rowNew);
            (void)chk;
            if (threadIdx.x == 0) {
                // active rows: #{a : key(a,0) <= tauHi}
                int lo = 0, hi = T;
                const double k0 = kd(sr2, 0);
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (kd(sr1, mid) + k0 <= tauHi) lo = mid + 1; else hi = mid;
                }
                S.arows = lo;
            }
            __syncthreads();
            const int arows = S.arows;
            // flatten: rowPre[a] = sum_{a' < a} (rowNew - rowB)
            uint32_t run = 0;
            for (int base = 0; base < arows; base += NT) {
                int a = base + threadIdx.x;
                uint32_t len = a < arows ? (uint32_t)(rowNew[a] - rowB[a]) : 0u;
                uint32_t tot;
                uint32_t ex = block_excl_scan(S, len, &tot);
                if (a < arows) rowPre[a] = run + ex;
                run += tot;
            }
            const uint32_t sband = run;
            if (threadIdx.x == 0) S.nlist = 0;
            __syncthreads();
            unsigned long long wb = 0;
            for (uint32_t f = threadIdx.x; f < sband; f += NT) {
                int lo = 0, hi = arows;  // largest a with rowPre[a] <= f
                while (hi - lo > 1) {
                    int mid = (lo + hi) >> 1;
                    if (rowPre[mid] <= f) lo = mid; else hi = mid;
                }
                const int a = lo;
                const int b = rowB[a] + (int)(f - rowPre[a]);
                const unsigned long long lin = lin_of(a, b);
                const OffT g0 = __ldg(A.goff + lin), g1 = __ldg(A.goff + lin + 1);
                if (g1 > g0) {
                    uint32_t lst, lcn;
                    if (A.sharded) {
                        OffT l0 = __ldg(A.loff + lin), l1 = __ldg(A.loff + lin + 1);
                        lst = (uint32_t)l0;
                        lcn = (uint32_t)(l1 - l0);
                    } else {
                        lst = (uint32_t)g0;
                        lcn = (uint32_t)(g1 - g0);
                    }
                    uint32_t pos = atomicAdd(&S.nlist, 1u);
                    listA[pos] = make_int4((a << 16) | b, (int)(uint32_t)(g1 - g0), (int)lst, (int)lcn);
                    wb += (unsigned long long)(g1 - g0);
                }
            }
            wb = block_sum_u64(S, wb);
            const int n = (int)S.nlist;
            if (W + wb < L) {
                emit(listA, n, -1, 0);
                W += wb;
                Cprev = cHi;
                for (int a = threadIdx.x; a < arows; a += NT) rowB[a] = rowNew[a];
                __syncthreads();
                tauLo = tauHi;
                if (cHi == Tall) {
                    popped = Tall;
                    break;
                }
                double rho = (double)(W > 0 ? W : 1) / (double)Cprev;
                target = (double)(L - W) / rho * 1.3 + 64.0;
            } else {
                final_select(listA, listB, n, L - W);
                if (A.out_popped) {
                    __syncthreads();
                    popped = count_le(__longlong_as_double((long long)S.cut_key), rowB, nullptr);
                }
                break;
            }
        }
    }

    __device__ void finish() {
        if constexpr (ENGINE == ENGINE_TRAVERSE) return;
        __syncthreads();
        const int k = A.k;
        const int64_t qo = A.q0 + qi;
        if (S.err) {
            for (int x = threadIdx.x; x < k; x += NT) {
                A.out_d[qo * k + x] = INFINITY;
                A.out_ids[qo * k + x] = 0xFFFFFFFFu;
            }
            if (threadIdx.x == 0) {
                A.out_count[qo] = -1;
                if (A.out_ncand) A.out_ncand[qo] = -1;
                if (A.out_popped) A.out_popped[qo] = -1;
            }
            return;
        }
        uint32_t n = S.ntk;
        int P = 1;
        while (P < (int)n) P <<= 1;
        for (int i = threadIdx.x; i < P; i += NT)
            if (i >= (int)n) S.tk[i] = ~0ull;
        __syncthreads();
        bitonic_sort_u64(S.tk, P);
        int cnt = (int)min((unsigned long long)k, ncand);
        for (int x = threadIdx.x; x < k; x += NT) {
            if (x < cnt) {
                unsigned long long kk = S.tk[x];
                A.out_d[qo * k + x] = __uint_as_float((uint32_t)(kk >> 32));
                A.out_ids[qo * k + x] = (uint32_t)kk;
            } else {
                A.out_d[qo * k + x] = INFINITY;
                A.out_ids[qo * k + x] = 0xFFFFFFFFu;
            }
        }
        if (threadIdx.x == 0) {
            A.out_count[qo] = cnt;
            if (A.out_ncand) A.out_ncand[qo] = (int64_t)ncand;
            if (A.out_popped) A.out_popped[qo] = (int64_t)popped;
        }
    }
};

template <int ENGINE, int M, typename KT, typename OffT>
__global__ void __launch_bounds__(NT) search_kernel(Args<KT, OffT> A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    for (;;) {
        if (threadIdx.x == 0) S.qidx = (int64_t)atomicAdd(A.counter, 1u);
        __syncthreads();
        const int64_t qi = S.qidx;
        if (qi >= A.nq) return;
        Query<ENGINE, M, KT, OffT> Q(A, S, qi);
        if constexpr (ENGINE != ENGINE_TRAVERSE) {
            const float *q = A.queries + qi * A.D;
            if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                // fold = fine_norms - 2 * (book . q_p)   (fbpq.py:140-143)
                const int K = A.K, ds = A.ds;
                for (int idx = threadIdx.x; idx < M * K; idx += NT) {
                    const int p = idx / K;
                    const float *bk = A.books + (size_t)idx * ds;
                    const float *qp = q + p * ds;
                    float dot = 0.f;
                    for (int u = 0; u < ds; u++) dot = fmaf(__ldg(bk + u), __ldg(qp + u), dot);
                    S.tab[idx] = __fsub_rn(__ldg(A.fine_norms + idx), __fmul_rn(2.f, dot));
                }
                // q_norm = qr @ qr (fbpq.py:144)
                float part = 0.f;
                for (int x = threadIdx.x; x < A.D; x += NT) {
                    float v = __ldg(q + x);
                    part = fmaf(v, v, part);
                }
                float qn = block_sum_f32_ordered(S, part);
                if (threadIdx.x == 0) S.qnorm = qn;
            } else {
                for (int x = threadIdx.x; x < A.D; x += NT) S.tab[x] = __ldg(q + x);
            }
        }
        __syncthreads();
        Q.run();
        Q.finish();
        __syncthreads();
    }
}

template <int ENGINE, int M, typename KT, typename OffT>
int configure(int *n_cta_out) {
    static int n_cta = 0;
    if (n_cta == 0) {
        auto kfn = search_kernel<ENGINE, M, KT, OffT>;
        BPQ_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sizeof(Smem)));
        int dev = 0, sms = 0, occ = 0;
        BPQ_CUDA_TRY(cudaGetDevice(&dev));
        BPQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        BPQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, NT, sizeof(Smem)));
        if (occ < 1) return fail(BPQ_ERR_CUDA, "search kernel does not fit on an SM");
        n_cta = occ * sms;
    }
    *n_cta_out = n_cta;
    return BPQ_OK;
}

template <int ENGINE, int M>
int launch_one(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
               int32_t k, const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids,
               int32_t *out_count, int64_t *out_ncand, int64_t *out_popped, cudaStream_t stream) {
    int n_cta = 0;
    int rc = configure<ENGINE, M, float, uint32_t>(&n_cta);
    if (rc) return rc;
    if (n_cta > ws.n_cta) n_cta = ws.n_cta;
    Args<float, uint32_t> A{};
    A.T = ix.T;
    A.D = ix.D;
    A.dh = ix.dh;
    A.ds = ix.ds;
    A.K = ix.K;
    A.c1 = ix.c1;
    A.c2 = ix.c2;
    A.cn1 = ix.cn1;
    A.cn2 = ix.cn2;
    A.loff = ix.loff;
    A.goff = ix.goff;
    A.sharded = ix.goff != ix.loff;
    A.ids = ix.ids;
    A.codes = ix.codes;
    A.books = ix.books;
    A.fine_norms = ix.fine_norms;
    A.cross1 = ix.cross1;
    A.cross2 = ix.cross2;
    A.bank1 = ix.bank1;
    A.bank2 = ix.bank2;
    A.n_global = (unsigned long long)ix.N_global;
    A.rho = (double)(ix.N_global > 0 ? ix.N_global : 1) / ((double)ix.T * ix.T);
    A.queries = queries;
    A.q0 = q0;
    A.nq = nq;
    A.dots1 = ws.dots1;
    A.dots2 = ws.dots2;
    A.sr1 = ws.sr1;
    A.sr2 = ws.sr2;
    A.ord1 = ws.ord1;
    A.ord2 = ws.ord2;
    A.L = budget;
    A.k = k;
    A.out_d = out_dist;
    A.out_ids = out_ids;
    A.out_count = out_count;
    A.out_ncand = out_ncand;
    A.out_popped = out_popped;
    A.counter = ws.counter;
    A.scratch = ws.cta_scratch;
    A.stride = ws.cta_stride;
    BPQ_CUDA_TRY(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned int), stream));
    search_kernel<ENGINE, M, float, uint32_t><<<n_cta, NT, sizeof(Smem), stream>>>(A);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

template <int ENGINE>
int dispatch_m(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
               int32_t k, const SearchWorkspace &ws, float *od, uint32_t *oi, int32_t *oc,
               int64_t *on, int64_t *op, cudaStream_t s) {
    switch (ix.M) {
        case 2: return launch_one<ENGINE, 2>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 4: return launch_one<ENGINE, 4>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 6: return launch_one<ENGINE, 6>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 8: return launch_one<ENGINE, 8>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 10: return launch_one<ENGINE, 10>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 12: return launch_one<ENGINE, 12>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 14: return launch_one<ENGINE, 14>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
        case 16: return launch_one<ENGINE, 16>(ix, queries, q0, nq, budget, k, ws, od, oi, oc, on, op, s);
    }
    return fail(BPQ_ERR_UNSUPPORTED, "num_parts must be even and in [2, 16]");
}

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
    o += al(search_cta_scratch_bytes((int32_t)t));
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

size_t search_cta_scratch_bytes(int32_t T) {
    return (((size_t)3 * T * 4 + 15) & ~(size_t)15) + (size_t)2 * kBandCap * sizeof(int4);
}

int search_grid_ctas(int engine, int M) {
    int n = 0;
    int rc;
    // all instantiations share the shared-memory footprint; FBPQ M=8 is representative
    (void)engine;
    (void)M;
    rc = configure<BPQ_ENGINE_FBPQ, 8, float, uint32_t>(&n);
    if (rc) return -1;
    return n;
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
    int n_cta = 0;
    int rc = configure<ENGINE_TRAVERSE, 2, double, int64_t>(&n_cta);
    if (rc) return rc;
    Args<double, int64_t> A{};
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
    search_kernel<ENGINE_TRAVERSE, 2, double, int64_t><<<1, NT, sizeof(Smem), stream>>>(A);
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
