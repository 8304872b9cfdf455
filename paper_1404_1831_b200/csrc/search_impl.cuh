#pragma once
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
//   * pick a key threshold tau (secant/geometric search on the staircase
//     cell count C(tau) = sum_a #{b : key(a,b) <= tau}; each row's count is
//     a galloping search from its current boundary over the sorted keys
//     staged in shared memory);
//   * enumerate the band of cells with tauLo < key <= tau (each thread takes
//     a contiguous run of the flattened band, 8 cell-table reads in flight)
//     and read their entry counts from the cell table;
//   * if the band keeps the running total < L, every band cell is visited:
//     scan it and continue; otherwise the cutoff lies inside the band and a
//     weighted radix select over the 96-bit key (f64 key bits, oi*T+oj),
//     finished by a shared-memory bitonic sort, finds the exact cutoff.
// The per-row staircase state (rowB) replaces the reference's T*T popped
// bitmap (numba_backend.py:25).
//
// Scan.  Visited cells are scanned from a list in chunks of 256 cells; the
// chunk's entries are flattened over the CTA, each thread scoring 4
// candidates per round (code + id loads, per-part table lookups) so 4
// independent load chains are in flight.  Arithmetic follows the
// reference's operation order with explicit round-to-nearest intrinsics (no
// FMA contraction), so a candidate's distance is bit-exact given the same
// per-query tables.
//
// Top-k.  Candidates below the current k-th best key ((dist bits << 32) |
// id, i.e. (dist asc, id asc) as select_top, multi_index.py:326-339) are
// appended to a shared-memory buffer that is bitonic-compacted to k when
// it fills.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "bpq_internal.cuh"

namespace bpq {
// phase-profiling counters (bpq_debug_set_phase_buffer), one for all TUs
extern unsigned long long *g_prof_buffer;

// launches one fused-search instantiation; each (engine, M) pair is defined
// in its own translation unit (search_inst.cu) so the ptxas runs go parallel
template <int MT>
int launch_big_inst(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget, int32_t k,
                    const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids, int32_t *out_count,
                    cudaStream_t stream);
template <int ENGINE, int MT>
int launch_search_inst(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                       int32_t k, const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids,
                       int32_t *out_count, int64_t *out_ncand, int64_t *out_popped, cudaStream_t stream);

namespace {

constexpr int NT = kSearchThreads;
constexpr int NW = NT / 32;
constexpr int ENGINE_TRAVERSE = 3;
#ifndef BPQ_MINB
#define BPQ_MINB 4
#endif
constexpr int kUnroll = 4;                // candidates per thread per round
constexpr int kSrSmem = 4096;             // sorted half-distances staged in smem
constexpr int kEnumBatch = 8;             // cell-table reads in flight per thread
// Large-cell scan (point-term FBPQ, M = 8 or 16): contiguous cell ranges of
// codes and point terms stream into a ring of kBigS shared-memory stages by
// TMA bulk copies (cp.async.bulk, one elected thread, mbarrier completion),
// kBigCh entries per stage.
#ifndef BPQ_BIG_S
#define BPQ_BIG_S 3
#endif
constexpr int kBigS = BPQ_BIG_S;
__host__ __device__ constexpr int big_chunk(int m) { return m == 16 ? 256 : 512; }
// shared-memory bytes of the large-cell stages for M parts (code + point term per entry)
__host__ __device__ constexpr int pipe_stage_bytes(int m) { return kBigS * big_chunk(m) * (m + 4); }
constexpr int kSortBytes = kSortCap * (8 + 4 + 2);  // skey + slin + sidx

// Conflict-free fold table (FBPQ, M = 8 or 16).  fold[p][c] is stored R =
// 32 / M times, at float index (c * M + p) * R + r.  Lane (g = lane / M,
// x = lane % M) scores its own entry reading part (x + i) % M at step i from
// replica g, so the 32 lanes of a warp hit 32 distinct banks on every
// lookup (a plain [p][c] table costs ~3.5 wavefronts per random gather).
template <int MT>
__host__ __device__ constexpr bool rep_fold() { return MT == 8 || MT == 16; }
template <int MT>
__host__ __device__ constexpr int fold_floats_per_code() { return rep_fold<MT>() ? 32 : MT; }
template <int MT>
__device__ __forceinline__ int fold_index(int p, int c, int K) {
    if constexpr (rep_fold<MT>()) return (c * MT + p) * (32 / MT);
    else return p * K + c;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// TMA bulk copy global -> shared (16-byte aligned, size a multiple of 16), completion on *bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

struct __align__(16) Smem {
    uint32_t cpre[NT + 1];
    int32_t coi[NT];
    int32_t coj[NT];
    uint32_t cstart[NT];
    float cbase[NT];
    uint32_t ccnt[NT];
    uint16_t bigs[NT];
    uint32_t hist_w[256];
    uint32_t hist_c[256];
    unsigned long long red[NW];
    uint32_t wscan[NW];
    unsigned long long thr;
    unsigned long long sel_below;
    unsigned long long cut_key;
    int64_t qidx;
    uint32_t ntk;
    uint32_t nlist;
    float qnorm;
    int sel_v;
    int cnt_nr;
    int cnt_nc;
    double mtau[NW];
    unsigned long long mcnt[NW];
    unsigned long long tor[NW];  // top-k compaction: per-warp OR of the buffered keys
    uint32_t nbig;
    int err;
    int prof_ph;
    long long prof_t;
    // top-k compaction scratch (separate: compaction runs inside final_select)
    int tsel_v;
    uint32_t tcnt;
    unsigned long long tsel_below;
    unsigned long long tkey;
    uint32_t nholes;
    uint32_t tphase;  // large-cell stage mbarrier parities (bit s = slot s)
    unsigned long long mbar[kBigS];
    uint16_t holes[kMaxK];
};

#ifdef BPQ_PHASE_PROF
template <typename SM>
__device__ __forceinline__ int prof_switch(SM &S, unsigned long long *acc, int ph) {
    int prev = S.prof_ph;
    __syncwarp();
    if (threadIdx.x == 0 && acc) {
        long long now = clock64();
        atomicAdd(acc + S.prof_ph, (unsigned long long)(now - S.prof_t));
        S.prof_t = now;
        S.prof_ph = ph;
    }
    return prev;
}
#define PROF(ph) prof_switch(S, A.prof, (ph))
#else
__device__ __forceinline__ int prof_nop() { return 0; }
#define PROF(ph) prof_nop()
#endif

// Optional per-phase cycle accounting (compile with -DBPQ_PHASE_PROF): thread 0
// of each CTA attributes elapsed clock64 cycles to the current phase.
// (PH_B*: the large-cell stream kernel)
enum Phase { PH_PROLOGUE, PH_TAU, PH_BOUNDS, PH_ENUM, PH_SCAN, PH_LUT, PH_COMPACT, PH_FINAL, PH_FINISH, PH_IDLE, PH_EXTEND,
             PH_BPRO, PH_BWAIT, PH_BSCORE, PH_BCOMPACT, PH_BFIN, PH_LUTBUILD, PH_N };
// counter slots after the phase cycles (phase-profiling builds): residual-table halves built
constexpr int PROF_LUT_HALVES = PH_N;
// (every build, when a buffer is set) entries the large-cell stream kernel scans
constexpr int PROF_STREAM_CAND = PH_N + 1;

template <typename KT, typename OffT>
struct Args {
    int T, D, dh, ds, K, M;
    const float *c1, *c2, *cn1, *cn2;
    const OffT *loff, *goff;
    bool sharded;
    const uint32_t *ids;
    const uint8_t *codes;
    const float *books, *fine_norms, *cross1, *cross2, *bank1, *bank2;
    const float *pterm;        // FBPQ per-entry point term (null: exact reference order)
    const uint8_t *codes_rot;  // codes with entry e's bytes rotated by e % M (point-term FBPQ, M = 8 / 16)
    // deferred large cells (point-term FBPQ, M = 8 / 16): the traversal kernel
    // records them here and big_scan_kernel streams them (null: scan in place)
    int4 *big_cells;           // [nq][big_cap] (start, count, cell_base bits, 0)
    uint32_t *big_n;           // [nq] cells recorded
    int big_cap;
    unsigned long long *tk_part;  // [nq][k] top-k keys of the small cells
    uint32_t *tk_n;            // [nq]
    unsigned long long *ncand_q;  // [nq] candidate count (small + large cells)
    unsigned int *bigq_list, *bigq_count;  // queries with deferred cells
    const uint32_t *big_start; // [nq + 1] packed per-query cell ranges (split scan; null: big_cap stride)
    // record mode (query-split sharding): every visited non-empty cell is recorded as
    // (oi * T + oj, global count, cell_base bits, 0) instead of scanned
    int4 *record;
    uint32_t *record_n;
    int record_cap;
    const float *rot1, *rot2;  // HBPQ per-half rotations (optional)
    bool exact;                // reference operation order for every engine (bpq_index_desc.fbpq_exact)
    double rho;
    unsigned long long n_global;
    uint32_t n_local;          // entries in this index's (shard's) code / point-term arrays
    const float *queries;
    int64_t q0, nq;
    const float *dots1, *dots2, *fold;
    const float *ru1, *ru2;          // unsorted half-distances [nq, T] (sparse mode)
    int topP;                        // sorted prefix length available in sr/ord
    const int32_t *plen;             // per (query, half) prefix length (partial sort) or null
    unsigned int *retry_list, *retry_count;   // queries needing the full sort
    const unsigned int *qlist, *qlist_count;  // indirect query list (retry pass)
    const KT *sr1, *sr2;
    const int32_t *ord1, *ord2;
    const int32_t *pos1, *pos2;
    const uint32_t *rowptr, *colptr;
    const uint16_t *rowcols, *colrows;
    long long L;
    int k;
    int lut_min;     // cells with >= lut_min entries take the per-cell scan
    int nb0;         // lines activated by the first sparse-traversal batch
    int flow_growth; // large-cell stream: cap on an optimistic segment's length, in multiples of the chunks seen (0: none)
    int tkcap;       // top-k buffer capacity (keys) in dynamic shared memory
    int tk_off;      // its byte offset in dynamic shared memory
    int tab_floats;  // floats of the per-query table staged after Smem
    int sr_smem;     // sorted-key prefix length staged in smem
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
    unsigned long long *prof;  // [PH_N] cycle counters (phase-profiling builds)
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
template <typename SM>
__device__ __forceinline__ uint32_t block_excl_scan(SM &S, uint32_t v, uint32_t *total) {
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

template <int BT = NT>
__device__ __forceinline__ void bitonic_sort_u64(unsigned long long *a, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += BT) {
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
__device__ __forceinline__ void bitonic_sort_cells(unsigned long long *skey, uint32_t *slin, uint16_t *sidx, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool up = (i & k) == 0;
                    unsigned long long ka = skey[i], kb = skey[ixj];
                    uint32_t la = slin[i], lb = slin[ixj];
                    bool gt = (ka > kb) || (ka == kb && la > lb);
                    if (gt == up) {
                        skey[i] = kb;
                        skey[ixj] = ka;
                        slin[i] = lb;
                        slin[ixj] = la;
                        uint16_t t = sidx[i];
                        sidx[i] = sidx[ixj];
                        sidx[ixj] = t;
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

// ------------------------------------------------------------ code loading
// MT = compile-time number of parts (8 or 16, the BASELINE configs), or 0
// for the generic path where M (even, <= 16) is a runtime value.
template <int MT>
__device__ __forceinline__ void load_code(const uint8_t *p, uint32_t (&w)[4], int M) {
    if constexpr (MT == 16) {
        uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else if constexpr (MT == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = v.x; w[1] = v.y; w[2] = 0; w[3] = 0;
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) w[i] = 0;
        if ((M & 3) == 0) {
            for (int i = 0; i < M / 4; i++) w[i] = __ldg(reinterpret_cast<const uint32_t *>(p) + i);
        } else {
            for (int i = 0; i < M / 2; i++) {
                uint32_t h = __ldg(reinterpret_cast<const uint16_t *>(p) + i);
                w[i >> 1] |= h << ((i & 1) * 16);
            }
        }
    }
}

__device__ __forceinline__ int code_at(const uint32_t (&w)[4], int p) {
    return (w[p >> 2] >> ((p & 3) * 8)) & 0xFF;
}

// --------------------------------------------------- per-candidate distances
template <int MT, typename KT, typename OffT>
__device__ __forceinline__ float dist_fbpq(const Args<KT, OffT> &A, const float *tab, int oi, int oj,
                                           float cbase, const uint32_t (&w)[4]) {
    const int M = MT ? MT : A.M;
    const int M2 = M / 2;
    const int K = A.K;
    float x[16];
#pragma unroll
    for (int p = 0; p < M; p++) {
        const int c = code_at(w, p);
        x[p] = p < M2 ? __ldg(A.cross1 + ((size_t)oi * M2 + p) * K + c)
                      : __ldg(A.cross2 + ((size_t)oj * M2 + (p - M2)) * K + c);
    }
    float acc = cbase;
#pragma unroll
    for (int p = 0; p < M; p++) {
        const int c = code_at(w, p);
        acc = __fadd_rn(acc, __fadd_rn(tab[p * K + c], __fmul_rn(2.f, x[p])));
    }
    if (acc < 0.f) acc = 0.f;  // numba_backend.py:241-242
    return acc;
}

// FBPQ through the index's point term pt = sum_p 2*cross[row][p][c_p]
// (bpq_index_desc.fbpq_exact == 0): ((sum_p fold[p][c_p]) + pt) + cell_base,
// M shared-memory lookups and no cross-table gathers.  Same quantity as the
// reference's cell_base + sum_p (fold + 2*cross) (numba_backend.py:231-242),
// summed in another order (max 4.3e-7 relative on the config-0 captures).
// Generic-M path (plain [p][c] fold table).
template <int MT>
__device__ __forceinline__ float dist_fbpq_pt(const float *tab, int M, int K, float cbase, float pt,
                                              const uint32_t (&w)[4]) {
    if constexpr (MT != 0) M = MT;
    float s = tab[code_at(w, 0)];
#pragma unroll
    for (int p = 1; p < (MT ? MT : 16); p++)
        if (MT || p < M) s = __fadd_rn(s, tab[p * K + code_at(w, p)]);
    const float acc = __fadd_rn(__fadd_rn(s, pt), cbase);
    return acc < 0.f ? 0.f : acc;
}

// Rotation and replica of the conflict-free fold lookups (M = 8 or 16) for
// an entry with y = (local entry index) & 31: the code bytes rotate by
// x = y % M and, per step i, the lookup reads replica g = y / M of part
// (x + i) % M at float offset ((x + i) % M) * R + g.  32 consecutive entries
// scored by the 32 lanes of a warp therefore hit 32 distinct banks, and an
// entry's summation order depends only on its position in the index (not on
// the traversal, the lane or the scan path).
template <int MT>
struct LaneLut {
    int rot;
    int off[MT];
    __device__ __forceinline__ explicit LaneLut(int y) {
        constexpr int R = 32 / MT;
        const int x = y % MT, g = (y / MT) % R;
        rot = x;
#pragma unroll
        for (int i = 0; i < MT; i++) off[i] = ((x + i) % MT) * R + g;
    }
};

// Pairwise sum of the M step values, ((v0 + v1) + (v2 + v3)) + ..., fixed
// structure (3 or 4 dependent adds instead of M - 1)
template <int MT>
__device__ __forceinline__ float tree_sum(float (&v)[MT]) {
#pragma unroll
    for (int w = 1; w < MT; w *= 2)
#pragma unroll
        for (int i = 0; i < MT; i += 2 * w) v[i] = __fadd_rn(v[i], v[i + w]);
    return v[0];
}

// the same sum through the plain [p][c] fold table (small cells in the
// traversal kernel): identical operation order, so an entry scores the same
// bits whichever kernel scans it
// (codes_rot: the index's copy of the codes with entry e's bytes already
// rotated by e % M, bpq_index_create; no per-entry rotation here)
template <int MT>
__device__ __forceinline__ float dist_pt_plain(const float *tab, int K, int y, float cbase, float pt,
                                               const uint32_t (&r)[4]) {
    const int x = y % MT;
    float v[MT];
#pragma unroll
    for (int i = 0; i < MT; i++) {
        const uint32_t c = __byte_perm(r[i >> 2], 0u, 0x4440u | (uint32_t)(i & 3));
        v[i] = tab[((x + i) & (MT - 1)) * K + (int)c];
    }
    const float acc = __fadd_rn(__fadd_rn(tree_sum<MT>(v), pt), cbase);
    return acc < 0.f ? 0.f : acc;
}

// point-term FBPQ distance through the replicated fold table (M = 8 or 16):
// the parts are summed in the lane's rotated order (pairwise), then + pt +
// cell_base.  offb[i] = byte offset of the lane's slot for step i.
template <int MT>
__device__ __forceinline__ float dist_pt_rep(const char *tabb, const int (&offb)[MT], float cbase, float pt,
                                             const uint32_t (&r)[4]) {
    float v[MT];
#pragma unroll
    for (int i = 0; i < MT; i++) {
        const uint32_t c = __byte_perm(r[i >> 2], 0u, 0x4440u | (uint32_t)(i & 3));
        v[i] = *reinterpret_cast<const float *>(tabb + (c << 7) + offb[i]);
    }
    const float acc = __fadd_rn(__fadd_rn(tree_sum<MT>(v), pt), cbase);
    return acc < 0.f ? 0.f : acc;
}

// Multi-D-ADC explicit reconstruction (ENGINE 0) and HBPQ local books
// (ENGINE 2): e = q_h - c_h[row] (one rounding, multi_index.py:345-346),
// d = e - book, acc += d*d sequentially (numba_backend.py:165-176, 198-210).
template <int ENGINE, int MT, typename KT, typename OffT>
__device__ __forceinline__ float dist_recon(const Args<KT, OffT> &A, const float *tab, int oi, int oj,
                                            const uint32_t (&w)[4], const float *erow = nullptr) {
    const int M = MT ? MT : A.M;
    const int M2 = M / 2;
    const int K = A.K, ds = A.ds, dh = A.dh;
    float acc = 0.f;
    // M = 16: a rolled part loop (the fully unrolled 16-part reconstruction, times the
    // emit loop's 4 candidates, made these instantiations take ~15 minutes in ptxas)
    constexpr int kPartUnroll = MT == 16 ? 1 : 8;
#pragma unroll kPartUnroll
    for (int p = 0; p < M; p++) {
        const int hp = p < M2 ? p : p - M2;
        const int row = p < M2 ? oi : oj;
        const float *cr = (p < M2 ? A.c1 : A.c2) + (size_t)row * dh + hp * ds;
        const float *qv = tab + (p < M2 ? 0 : dh) + hp * ds;
        const int c = code_at(w, p);
        const float *bk;
        if constexpr (ENGINE == BPQ_ENGINE_HBPQ)
            bk = (p < M2 ? A.bank1 : A.bank2) + (((size_t)row * M2 + hp) * K + c) * ds;
        else
            bk = A.books + ((size_t)p * K + c) * ds;
        if (erow != nullptr) {  // rotated displacement row (HBPQ with bank rotations)
            const float *er = erow + (p < M2 ? 0 : dh) + hp * ds;
            for (int u = 0; u < ds; u++) {
                float d = __fsub_rn(er[u], __ldg(bk + u));
                acc = __fadd_rn(acc, __fmul_rn(d, d));
            }
        } else if ((ds & 3) == 0) {
            for (int u = 0; u < ds; u += 4) {
                const float4 cv = __ldg(reinterpret_cast<const float4 *>(cr + u));
                const float4 bv = __ldg(reinterpret_cast<const float4 *>(bk + u));
                const float ce[4] = {cv.x, cv.y, cv.z, cv.w};
                const float be[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int z = 0; z < 4; z++) {
                    float d = __fsub_rn(__fsub_rn(qv[u + z], ce[z]), be[z]);
                    acc = __fadd_rn(acc, __fmul_rn(d, d));
                }
            }
        } else {
            for (int u = 0; u < ds; u++) {
                float d = __fsub_rn(__fsub_rn(qv[u], __ldg(cr + u)), __ldg(bk + u));
                acc = __fadd_rn(acc, __fmul_rn(d, d));
            }
        }
    }
    return acc;
}

// ------------------------------------------------------------ top-k buffer
// Keep the k smallest of the n > k buffered keys (keys are unique: the id
// is in the low word).  An MSB-first radix select on the 64-bit keys finds
// the k-th smallest in a few 256-bin histogram passes, then the survivors
// are compacted to the front and the admission threshold becomes that key.
template <int BT = NT, typename SM>
__device__ void topk_compact(SM &S, unsigned long long *__restrict__ tk, int k) {
    const uint32_t n = S.ntk;
    if ((int)n <= k) return;
    // bits shared by every buffered key (AND == OR) need no histogram pass:
    // start at the digit holding the highest differing bit
    unsigned long long ka = ~0ull, ko = 0ull;
    for (uint32_t i = threadIdx.x; i < n; i += BT) {
        ka &= tk[i];
        ko |= tk[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ka &= __shfl_xor_sync(0xffffffffu, ka, o);
        ko |= __shfl_xor_sync(0xffffffffu, ko, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        S.red[threadIdx.x >> 5] = ka;
        S.tor[threadIdx.x >> 5] = ko;
    }
    __syncthreads();
    ka = ~0ull;
    ko = 0ull;
#pragma unroll
    for (int w = 0; w < BT / 32; w++) {
        ka &= S.red[w];
        ko |= S.tor[w];
    }
    const int hb = 63 - __clzll((long long)(ka ^ ko));  // keys are unique: ka != ko
    // digits of up to 8 bits, the first one ending at the highest differing bit (a byte-aligned
    // first digit can hold a single useful bit: a wasted pass of same-address atomics)
    unsigned long long pmask = hb >= 63 ? 0ull : ~0ull << (hb + 1);
    unsigned long long prefix = ka & pmask;
    uint32_t rank = (uint32_t)k;  // 1-based rank of the wanted key among matches
    for (int hi = hb; hi >= 0; hi -= 8) {
        const int shift = hi >= 7 ? hi - 7 : 0;
        const uint32_t dmask = (1u << (hi - shift + 1)) - 1u;
        for (int i = threadIdx.x; i < 256; i += BT) S.hist_c[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += BT) {
            const unsigned long long key = tk[i];
            if ((key & pmask) == prefix) atomicAdd(&S.hist_c[(uint32_t)(key >> shift) & dmask], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // warp scan over 256 bins (8 per lane)
            const int lane = threadIdx.x;
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                loc[x] = S.hist_c[lane * 8 + x];
                sum += loc[x];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t run = incl - sum;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                if (run < rank && run + loc[x] >= rank) {
                    S.tsel_v = lane * 8 + x;
                    S.tsel_below = run;
                    S.tcnt = loc[x];
                }
                run += loc[x];
            }
        }
        __syncthreads();
        const unsigned long long d = (unsigned long long)S.tsel_v;
        rank -= (uint32_t)S.tsel_below;
        prefix |= d << shift;
        pmask |= (unsigned long long)dmask << shift;
        if (S.tcnt == 1u) {
            // a single key carries this prefix: it is the k-th smallest
            for (uint32_t i = threadIdx.x; i < n; i += BT)
                if ((tk[i] & pmask) == prefix) S.tkey = tk[i];
            __syncthreads();
            prefix = S.tkey;
            break;
        }
        __syncthreads();
    }
    const unsigned long long kth = prefix;
    // move the survivors (keys <= kth, exactly k of them) into [0, k): slots
    // below k holding larger keys are holes, survivors at or above k fill them
    if (threadIdx.x == 0) {
        S.tcnt = 0;
        S.nholes = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += BT)
        if (tk[i] > kth) S.holes[atomicAdd(&S.nholes, 1u)] = (uint16_t)i;
    __syncthreads();
    for (uint32_t i = k + threadIdx.x; i < n; i += BT) {
        const unsigned long long key = tk[i];
        if (key <= kth) tk[S.holes[atomicAdd(&S.tcnt, 1u)]] = key;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        S.ntk = (uint32_t)k;
        S.thr = kth;
    }
    __syncthreads();
}

// Write the compacted top-k (S.ntk <= k unique keys in tk) as select_top's
// (dist asc, id asc) list of min(k, ncand) entries, padded with (+inf, ~0).
template <int BT = NT, typename SM>
__device__ void write_topk(SM &S, unsigned long long *__restrict__ tk, int k, unsigned long long ncand,
                           float *__restrict__ od, uint32_t *__restrict__ oi, int32_t *__restrict__ oc) {
    const uint32_t n = S.ntk;
    const int cnt = (int)min((unsigned long long)k, ncand);
    if (n <= 512) {
        // keys are unique: each key's rank is its output position
        for (int x = threadIdx.x; x < (int)n; x += BT) {
            const unsigned long long kx = tk[x];
            int rank = 0;
            for (uint32_t y = 0; y < n; y++) rank += tk[y] < kx ? 1 : 0;
            od[rank] = __uint_as_float((uint32_t)(kx >> 32));
            oi[rank] = (uint32_t)kx;
        }
    } else {
        int P2 = 1;
        while (P2 < (int)n) P2 <<= 1;
        for (int i = threadIdx.x; i < P2; i += BT)
            if (i >= (int)n) tk[i] = ~0ull;
        __syncthreads();
        bitonic_sort_u64<BT>(tk, P2);
        for (int x = threadIdx.x; x < cnt; x += BT) {
            const unsigned long long kk = tk[x];
            od[x] = __uint_as_float((uint32_t)(kk >> 32));
            oi[x] = (uint32_t)kk;
        }
    }
    for (int x = cnt + threadIdx.x; x < k; x += BT) {
        od[x] = INFINITY;
        oi[x] = 0xFFFFFFFFu;
    }
    if (threadIdx.x == 0) *oc = cnt;
}

// ------------------------------------------------------- per-query context
//
// Staircase state.  The popped region is a Young diagram in sorted
// coordinates.  It is split on the diagonal: row a owns its cells with
// b >= a (boundary rowB[a], initially a) and column b owns its cells with
// a > b (boundary colB[b], initially b + 1).  Rows whose diagonal key
// key(a, a) exceeds tau hold no cells <= tau, and likewise columns whose
// key(b + 1, b) exceeds tau, so a count or a band touches only O(active
// rows + active columns) lines even when the region is a long thin "L"
// (one very close codeword per half, which the BASELINE mixture produces).
// SPARSE_ONLY: the first pass over a partially sorted sparse table.  Any
// query the sparse traversal cannot finish is queued for the full-sort retry
// pass, so the band (dense) traversal is compiled out of this instantiation
// -- which keeps the scan loop free of register spills.
template <int ENGINE, int MT, typename KT, typename OffT, bool SPARSE_ONLY = false>
struct Query {
    const Args<KT, OffT> &A;
    Smem &S;
    int64_t qi;
    const KT *sr1, *sr2;     // global sorted half-distances of this query
    const KT *s1s, *s2s;     // smem prefixes [0, P)
    const float *tab;        // smem per-query table (fold or query vector)
    float *lut;              // smem per-cell lookup table (FBPQ)
    unsigned long long *tk;  // smem top-k buffer [A.tkcap]
    // final-band / prefix-extension sort arrays [kSortCap]: they alias the
    // per-cell LUT or cp.async stages, which are dead whenever they are live
    unsigned long long *skey;
    uint32_t *slin;
    uint16_t *sidx;
    const int32_t *o1, *o2;  // sorted position -> codeword
    const int32_t *p1, *p2;  // codeword -> sorted position
    const float *d1, *d2;
    const float *u1, *u2;    // unsorted half-distances (codeword-keyed entries)
    float *erot;             // [NT][D] rotated displacement rows of the current chunk (HBPQ)
    int lut_i, lut_j;        // coarse codewords the two LUT halves were built for (-1: none)
    bool cw;                 // list entries hold codewords (i, j) instead of positions (a, b)
    int T, P, M;
    int tp1, tp2;              // valid sorted prefix per half (partial sort), block-uniform
    unsigned long long ncand;  // uniform across the CTA
    unsigned long long popped;
    uint32_t nbig_q;           // large cells deferred to big_scan_kernel (block-uniform)
    uint32_t nrec_q;           // cells recorded (record mode, block-uniform)

    __device__ Query(const Args<KT, OffT> &a, Smem &s, int64_t q, const float *tab_, float *lut_,
                     const KT *s1, const KT *s2, unsigned long long *tk_)
        : A(a), S(s), qi(q), s1s(s1), s2s(s2), tab(tab_), lut(lut_), tk(tk_) {
        skey = reinterpret_cast<unsigned long long *>(lut_);
        slin = reinterpret_cast<uint32_t *>(skey + kSortCap);
        sidx = reinterpret_cast<uint16_t *>(slin + kSortCap);
        T = A.T;
        M = MT ? MT : A.M;
        P = A.sr_smem;
        sr1 = A.sr1 + q * T;
        sr2 = A.sr2 + q * T;
        o1 = A.ord1 + q * T;
        o2 = A.ord2 + q * T;
        p1 = A.pos1 ? A.pos1 + q * T : nullptr;
        p2 = A.pos2 ? A.pos2 + q * T : nullptr;
        d1 = A.dots1 ? A.dots1 + q * T : nullptr;
        d2 = A.dots2 ? A.dots2 + q * T : nullptr;
        u1 = A.ru1 ? A.ru1 + q * T : nullptr;
        u2 = A.ru2 ? A.ru2 + q * T : nullptr;
        cw = false;
        erot = nullptr;
        lut_i = lut_j = -1;
        ncand = 0;
        popped = 0;
        nbig_q = 0;
        nrec_q = 0;
    }

    // plain (not read-only-path) loads: extend() appends to sr/ord in-kernel
    __device__ __forceinline__ double k1(int a) const { return a < P ? (double)s1s[a] : (double)sr1[a]; }
    __device__ __forceinline__ double k2(int b) const { return b < P ? (double)s2s[b] : (double)sr2[b]; }
    __device__ __forceinline__ double key(int a, int b) const { return k1(a) + k2(b); }

    __device__ __forceinline__ unsigned long long lin_of(int a, int b) const {
        return (unsigned long long)o1[a] * (unsigned long long)T + (unsigned)o2[b];
    }

    // List entries: x = (hi << 16) | lo, positions (a, b) in the band
    // traversal or codewords (i, j) in the sparse one (cw).  Both give the
    // same key value: f64(r1[i]) + f64(r2[j]) == f64(sr1[a]) + f64(sr2[b]).
    __device__ __forceinline__ double ekey(int4 e) const {
        const int x = (unsigned)e.x >> 16, y = e.x & 0xFFFF;
        return cw ? (double)__ldg(u1 + x) + (double)__ldg(u2 + y) : key(x, y);
    }
    __device__ __forceinline__ unsigned long long elin(int4 e) const {
        const int x = (unsigned)e.x >> 16, y = e.x & 0xFFFF;
        return cw ? (unsigned long long)x * T + (unsigned)y : lin_of(x, y);
    }
    __device__ __forceinline__ void eij(int4 e, int &oi, int &oj) const {
        const int x = (unsigned)e.x >> 16, y = e.x & 0xFFFF;
        if (cw) {
            oi = x;
            oj = y;
        } else {
            oi = o1[x];
            oj = o2[y];
        }
    }

    // 12-byte composite sort key digit d (0 = most significant)
    __device__ __forceinline__ int digit(int d, int4 e) const {
        if (d < 8) {
            unsigned long long kb = (unsigned long long)__double_as_longlong(ekey(e));
            return (int)((kb >> (56 - 8 * d)) & 0xFF);
        }
        unsigned long long lin = elin(e);
        return (int)((lin >> (24 - 8 * (d - 8))) & 0xFF);
    }

    __device__ __forceinline__ void offer(float dist, uint32_t id) {
        const unsigned long long kk = ((unsigned long long)canon_bits(dist) << 32) | id;
        if (kk < S.thr) {
            uint32_t pos = atomicAdd(&S.ntk, 1u);
            tk[pos] = kk;
        }
    }

    // Offer with the id loaded only when the distance can enter the top-k
    // (dist bits <= threshold's): most candidates are rejected on the
    // distance alone, which saves the id read (4 of the 12 B per candidate).
    __device__ __forceinline__ void offer_lazy(float dist, const uint32_t *idp) {
        const uint32_t db = canon_bits(dist);
        if (db <= (uint32_t)(S.thr >> 32)) offer(dist, __ldg(idp));
    }

    __device__ __forceinline__ void round_end(int cap = NT * kUnroll) {
        __syncthreads();
        if (S.ntk > (uint32_t)(A.tkcap - cap)) {
            const int pv = PROF(PH_COMPACT);
            topk_compact(S, tk, A.k);
            PROF(pv);
            (void)pv;
        }
    }

    // FBPQ, one large cell: LUT[p][c] = fold[p][c] + 2*cross[row][p][c] is
    // exactly the reference's per-part increment (numba_backend.py:236-240),
    // staged once so each entry costs M shared-memory lookups.
    __device__ void scan_cell_lut(int oi, int oj, uint32_t lst, uint32_t lc, float cb) {
        const int pv = PROF(PH_LUT);
        (void)pv;
        const int M2 = M / 2;
        const int K = A.K;
        // each half of the LUT depends on one coarse codeword only: rebuild a
        // half only when the cell's row (or column) changed since the last cell
        const int lo_idx = oi == lut_i ? M2 * K : 0;
        const int hi_idx = oj == lut_j ? M2 * K : M * K;
        if (A.pterm == nullptr && lo_idx < hi_idx) {
            for (int idx = lo_idx + threadIdx.x; idx < hi_idx; idx += NT) {
                const int p = idx / K, c = idx - p * K;
                const float x = p < M2 ? __ldg(A.cross1 + ((size_t)oi * M2 + p) * K + c)
                                       : __ldg(A.cross2 + ((size_t)oj * M2 + (p - M2)) * K + c);
                lut[idx] = __fadd_rn(tab[idx], __fmul_rn(2.f, x));
            }
            __syncthreads();
        }
        lut_i = oi;
        lut_j = oj;
        // kLutUnroll codes per thread per round keep 2x the bytes in flight
        for (uint32_t e0 = 0; e0 < lc; e0 += NT * kLutUnroll) {
            uint32_t w[kLutUnroll][4];
            float ptv[kLutUnroll];
#pragma unroll
            for (int u = 0; u < kLutUnroll; u++) {
                const uint32_t e = e0 + u * NT + threadIdx.x;
                if (e < lc) {
                    load_code<MT>(A.codes + (size_t)(lst + e) * M, w[u], M);
                    if (A.pterm) ptv[u] = __ldg(A.pterm + lst + e);
                }
            }
#pragma unroll
            for (int u = 0; u < kLutUnroll; u++) {
                const uint32_t e = e0 + u * NT + threadIdx.x;
                if (e < lc) {
                    float acc;
                    if (A.pterm) {
                        acc = dist_fbpq_pt<MT>(tab, M, K, cb, ptv[u], w[u]);
                    } else {
                        acc = cb;
#pragma unroll
                        for (int p = 0; p < M; p++) acc = __fadd_rn(acc, lut[p * K + code_at(w[u], p)]);
                        if (acc < 0.f) acc = 0.f;
                    }
                    offer_lazy(acc, A.ids + lst + e);
                }
            }
            round_end(NT * kLutUnroll);
        }
        __syncthreads();
        PROF(pv);
    }

    // Point-term FBPQ (M = 8 / 16): the band's large cells are recorded for
    // big_scan_kernel, which streams their contiguous code / point-term
    // ranges through a deep TMA ring (the traversal kernel keeps its
    // occupancy; the stream gets the shared memory).  At most L / lut_min + 1
    // large cells are visited per query: every visited cell but the cutoff
    // cell lies inside the budget.
    __device__ void defer_big(uint32_t nb) {
        unsigned long long add = 0;
        for (uint32_t x = threadIdx.x; x < nb; x += NT) {
            const int t = S.bigs[x];
            const uint32_t pos = nbig_q + x;
            if (pos < (uint32_t)A.big_cap)
                A.big_cells[(size_t)qi * A.big_cap + pos] =
                    make_int4((int)S.cstart[t], (int)S.ccnt[t], __float_as_int(S.cbase[t]), 0);
            else
                S.err = 1;  // cannot happen within the L / lut_min + 2 bound; fail loudly if it does
            add += S.ccnt[t];
        }
        ncand += block_sum_u64(S, add);
        nbig_q += nb;
        __syncthreads();
    }

    // Multi-D-ADC / HBPQ, one large cell: the cell's residual lookup table
    // LUT[p][c] = sum_u ((q_h[u] - c_h[row][u]) - book[c][u])^2 with the
    // global books (Multi-D-ADC) or the row's / column's local books (HBPQ,
    // the per-cell tables of BASELINE configs[2]), each part summed in the
    // reference's order (numba_backend.py:165-176, 198-210); an entry then
    // costs M shared-memory lookups.  Each half is rebuilt only when the
    // cell's row (column) codeword changes.  The per-part split regroups the
    // reference's single running sum (within 1e-6 relative).
    __device__ void scan_cell_recon_lut(int oi, int oj, uint32_t lst, uint32_t lc) {
        const int pv = PROF(PH_LUT);
        (void)pv;
        const int M2 = M / 2, K = A.K, ds = A.ds, dh = A.dh;
        const int lo_idx = oi == lut_i ? M2 * K : 0;
        const int hi_idx = oj == lut_j ? M2 * K : M * K;
        if (lo_idx < hi_idx) {
            PROF(PH_LUTBUILD);
#ifdef BPQ_PHASE_PROF
            if (threadIdx.x == 0 && A.prof) atomicAdd(A.prof + PROF_LUT_HALVES, (unsigned long long)((hi_idx - lo_idx) / (M2 * K)));
#endif
            for (int idx = lo_idx + threadIdx.x; idx < hi_idx; idx += NT) {
                const int p = idx / K, c = idx - p * K;
                const int hp = p < M2 ? p : p - M2;
                const int row = p < M2 ? oi : oj;
                const float *cr = (p < M2 ? A.c1 : A.c2) + (size_t)row * dh + hp * ds;
                const float *qv = tab + (p < M2 ? 0 : dh) + hp * ds;
                const float *bk;
                if constexpr (ENGINE == BPQ_ENGINE_HBPQ)
                    bk = (p < M2 ? A.bank1 : A.bank2) + (((size_t)row * M2 + hp) * K + c) * ds;
                else
                    bk = A.books + ((size_t)p * K + c) * ds;
                float acc = 0.f;
                if ((ds & 3) == 0) {
                    for (int u = 0; u < ds; u += 4) {
                        const float4 cv = __ldg(reinterpret_cast<const float4 *>(cr + u));
                        const float4 bv = __ldg(reinterpret_cast<const float4 *>(bk + u));
                        const float ce[4] = {cv.x, cv.y, cv.z, cv.w};
                        const float be[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                        for (int z = 0; z < 4; z++) {
                            const float d = __fsub_rn(__fsub_rn(qv[u + z], ce[z]), be[z]);
                            acc = __fadd_rn(acc, __fmul_rn(d, d));
                        }
                    }
                } else {
                    for (int u = 0; u < ds; u++) {
                        const float d = __fsub_rn(__fsub_rn(qv[u], __ldg(cr + u)), __ldg(bk + u));
                        acc = __fadd_rn(acc, __fmul_rn(d, d));
                    }
                }
                lut[idx] = acc;
            }
            __syncthreads();
            PROF(PH_LUT);
        }
        lut_i = oi;
        lut_j = oj;
        for (uint32_t e0 = 0; e0 < lc; e0 += NT * kLutUnroll) {
            uint32_t w[kLutUnroll][4];
#pragma unroll
            for (int u = 0; u < kLutUnroll; u++) {
                const uint32_t e = e0 + u * NT + threadIdx.x;
                if (e < lc) load_code<MT>(A.codes + (size_t)(lst + e) * M, w[u], M);
            }
#pragma unroll
            for (int u = 0; u < kLutUnroll; u++) {
                const uint32_t e = e0 + u * NT + threadIdx.x;
                if (e < lc) {
                    float acc = 0.f;
#pragma unroll
                    for (int p = 0; p < M; p++) acc = __fadd_rn(acc, lut[p * K + code_at(w[u], p)]);
                    offer_lazy(acc, A.ids + lst + e);
                }
            }
            round_end(NT * kLutUnroll);
        }
        __syncthreads();
        PROF(pv);
    }

    // Visit a list of cells: scan their entries (search) or record them
    // (traversal stage).  filt_d < 0: all cells; else only cells whose digit
    // filt_d is < filt_v.
    __device__ void emit(const int4 *list, int n, int filt_d, int filt_v) {
        const int pv = PROF(PH_SCAN);
        (void)pv;
        for (int base = 0; base < n; base += NT) {
            int c = base + threadIdx.x;
            uint32_t lc = 0;
            int oi = 0, oj = 0;
            uint32_t lst = 0;
            float cb = 0.f;
            bool big = false;
            if (threadIdx.x == 0) S.nbig = 0;
            if (c < n) {
                int4 e = list[c];
                bool pass = filt_d < 0 || digit(filt_d, e) < filt_v;
                if (pass) {
                    eij(e, oi, oj);
                    lst = (uint32_t)e.z;
                    lc = (uint32_t)e.w;
                    if constexpr (ENGINE == ENGINE_TRAVERSE) {
                        unsigned long long pos = atomicAdd(A.tv_n, 1ull);
                        A.tv_key[pos] = (unsigned long long)__double_as_longlong(ekey(e));
                        A.tv_lin[pos] = (uint32_t)oi * (uint32_t)T + (uint32_t)oj;
                        A.tv_start[pos] = (int64_t)lst;
                        A.tv_end[pos] = (int64_t)lst + lc;
                    }
                    if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                        // cell_base, numba_backend.py:232
                        float s = __fadd_rn(__ldg(d1 + oi), __ldg(d2 + oj));
                        float t0 = __fsub_rn(S.qnorm, __fmul_rn(2.f, s));
                        cb = __fadd_rn(__fadd_rn(t0, __ldg(A.cn1 + oi)), __ldg(A.cn2 + oj));
                        big = lc >= (uint32_t)A.lut_min;
                    } else if constexpr (ENGINE == BPQ_ENGINE_BASELINE || ENGINE == BPQ_ENGINE_HBPQ) {
                        // decided on the GLOBAL cell count (e.y), so a cell takes the same
                        // path on one GPU and on every shard; exact mode keeps the
                        // reference's single running sum (no per-part regrouping)
                        big = MT != 0 && erot == nullptr && !A.exact && (uint32_t)e.y >= (uint32_t)A.lut_min;
                    }
                }
            }
            if constexpr (ENGINE == ENGINE_TRAVERSE) {
                continue;
            } else {
                if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                    if (A.record != nullptr) {
                        // record mode: the cell, its global count and its base, in visit order
                        const bool has = c < n && (filt_d < 0 || digit(filt_d, list[c]) < filt_v);
                        uint32_t tot;
                        const uint32_t ex = block_excl_scan(S, has ? 1u : 0u, &tot);
                        unsigned long long g = 0;
                        if (has) {
                            const int4 e = list[c];
                            g = (uint32_t)e.y;
                            const uint32_t pos = nrec_q + ex;
                            if (pos < (uint32_t)A.record_cap)
                                A.record[(size_t)qi * A.record_cap + pos] =
                                    make_int4((int)((uint32_t)oi * (uint32_t)T + (uint32_t)oj), e.y, __float_as_int(cb), 0);
                            else
                                S.err = 1;
                        }
                        ncand += block_sum_u64(S, g);
                        nrec_q += tot;
                        __syncthreads();
                        continue;
                    }
                }
                uint32_t E;
                uint32_t ex = block_excl_scan(S, big ? 0u : lc, &E);
                S.cpre[threadIdx.x] = ex;
                S.coi[threadIdx.x] = oi;
                S.coj[threadIdx.x] = oj;
                S.cstart[threadIdx.x] = lst;
                S.cbase[threadIdx.x] = cb;
                S.ccnt[threadIdx.x] = lc;
                if (big) S.bigs[atomicAdd(&S.nbig, 1u)] = (uint16_t)threadIdx.x;
                if constexpr (ENGINE == BPQ_ENGINE_HBPQ) {
                    if (erot != nullptr && lc > 0) {
                        // e_h = (q_h - c_h[row]) @ R_h per half (hbpq.py:326-331)
                        const int dh = A.dh;
                        float *er = erot + (size_t)threadIdx.x * A.D;
                        for (int h = 0; h < 2; h++) {
                            const float *R = h ? A.rot2 : A.rot1;
                            const float *cr = (h ? A.c2 : A.c1) + (size_t)(h ? oj : oi) * dh;
                            const float *qh = tab + h * dh;
                            for (int x = 0; x < dh; x++) {
                                if (R == nullptr) {
                                    er[h * dh + x] = __fsub_rn(qh[x], __ldg(cr + x));
                                } else {
                                    float acc = 0.f;
                                    for (int y = 0; y < dh; y++)
                                        acc = fmaf(__fsub_rn(qh[y], __ldg(cr + y)), __ldg(R + (size_t)y * dh + x), acc);
                                    er[h * dh + x] = acc;
                                }
                            }
                        }
                    }
                }
                __syncthreads();
                ncand += E;
                for (uint32_t e0 = 0; e0 < E; e0 += NT * kUnroll) {
                    uint32_t entry[kUnroll];
                    int own[kUnroll];
                    uint32_t w[kUnroll][4];
                    float ptv[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; u++) {
                        const uint32_t e = e0 + u * NT + threadIdx.x;
                        own[u] = -1;
                        if (e < E) {
                            int lo = 0, hi = NT;
                            while (hi - lo > 1) {
                                int mid = (lo + hi) >> 1;
                                if (S.cpre[mid] <= e) lo = mid; else hi = mid;
                            }
                            own[u] = lo;
                            entry[u] = S.cstart[lo] + (e - S.cpre[lo]);
                            // point-term FBPQ at M = 8 / 16 reads the pre-rotated copy (dist_pt_plain)
                            const uint8_t *cbase_arr = (ENGINE == BPQ_ENGINE_FBPQ && rep_fold<MT>() && A.pterm)
                                                           ? A.codes_rot : A.codes;
                            load_code<MT>(cbase_arr + (size_t)entry[u] * M, w[u], M);
                            if constexpr (ENGINE == BPQ_ENGINE_FBPQ)
                                ptv[u] = A.pterm ? __ldg(A.pterm + entry[u]) : 0.f;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kUnroll; u++) {
                        if (own[u] < 0) continue;
                        const int lo = own[u];
                        float dist;
                        if constexpr (ENGINE == BPQ_ENGINE_FBPQ && rep_fold<MT>())
                            dist = A.pterm ? dist_pt_plain<MT>(tab, A.K, (int)(entry[u] & 31u), S.cbase[lo], ptv[u],
                                                               w[u])
                                           : dist_fbpq<MT>(A, tab, S.coi[lo], S.coj[lo], S.cbase[lo], w[u]);
                        else if constexpr (ENGINE == BPQ_ENGINE_FBPQ)
                            dist = A.pterm ? dist_fbpq_pt<MT>(tab, M, A.K, S.cbase[lo], ptv[u], w[u])
                                           : dist_fbpq<MT>(A, tab, S.coi[lo], S.coj[lo], S.cbase[lo], w[u]);
                        else
                            dist = dist_recon<ENGINE, MT>(A, tab, S.coi[lo], S.coj[lo], w[u],
                                                          erot ? erot + (size_t)lo * A.D : nullptr);
                        offer_lazy(dist, A.ids + entry[u]);
                    }
                    round_end();
                }
                if constexpr (ENGINE == BPQ_ENGINE_FBPQ && MT != 0) {
                    if (A.pterm != nullptr) {
                        if (S.nbig) defer_big(S.nbig);
                    } else {
                        const uint32_t nb = S.nbig;
                        for (uint32_t x = 0; x < nb; x++) {
                            const int t = S.bigs[x];
                            ncand += S.ccnt[t];
                            scan_cell_lut(S.coi[t], S.coj[t], S.cstart[t], S.ccnt[t], S.cbase[t]);
                        }
                    }
                } else if constexpr ((ENGINE == BPQ_ENGINE_BASELINE || ENGINE == BPQ_ENGINE_HBPQ) && MT != 0) {
                    const uint32_t nb = S.nbig;
                    for (uint32_t x = 0; x < nb; x++) {
                        const int t = S.bigs[x];
                        ncand += S.ccnt[t];
                        scan_cell_recon_lut(S.coi[t], S.coj[t], S.cstart[t], S.ccnt[t]);
                    }
                } else if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                    const uint32_t nb = S.nbig;
                    for (uint32_t x = 0; x < nb; x++) {
                        const int t = S.bigs[x];
                        ncand += S.ccnt[t];
                        scan_cell_lut(S.coi[t], S.coj[t], S.cstart[t], S.ccnt[t], S.cbase[t]);
                    }
                }
                __syncthreads();
            }
        }
        if constexpr (ENGINE == ENGINE_TRAVERSE) __syncthreads();
        PROF(pv);
    }

    // first x in [lo, T) with base + k(x) > tau, galloping from lo (every x
    // below lo is already known to satisfy base + k(x) <= tau)
    template <bool ALONG_ROW>
    __device__ __forceinline__ int gallop(double base, int lo, double tau) const {
        auto kk = [&](int x) { return ALONG_ROW ? k2(x) : k1(x); };
        if (lo >= T || !(base + kk(lo) <= tau)) return lo;
        int p = lo, step = 1, hi = T;
        for (;;) {
            const int q = p + step;
            if (q >= T) break;
            if (base + kk(q) <= tau) {
                p = q;
                step <<= 1;
            } else {
                hi = q;
                break;
            }
        }
        int l2 = p + 1, h2 = hi;
        while (l2 < h2) {
            const int mid = (l2 + h2) >> 1;
            if (base + kk(mid) <= tau) l2 = mid + 1; else h2 = mid;
        }
        return l2;
    }

    __device__ __forceinline__ int row_lo(const int32_t *rowB, int RA, int a) const { return a < RA ? rowB[a] : a; }
    __device__ __forceinline__ int col_lo(const int32_t *colB, int CA, int b) const { return b < CA ? colB[b] : b + 1; }

    // First x in [lo, hi) where the monotone predicate turns false (hi if
    // never), found by the whole warp: one 32-wide galloping probe round,
    // then 32-ary narrowing -- about log32(range) + 1 dependent loads.
    template <class F>
    __device__ __forceinline__ int warp_first_false(F pred, int lo, int hi) const {
        const int lane = threadIdx.x & 31;
        if (lo >= hi) return lo;
        const long long p = (long long)lo + ((1ll << lane) - 1);
        const unsigned m = __ballot_sync(0xffffffffu, p < hi && pred((int)p));
        const int c = __popc(m);
        if (c == 0) return lo;
        int a = lo + (int)((1ll << (c - 1)) - 1);  // last true probe
        int b = c < 31 ? (int)min((long long)hi, (long long)lo + (1ll << c) - 1) : hi;
        while (b - a > 1) {
            const int step = (b - a + 31) / 32;
            const long long pp = (long long)a + (long long)(lane + 1) * step;
            const unsigned mm = __ballot_sync(0xffffffffu, pp < b && pred((int)pp));
            const int cc = __popc(mm);
            const int na = a + cc * step;
            b = (int)min((long long)b, (long long)a + (long long)(cc + 1) * step);
            a = na;
        }
        return b;
    }

    // Cells with key <= tau (block-uniform result); rowNew/colNew (optional)
    // receive the new boundaries of the active lines and S.cnt_nr/cnt_nc the
    // active line counts.  Few active lines (the common, thin staircase):
    // one warp per line; many: one thread per line with a galloping search.
    __device__ unsigned long long count_le(double tau, const int32_t *rowB, int RA, const int32_t *colB,
                                           int CA, int32_t *rowNew, int32_t *colNew) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp == 0) {
            const int nr = warp_first_false([&](int a) { return k1(a) + k2(a) <= tau; }, 0, T);
            const int nc = warp_first_false([&](int b) { return k1(b + 1) + k2(b) <= tau; }, 0, T - 1);
            if (lane == 0) {
                S.cnt_nr = nr;
                S.cnt_nc = nc;
            }
        }
        __syncthreads();
        const int nR = S.cnt_nr, nC = S.cnt_nc, nl = nR + nC;
        unsigned long long cnt = 0;
        if (nl <= 4 * NW) {
            for (int line = warp; line < nl; line += NW) {
                int B, start;
                if (line < nR) {
                    const int a = line;
                    const double ka = k1(a);
                    start = a;
                    B = warp_first_false([&](int x) { return ka + k2(x) <= tau; }, row_lo(rowB, RA, a), T);
                    if (rowNew && lane == 0) rowNew[a] = B;
                } else {
                    const int b = line - nR;
                    const double kb = k2(b);
                    start = b + 1;
                    B = warp_first_false([&](int x) { return k1(x) + kb <= tau; }, col_lo(colB, CA, b), T);
                    if (colNew && lane == 0) colNew[b] = B;
                }
                if (lane == 0) cnt += (unsigned)(B - start);
            }
        } else {
            for (int a = threadIdx.x; a < nR; a += NT) {
                const double ka = k1(a);
                const int B = gallop<true>(ka, row_lo(rowB, RA, a), tau);
                cnt += (unsigned)(B - a);
                if (rowNew) rowNew[a] = B;
            }
            for (int b = threadIdx.x; b < nC; b += NT) {
                const double kb = k2(b);
                const int Av = gallop<false>(kb, col_lo(colB, CA, b), tau);
                cnt += (unsigned)(Av - (b + 1));
                if (colNew) colNew[b] = Av;
            }
        }
        return block_sum_u64(S, cnt);
    }

    // C(tau) at NW thresholds at once: warp w evaluates S.mtau[w] over its
    // active lines.  Returns false when some threshold activates more than
    // kMultiLines lines (the caller then falls back to count_le).
    __device__ bool count_multi(const int32_t *rowB, int RA, const int32_t *colB, int CA) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const double tau = S.mtau[warp];
        const int nr = warp_first_false([&](int a) { return k1(a) + k2(a) <= tau; }, 0, T);
        const int nc = warp_first_false([&](int b) { return k1(b + 1) + k2(b) <= tau; }, 0, T - 1);
        unsigned long long cnt = 0;
        const bool ok = nr + nc <= kMultiLines;
        if (ok) {
            for (int line = 0; line < nr + nc; line++) {
                if (line < nr) {
                    const double ka = k1(line);
                    const int B = warp_first_false([&](int x) { return ka + k2(x) <= tau; }, row_lo(rowB, RA, line), T);
                    cnt += (unsigned)(B - line);
                } else {
                    const int b = line - nr;
                    const double kb = k2(b);
                    const int Av = warp_first_false([&](int x) { return k1(x) + kb <= tau; }, col_lo(colB, CA, b), T);
                    cnt += (unsigned)(Av - (b + 1));
                }
            }
        }
        if (lane == 0) S.mcnt[warp] = ok ? cnt : ~0ull;
        __syncthreads();
        bool all = true;
#pragma unroll
        for (int w = 0; w < NW; w++) all = all && S.mcnt[w] != ~0ull;
        return all;
    }

    // exact cutoff inside the final band (weighted select, then smem sort)
    __device__ void final_select(int4 *cur, int4 *other, int n, unsigned long long need) {
        PROF(PH_FINAL);
        lut_i = lut_j = -1;  // the sort arrays below alias the per-cell LUT
        for (int d = 0;; d++) {
            if (n <= kSortCap) {
                int P2 = 1;
                while (P2 < n) P2 <<= 1;
                for (int c = threadIdx.x; c < P2; c += NT) {
                    if (c < n) {
                        int4 e = cur[c];
                        skey[c] = (unsigned long long)__double_as_longlong(ekey(e));
                        slin[c] = (uint32_t)elin(e);
                    } else {
                        skey[c] = ~0ull;
                        slin[c] = ~0u;
                    }
                    sidx[c] = (uint16_t)c;
                }
                __syncthreads();
                if (n <= NT) {
                    // rank sort: (key, lin) pairs are unique (lin is the cell)
                    unsigned long long kc = 0;
                    uint32_t lc = 0;
                    int rank = 0;
                    const int c = threadIdx.x;
                    if (c < n) {
                        kc = skey[c];
                        lc = slin[c];
                        for (int y = 0; y < n; y++) {
                            const unsigned long long ky = skey[y];
                            rank += (ky < kc || (ky == kc && slin[y] < lc)) ? 1 : 0;
                        }
                    }
                    __syncthreads();
                    if (c < n) {
                        skey[rank] = kc;
                        slin[rank] = lc;
                        sidx[rank] = (uint16_t)c;
                    }
                    __syncthreads();
                } else {
                    bitonic_sort_cells(skey, slin, sidx, P2);
                }
                // first sorted position where the running count reaches need
                if (threadIdx.x == 0) S.nlist = 0xFFFFFFFFu;
                unsigned long long run = 0;
                for (int base = 0; base < n; base += NT) {
                    int pidx = base + threadIdx.x;
                    uint32_t g = pidx < n ? (uint32_t)cur[sidx[pidx]].y : 0u;
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
                if (threadIdx.x == 0) S.cut_key = skey[cut];
                for (int c = threadIdx.x; c <= cut; c += NT) other[c] = cur[sidx[c]];
                __syncthreads();
                lut_i = lut_j = -1;  // the sort overwrote the aliased LUT
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

    // Enumerate the band.  Segment r (seg[r] = {kind | sparse | line index,
    // lo | hi << 16, work prefix, list base}, segLine[r] = codeword) covers
    // cells [lo, hi) of one row (kind 0) or column (kind 1).  A dense
    // segment has one work unit per cell; a sparse one has one per populated
    // cell of its codeword's line, filtered by the cell's sorted position.
    // Each thread takes a contiguous run of work units with kEnumBatch
    // cell-table reads in flight.  Returns the band's global entry count.
    // Visit every populated cell of the band's segments: visit(ca, cb, lin,
    // global count, local start, local count) returns the weight to add.
    template <typename Visit>
    __device__ unsigned long long visit_band(const uint4 *seg, const uint32_t *segLine, int nseg, uint32_t swork,
                                             Visit visit) {
        unsigned long long wb = 0;
        const uint32_t per = (swork + NT - 1) / NT;
        uint32_t f = threadIdx.x * per;
        const uint32_t f1 = min(swork, f + per);
        if (f < f1) {
            int lo = 0, hi = nseg;  // largest r with pre <= f
            while (hi - lo > 1) {
                int mid = (lo + hi) >> 1;
                if (seg[mid].z <= f) lo = mid; else hi = mid;
            }
            int r = lo;
            uint4 sg = seg[r];
            uint32_t line = segLine[r];
            uint32_t u = f - sg.z;
            uint32_t nxt = (r + 1 < nseg) ? seg[r + 1].z : swork;
            while (f < f1) {
                int ca[kEnumBatch], cbv[kEnumBatch];
                unsigned long long lin[kEnumBatch];
                bool ok[kEnumBatch];
#pragma unroll
                for (int x = 0; x < kEnumBatch; x++) {
                    ok[x] = false;
                    if (f < f1) {
                        if (f >= nxt) {
                            r++;
                            sg = seg[r];
                            line = segLine[r];
                            u = 0;
                            nxt = (r + 1 < nseg) ? seg[r + 1].z : swork;
                        }
                        const bool col = (sg.x >> 31) != 0, sparse = ((sg.x >> 30) & 1) != 0;
                        const int idx = (int)(sg.x & 0xFFFF);
                        const int slo = (int)(sg.y & 0xFFFF), shi = (int)(sg.y >> 16);
                        if (!sparse) {
                            const int v = slo + (int)u;
                            ca[x] = col ? v : idx;
                            cbv[x] = col ? idx : v;
                            lin[x] = col ? (unsigned long long)__ldg(o1 + v) * T + line
                                         : (unsigned long long)line * T + (unsigned)__ldg(o2 + v);
                            ok[x] = true;
                        } else if (!col) {
                            const uint32_t j = A.rowcols[sg.w + u];
                            const int b = __ldg(p2 + j);
                            ca[x] = idx;
                            cbv[x] = b;
                            lin[x] = (unsigned long long)line * T + j;
                            ok[x] = b >= slo && b < shi;
                        } else {
                            const uint32_t i = A.colrows[sg.w + u];
                            const int a = __ldg(p1 + i);
                            ca[x] = a;
                            cbv[x] = idx;
                            lin[x] = (unsigned long long)i * T + line;
                            ok[x] = a >= slo && a < shi;
                        }
                        u++;
                        f++;
                    }
                }
                OffT g0[kEnumBatch], g1[kEnumBatch];
#pragma unroll
                for (int x = 0; x < kEnumBatch; x++) {
                    if (ok[x]) {
                        g0[x] = __ldg(A.goff + lin[x]);
                        g1[x] = __ldg(A.goff + lin[x] + 1);
                    }
                }
#pragma unroll
                for (int x = 0; x < kEnumBatch; x++) {
                    if (ok[x] && g1[x] > g0[x]) {
                        uint32_t lst, lcn;
                        if (A.sharded) {
                            OffT l0 = __ldg(A.loff + lin[x]), l1 = __ldg(A.loff + lin[x] + 1);
                            lst = (uint32_t)l0;
                            lcn = (uint32_t)(l1 - l0);
                        } else {
                            lst = (uint32_t)g0[x];
                            lcn = (uint32_t)(g1[x] - g0[x]);
                        }
                        wb += visit(ca[x], cbv[x], lin[x], (uint32_t)(g1[x] - g0[x]), lst, lcn);
                    }
                }
            }
        }
        return block_sum_u64(S, wb);
    }

    // Append the band's populated cells to list (at most kBandCap: S.nlist
    // counts them all, so the caller detects an overflow).
    __device__ unsigned long long enumerate_band(const uint4 *seg, const uint32_t *segLine, int nseg,
                                                 uint32_t swork, int4 *list) {
        return visit_band(seg, segLine, nseg, swork,
                          [&](int ca, int cb, unsigned long long, uint32_t gc, uint32_t lst, uint32_t lcn) {
                              const uint32_t pos = atomicAdd(&S.nlist, 1u);
                              if (pos < (uint32_t)kBandCap)
                                  list[pos] = make_int4((ca << 16) | cb, (int)gc, (int)lst, (int)lcn);
                              return (unsigned long long)gc;
                          });
    }

    // A band holding more than kBandCap populated cells (a tie plateau: one
    // key value shared by that many cells, which no key threshold can split)
    // is taken in windows of the reference heap's full order (key, oi * T +
    // oj): each window's upper bound is the kBandCap-th smallest composite key
    // above the previous window, found by an MSB radix select whose digit
    // histograms re-enumerate the band (12 passes over 8 key + 4 lin bytes).
    // Returns true when the cutoff fell inside the band (query done), false
    // when the whole band was scanned (W updated).
    __device__ __noinline__ bool plateau_windows(const uint4 *seg, const uint32_t *segLine, int nseg, uint32_t swork,
                                    int4 *listA, int4 *listB, unsigned long long &W, unsigned long long L) {
        unsigned long long lo_k = 0;
        uint32_t lo_l = 0;
        bool have_lo = false;
        auto above_lo = [&](unsigned long long kb, uint32_t ln) {
            return !have_lo || kb > lo_k || (kb == lo_k && ln > lo_l);
        };
        for (;;) {
            // kBandCap-th smallest composite key above lo, digit by digit
            unsigned long long pk = 0, mk = 0;  // key-byte prefix / mask
            uint32_t pl = 0, ml = 0;            // lin-byte prefix / mask
            uint32_t rank = (uint32_t)kBandCap;
            bool all = false;
            for (int d = 0; d < 12; d++) {
                for (int i = threadIdx.x; i < 256; i += NT) S.hist_c[i] = 0;
                __syncthreads();
                visit_band(seg, segLine, nseg, swork,
                           [&](int ca, int cb, unsigned long long lin, uint32_t, uint32_t, uint32_t) {
                               const unsigned long long kb = (unsigned long long)__double_as_longlong(key(ca, cb));
                               const uint32_t ln = (uint32_t)lin;
                               if (above_lo(kb, ln) && (kb & mk) == pk && (ln & ml) == pl) {
                                   const int v = d < 8 ? (int)((kb >> (56 - 8 * d)) & 0xFF)
                                                       : (int)((ln >> (24 - 8 * (d - 8))) & 0xFF);
                                   atomicAdd(&S.hist_c[v], 1u);
                               }
                               return 0ull;
                           });
                __syncthreads();
                if (threadIdx.x == 0) {
                    uint32_t run = 0, tot = 0;
                    for (int v = 0; v < 256; v++) tot += S.hist_c[v];
                    S.sel_v = -1;
                    if (d == 0 && tot <= rank) {
                        S.sel_v = 256;  // everything left fits in one window
                    } else {
                        for (int v = 0; v < 256; v++) {
                            if (run + S.hist_c[v] >= rank) {
                                S.sel_v = v;
                                S.tsel_below = run;
                                break;
                            }
                            run += S.hist_c[v];
                        }
                    }
                }
                __syncthreads();
                const int v = S.sel_v;
                if (v == 256) {
                    all = true;
                    break;
                }
                rank -= (uint32_t)S.tsel_below;
                if (d < 8) {
                    pk |= (unsigned long long)v << (56 - 8 * d);
                    mk |= 0xFFull << (56 - 8 * d);
                } else {
                    pl |= (uint32_t)v << (24 - 8 * (d - 8));
                    ml |= 0xFFu << (24 - 8 * (d - 8));
                }
                __syncthreads();
            }
            // the window (lo, hi] into listA
            if (threadIdx.x == 0) S.nlist = 0;
            __syncthreads();
            const unsigned long long wb = visit_band(
                seg, segLine, nseg, swork,
                [&](int ca, int cb, unsigned long long lin, uint32_t gc, uint32_t lst, uint32_t lcn) {
                    const unsigned long long kb = (unsigned long long)__double_as_longlong(key(ca, cb));
                    const uint32_t ln = (uint32_t)lin;
                    if (!above_lo(kb, ln) || !(all || kb < pk || (kb == pk && ln <= pl))) return 0ull;
                    const uint32_t pos = atomicAdd(&S.nlist, 1u);
                    if (pos < (uint32_t)kBandCap) listA[pos] = make_int4((ca << 16) | cb, (int)gc, (int)lst, (int)lcn);
                    return (unsigned long long)gc;
                });
            const int n = (int)min(S.nlist, (uint32_t)kBandCap);
            if (W + wb < L) {
                emit(listA, n, -1, 0);
                W += wb;
                if (all) return false;
                lo_k = pk;
                lo_l = pl;
                have_lo = true;
                __syncthreads();
            } else {
                final_select(listA, listB, n, L - W);
                return true;
            }
        }
    }

    // ------------------------------------------------------------------
    // Sparse-table traversal (populated-cell lists present).  Lines become
    // active in order of their diagonal key (row a: key(a, a); column b:
    // key(b + 1, b)); activating a line moves its populated cells of its half
    // of the staircase into a pending pool.  With kappa = the smallest
    // activation key of a line not yet active, every populated cell with
    // key < kappa is in the pool, so those cells form the next band: scanned
    // whole while the running total stays < L, else the exact cutoff is
    // selected inside them.  No threshold search and no empty cell is ever
    // touched.  Returns false (nothing emitted) if the pool would overflow;
    // the caller then falls back to the band traversal.
    // Lazily extend half h's sorted prefix to at least `need` positions: the
    // next E smallest (r bits, codeword) keys after the current last one are
    // found by an MSB radix select over the unsorted r, bitonic-sorted in
    // shared memory and appended to sr/ord.  Only queries whose traversal
    // outgrows the partial sort pay for it.
    __device__ void extend(int h, int need) {
        lut_i = lut_j = -1;  // the sort arrays below alias the per-cell LUT
        int tp = h ? tp2 : tp1;
        const float *u = h ? u2 : u1;
        float *srw = const_cast<float *>(reinterpret_cast<const float *>(h ? sr2 : sr1));
        int32_t *ow = const_cast<int32_t *>(h ? o2 : o1);
        need = min(need, T);
        while (tp < need) {
            const int E = min(T - tp, kSortCap);
            const bool any = tp == 0;
            const unsigned long long klast =
                any ? 0ull : ((unsigned long long)__float_as_uint(srw[tp - 1]) << 32) | (uint32_t)ow[tp - 1];
            unsigned long long prefix = 0, pmask = 0;
            uint32_t rank = (uint32_t)E;
            for (int shift = 56; shift >= 0; shift -= 8) {
                for (int i = threadIdx.x; i < 256; i += NT) S.hist_c[i] = 0;
                __syncthreads();
                for (int x = threadIdx.x; x < T; x += NT) {
                    const unsigned long long key = ((unsigned long long)__float_as_uint(__ldg(u + x)) << 32) | (uint32_t)x;
                    if ((any || key > klast) && (key & pmask) == prefix)
                        atomicAdd(&S.hist_c[(key >> shift) & 0xFF], 1u);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    uint32_t run = 0;
                    for (int d = 0; d < 256; d++) {
                        if (run + S.hist_c[d] >= rank) {
                            S.tsel_v = d;
                            S.tsel_below = run;
                            break;
                        }
                        run += S.hist_c[d];
                    }
                }
                __syncthreads();
                rank -= (uint32_t)S.tsel_below;
                prefix |= (unsigned long long)S.tsel_v << shift;
                pmask |= 0xFFull << shift;
                __syncthreads();
            }
            const unsigned long long kE = prefix;  // E-th smallest key after klast
            if (threadIdx.x == 0) S.tcnt = 0;
            __syncthreads();
            for (int x = threadIdx.x; x < T; x += NT) {
                const unsigned long long key = ((unsigned long long)__float_as_uint(__ldg(u + x)) << 32) | (uint32_t)x;
                if ((any || key > klast) && key <= kE) skey[atomicAdd(&S.tcnt, 1u)] = key;
            }
            __syncthreads();
            int P2 = 1;
            while (P2 < E) P2 <<= 1;
            for (int i = E + threadIdx.x; i < P2; i += NT) skey[i] = ~0ull;
            __syncthreads();
            bitonic_sort_u64(skey, P2);
            for (int i = threadIdx.x; i < E; i += NT) {
                const unsigned long long kv = skey[i];
                srw[tp + i] = __uint_as_float((uint32_t)(kv >> 32));
                ow[tp + i] = (int32_t)(kv & 0xFFFFFFFFull);
            }
            __syncthreads();
            tp += E;
        }
        if (h) tp2 = tp; else tp1 = tp;
    }

    __device__ __forceinline__ double act_row(int a) const { return a < T ? k1(a) + k2(a) : INFINITY; }
    __device__ __forceinline__ double act_col(int b) const { return b < T - 1 ? k1(b + 1) + k2(b) : INFINITY; }

    // Returns 1 when done, 0 when the pool overflowed (nothing emitted is
    // kept: the caller restarts with the band traversal), 2 when activation
    // needs more sorted positions than the partial sort provided (the query
    // is queued for the full-sort retry pass).
    __device__ int run_sparse(int4 *band, int4 *pend, int4 *pend2, int4 *other) {
        const unsigned long long L = (unsigned long long)A.L;
        tp1 = A.plen ? A.plen[qi * 2] : A.topP;
        tp2 = A.plen ? A.plen[qi * 2 + 1] : A.topP;
        const bool partial = tp1 < T || tp2 < T;
        cw = true;
        unsigned long long W = 0;
        int nr = 0, nc = 0, npend = 0;
        int NB = A.nb0;
        for (;;) {
            // the batch probes rows < nr + NB and columns < nc + NB (column b
            // reads position b + 1): stay inside the sorted prefix
            if (partial) {
                const int need = max(nr + NB, nc + NB + 1) + 1;
                if (need > tp1 || need > tp2) PROF(PH_EXTEND);
                if (need > tp1) extend(0, need);
                if (need > tp2) extend(1, need);
            }
            PROF(PH_BOUNDS);
            // next NB lines in activation order (merge path over the two sequences)
            if (threadIdx.x < 32) {
                const int x = warp_first_false(
                    [&](int xx) { return act_row(nr + xx) <= act_col(nc + NB - 1 - xx); }, 0, NB);
                if (threadIdx.x == 0) {
                    S.cnt_nr = min(nr + x, T);
                    S.cnt_nc = min(nc + (NB - x), T - 1);
                }
            }
            __syncthreads();
            const int nr2 = S.cnt_nr, nc2 = S.cnt_nc;
            const double kappa = fmin(act_row(nr2), act_col(nc2));
            if (threadIdx.x == 0) {
                S.nlist = 0;
                S.tcnt = 0;
            }
            __syncthreads();
            // gather newly active lines' cells (one line per thread, flattened)
            PROF(PH_ENUM);
            unsigned long long wb = 0;
            const int nnew = (nr2 - nr) + (nc2 - nc);
            for (int base = 0; base < nnew; base += NT) {
                const int v = base + threadIdx.x;
                uint32_t nnz = 0, p0 = 0, line = 0;
                int idx = 0;
                bool col = false;
                if (v < nnew) {
                    col = v >= nr2 - nr;
                    idx = col ? nc + (v - (nr2 - nr)) : nr + v;
                    line = (uint32_t)(col ? o2 : o1)[idx];
                    const uint32_t *ptr = col ? A.colptr : A.rowptr;
                    p0 = __ldg(ptr + line);
                    nnz = __ldg(ptr + line + 1) - p0;
                }
                uint32_t E;
                const uint32_t ex = block_excl_scan(S, nnz, &E);
                S.cpre[threadIdx.x] = ex;
                S.cstart[threadIdx.x] = p0;
                S.coi[threadIdx.x] = (int)line;
                S.coj[threadIdx.x] = col ? -(idx + 1) : idx;
                __syncthreads();
                for (uint32_t e = threadIdx.x; e < E; e += NT) {
                    int lo = 0, hi = NT;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (S.cpre[mid] <= e) lo = mid; else hi = mid;
                    }
                    const uint32_t t = S.cstart[lo] + (e - S.cpre[lo]);
                    const uint32_t ln = (uint32_t)S.coi[lo];
                    const int tag = S.coj[lo];
                    uint32_t ci, cj;
                    bool own;
                    if (tag >= 0) {  // row position a = tag owns columns of rank >= a
                        const int a = tag;
                        cj = A.rowcols[t];
                        ci = ln;
                        const float rj = __ldg(u2 + cj), ra = (float)k2(a);
                        const uint32_t oa = (uint32_t)o2[a];
                        own = rj > ra || (rj == ra && cj >= oa);
                    } else {  // column position b owns rows of rank > b
                        const int b = -tag - 1;
                        ci = A.colrows[t];
                        cj = ln;
                        const float ri = __ldg(u1 + ci), rb = (float)k1(b);
                        const uint32_t ob = (uint32_t)o1[b];
                        own = ri > rb || (ri == rb && ci > ob);
                    }
                    if (!own) continue;
                    const unsigned long long lin = (unsigned long long)ci * T + cj;
                    const OffT g0 = __ldg(A.goff + lin), g1 = __ldg(A.goff + lin + 1);
                    if (!(g1 > g0)) continue;
                    uint32_t lst, lcn;
                    if (A.sharded) {
                        const OffT l0 = __ldg(A.loff + lin), l1 = __ldg(A.loff + lin + 1);
                        lst = (uint32_t)l0;
                        lcn = (uint32_t)(l1 - l0);
                    } else {
                        lst = (uint32_t)g0;
                        lcn = (uint32_t)(g1 - g0);
                    }
                    const int4 cell = make_int4((int)((ci << 16) | cj), (int)(uint32_t)(g1 - g0), (int)lst, (int)lcn);
                    if ((double)__ldg(u1 + ci) + (double)__ldg(u2 + cj) < kappa) {
                        const uint32_t pos = atomicAdd(&S.nlist, 1u);
                        if (pos < (uint32_t)kBandCap) band[pos] = cell;
                        wb += (unsigned long long)(g1 - g0);
                    } else {
                        const uint32_t pos = atomicAdd(&S.tcnt, 1u);
                        if (pos < (uint32_t)kBandCap) pend2[pos] = cell;
                    }
                }
                __syncthreads();
            }
            // re-classify the pool against the new kappa
            PROF(PH_TAU);
            for (int c = threadIdx.x; c < npend; c += NT) {
                const int4 cell = pend[c];
                if (ekey(cell) < kappa) {
                    const uint32_t pos = atomicAdd(&S.nlist, 1u);
                    if (pos < (uint32_t)kBandCap) band[pos] = cell;
                    wb += (unsigned long long)(uint32_t)cell.y;
                } else {
                    const uint32_t pos = atomicAdd(&S.tcnt, 1u);
                    if (pos < (uint32_t)kBandCap) pend2[pos] = cell;
                }
            }
            wb = block_sum_u64(S, wb);
            const uint32_t nband = S.nlist, npend2 = S.tcnt;
            if (nband > (uint32_t)kBandCap || npend2 > (uint32_t)kBandCap) return 0;
            if (W + wb < L) {
                emit(band, (int)nband, -1, 0);
                W += wb;
                if (!(kappa < INFINITY)) {
                    popped = (unsigned long long)T * T;
                    return 1;
                }
            } else {
                final_select(band, other, (int)nband, L - W);
                if (A.out_popped) {
                    __syncthreads();
                    popped = count_le(__longlong_as_double((long long)S.cut_key), nullptr, 0, nullptr, 0,
                                      nullptr, nullptr);
                }
                return 1;
            }
            int4 *t = pend;
            pend = pend2;
            pend2 = t;
            npend = (int)npend2;
            nr = nr2;
            nc = nc2;
            NB = min(NB * 2, NT);
            __syncthreads();
        }
    }

    __device__ void run() {
        char *scr = A.scratch + (size_t)blockIdx.x * A.stride;
        int32_t *rowB = reinterpret_cast<int32_t *>(scr);
        int32_t *colB = rowB + T;
        int32_t *rowNew = colB + T;
        int32_t *colNew = rowNew + T;
        uint32_t *segLine = reinterpret_cast<uint32_t *>(colNew + T);
        uint4 *seg = reinterpret_cast<uint4 *>(scr + (((size_t)6 * T * 4 + 15) & ~(size_t)15));
        int4 *listA = reinterpret_cast<int4 *>(seg + 2 * T);
        int4 *listB = listA + kBandCap;
        int4 *listC = listB + kBandCap;
        int4 *listD = listC + kBandCap;
        if constexpr (ENGINE == BPQ_ENGINE_HBPQ)
            erot = (A.rot1 != nullptr || A.rot2 != nullptr) ? reinterpret_cast<float *>(listD + kBandCap) : nullptr;

        if (threadIdx.x == 0) {
            S.ntk = 0;
            S.thr = ~0ull;
            S.err = 0;
        }
        __syncthreads();
        if (A.n_global == 0) return;
        if (SPARSE_ONLY || (A.rowptr != nullptr && A.ru1 != nullptr)) {
            const int rs = run_sparse(listA, listB, listC, listD);
            if (rs == 1) return;
            cw = false;
            if (SPARSE_ONLY || rs == 2 || A.plen != nullptr || A.topP < T) {
                // needs the full sort: queue for the retry pass (outputs written there)
                if (threadIdx.x == 0) {
                    S.err = 2;
                    A.retry_list[atomicAdd(A.retry_count, 1u)] = (unsigned int)qi;
                }
                __syncthreads();
                return;
            }
            // pool overflow: restart this query with the band traversal
            ncand = 0;
            popped = 0;
            nbig_q = 0;
            nrec_q = 0;
            if (threadIdx.x == 0) {
                S.ntk = 0;
                S.thr = ~0ull;
            }
            __syncthreads();
        }

        if constexpr (!SPARSE_ONLY) run_dense(rowB, colB, rowNew, colNew, segLine, seg, listA, listB, listC, listD);
    }

    __device__ void run_dense(int32_t *rowB, int32_t *colB, int32_t *rowNew, int32_t *colNew, uint32_t *segLine,
                              uint4 *seg, int4 *listA, int4 *listB, int4 *listC, int4 *listD) {
        const bool lists = A.rowptr != nullptr;
        const unsigned long long Tall = (unsigned long long)T * T;
        const unsigned long long L = (unsigned long long)A.L;
        unsigned long long W = 0, Cprev = 0;
        int RA = 0, CA = 0;  // lines whose boundary arrays are initialised
        double tauLo = -1.0;
        const double maxKey = key(T - 1, T - 1);
        const double k00 = key(0, 0);
        double target = (double)L / A.rho * 0.5;
        for (;;) {
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
                PROF(PH_TAU);
                // multi-probe rounds: NW thresholds per round, one per warp
                for (int round = 0; round < 8 && !accepted; round++) {
                    const double xlo = fmax(lo - k00, 0.0), xhi = hi - k00;
                    if (!(xhi > 0.0)) break;
                    __syncthreads();  // previous round's S.mtau / S.mcnt fully consumed
                    if (threadIdx.x < NW) {
                        const int w = threadIdx.x;
                        double x;
                        if (xlo > 0.0) {
                            x = xlo * pow(xhi / xlo, (double)(w + 1) / (NW + 1));
                        } else {
                            const double fr[NW] = {1.0 / 4096, 1.0 / 1024, 1.0 / 256, 1.0 / 64,
                                                   1.0 / 16, 1.0 / 4, 0.5, 0.75};
                            x = xhi * fr[w];
                        }
                        double t = k00 + x;
                        if (!(t > lo)) t = lo + (hi - lo) * (w + 1) / (NW + 1);
                        if (!(t < hi)) t = hi;
                        S.mtau[w] = t;
                    }
                    __syncthreads();
                    if (!count_multi(rowB, RA, colB, CA)) break;
                    // best accepted probe, else the tightest bracket
                    double nlo = lo, nhi = hi;
                    unsigned long long nclo = clo, nchi = chi;
                    int acc_w = -1;
                    for (int w = 0; w < NW; w++) {
                        const double t = S.mtau[w];
                        const unsigned long long cm = S.mcnt[w];
                        if (!(t > lo && t < hi)) continue;
                        const double band = (double)(cm - Cprev);
                        if (band > target) {
                            if (t < nhi) { nhi = t; nchi = cm; }
                        } else if (band < 0.5 * target) {
                            if (t > nlo) { nlo = t; nclo = cm; }
                        } else {
                            acc_w = w;  // largest accepted probe wins
                        }
                    }
                    if (acc_w >= 0) {
                        tauHi = S.mtau[acc_w];
                        cHi = S.mcnt[acc_w];
                        accepted = true;
                    } else {
                        if (nlo == lo && nhi == hi) break;  // no progress possible
                        lo = nlo;
                        hi = nhi;
                        clo = nclo;
                        chi = nchi;
                    }
                }
                for (int it = 0; it < 200 && !accepted; it++) {
                    const double xlo = fmax(lo - k00, 0.0), xhi = hi - k00;
                    if (!(xhi > 0.0)) break;
                    double mid;
                    if ((it & 1) == 0 && clo > 0 && xlo > 0.0) {
                        // secant on log C(tau) against log(tau - key00)
                        double ylo = log((double)clo), yhi = log((double)chi), yw = log(want);
                        double fr = (yw - ylo) / fmax(yhi - ylo, 1e-30);
                        fr = fmin(fmax(fr, 0.02), 0.98);
                        mid = k00 + exp(log(xlo) + (log(xhi) - log(xlo)) * fr);
                    } else {
                        // geometric bisection of (tau - key00)
                        double xl = xlo > 0.0 ? xlo : xhi * 1e-6;
                        mid = k00 + sqrt(xl * xhi);
                    }
                    if (!(mid > lo && mid < hi)) {
                        mid = lo + 0.5 * (hi - lo);
                        if (!(mid > lo && mid < hi)) break;
                    }
                    unsigned long long cm = count_le(mid, rowB, RA, colB, CA, nullptr, nullptr);
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
                // cHi - Cprev > kBandCap: a single key value shared by more than
                // kBandCap cells; the populated ones are counted below
            }
            // new line boundaries at tauHi and the active line counts
            PROF(PH_BOUNDS);
            count_le(tauHi, rowB, RA, colB, CA, rowNew, colNew);
            const int nR = S.cnt_nr, nC = S.cnt_nc;
            // compact the band's non-empty segments with their work counts
            uint32_t swork = 0, nseg = 0;
            for (int base = 0; base < nR + nC; base += NT) {
                const int v = base + threadIdx.x;
                uint32_t len = 0, work = 0, lo = 0, hi = 0, ln = 0, lb = 0, hdr = 0;
                bool sparse = false;
                if (v < nR) {
                    lo = (uint32_t)row_lo(rowB, RA, v);
                    hi = (uint32_t)rowNew[v];
                    len = hi - lo;
                    if (len) {
                        ln = (uint32_t)__ldg(o1 + v);
                        if (lists) {
                            const uint32_t p0 = __ldg(A.rowptr + ln), pe = __ldg(A.rowptr + ln + 1);
                            sparse = pe - p0 < len;
                            lb = p0;
                            work = sparse ? pe - p0 : len;
                        } else {
                            work = len;
                        }
                        hdr = (sparse ? (1u << 30) : 0u) | (uint32_t)v;
                    }
                } else if (v < nR + nC) {
                    const int b = v - nR;
                    lo = (uint32_t)col_lo(colB, CA, b);
                    hi = (uint32_t)colNew[b];
                    len = hi - lo;
                    if (len) {
                        ln = (uint32_t)__ldg(o2 + b);
                        if (lists) {
                            const uint32_t p0 = __ldg(A.colptr + ln), pe = __ldg(A.colptr + ln + 1);
                            sparse = pe - p0 < len;
                            lb = p0;
                            work = sparse ? pe - p0 : len;
                        } else {
                            work = len;
                        }
                        hdr = (1u << 31) | (sparse ? (1u << 30) : 0u) | (uint32_t)b;
                    }
                }
                uint32_t tot, totr;
                const uint32_t ex = block_excl_scan(S, work, &tot);
                const uint32_t exr = block_excl_scan(S, work > 0 ? 1u : 0u, &totr);
                if (work > 0) {
                    seg[nseg + exr] = make_uint4(hdr, lo | (hi << 16), swork + ex, lb);
                    segLine[nseg + exr] = ln;
                }
                swork += tot;
                nseg += totr;
            }
            if (threadIdx.x == 0) S.nlist = 0;
            __syncthreads();
            PROF(PH_ENUM);
            const unsigned long long wb = enumerate_band(seg, segLine, (int)nseg, swork, listA);
            const int n = (int)S.nlist;
            bool consumed;
            if (n > kBandCap) {
                // tie plateau: more populated cells than one band holds
                if (plateau_windows(seg, segLine, (int)nseg, swork, listA, listB, W, L)) {
                    if (A.out_popped) {
                        __syncthreads();
                        popped = count_le(__longlong_as_double((long long)S.cut_key), rowB, RA, colB, CA,
                                          nullptr, nullptr);
                    }
                    break;
                }
                consumed = true;
            } else {
                consumed = W + wb < L;
                if (consumed) {
                    emit(listA, n, -1, 0);
                    W += wb;
                }
            }
            if (consumed) {
                Cprev = cHi;
                for (int a = threadIdx.x; a < nR; a += NT) rowB[a] = rowNew[a];
                for (int b = threadIdx.x; b < nC; b += NT) colB[b] = colNew[b];
                __syncthreads();
                RA = max(RA, nR);
                CA = max(CA, nC);
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
                    popped = count_le(__longlong_as_double((long long)S.cut_key), rowB, RA, colB, CA,
                                      nullptr, nullptr);
                }
                break;
            }
        }
    }

    __device__ void finish() {
        if constexpr (ENGINE == ENGINE_TRAVERSE) return;
        PROF(PH_FINISH);
        __syncthreads();
        const int k = A.k;
        const int64_t qo = A.q0 + qi;
        if (S.err == 2) return;  // re-run by the full-sort retry pass
        if (A.record != nullptr) {  // record mode: the visited cells are the output
            if (threadIdx.x == 0) {
                A.record_n[qi] = S.err ? 0xFFFFFFFFu : nrec_q;
                if (A.out_ncand) A.out_ncand[qo] = S.err ? -1 : (int64_t)ncand;
                if (A.out_popped) A.out_popped[qo] = S.err ? -1 : (int64_t)popped;
            }
            return;
        }
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
        topk_compact(S, tk, k);
        if (A.big_cells != nullptr && nbig_q > 0) {
            // large cells pending: hand the small cells' top-k to big_scan_kernel
            const uint32_t n = S.ntk;
            for (uint32_t x = threadIdx.x; x < n; x += NT) A.tk_part[(size_t)qi * k + x] = tk[x];
            if (threadIdx.x == 0) {
                A.tk_n[qi] = n;
                A.big_n[qi] = nbig_q;
                A.ncand_q[qi] = ncand;
                if (A.out_ncand) A.out_ncand[qo] = (int64_t)ncand;
                if (A.out_popped) A.out_popped[qo] = (int64_t)popped;
                A.bigq_list[atomicAdd(A.bigq_count, 1u)] = (unsigned int)qi;
            }
            return;
        }
        write_topk(S, tk, k, ncand, A.out_d + qo * k, A.out_ids + qo * k, A.out_count + qo);
        if (threadIdx.x == 0) {
            if (A.out_ncand) A.out_ncand[qo] = (int64_t)ncand;
            if (A.out_popped) A.out_popped[qo] = (int64_t)popped;
        }
    }
};

template <int ENGINE, int MT, typename KT, typename OffT, bool SPARSE_ONLY = false>
__global__ void __launch_bounds__(NT, BPQ_MINB) search_kernel(Args<KT, OffT> A) {
    const int M = MT ? MT : A.M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    float *tab = reinterpret_cast<float *>(smem_raw + sizeof(Smem));
    // per-cell LUT / cp.async stages (FBPQ) and the sort arrays share the region after the table
    float *lut = tab + (ENGINE == BPQ_ENGINE_FBPQ ? M * A.K : ((A.D + 3) & ~3));
    KT *s1s = reinterpret_cast<KT *>(tab + A.tab_floats);
    KT *s2s = s1s + A.sr_smem;
    if (threadIdx.x == 0) {
        // large-cell stage barriers: one arrival (the issuing thread's expect_tx) per chunk
        for (int s = 0; s < kBigS; s++) mbar_init(&S.mbar[s], 1);
        S.tphase = 0;
        mbar_fence_init();
    }
#ifdef BPQ_PHASE_PROF
    if (threadIdx.x == 0) {
        S.prof_ph = PH_IDLE;
        S.prof_t = clock64();
    }
#endif
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned int c = atomicAdd(A.counter, 1u);
            if (A.qlist == nullptr) {
                S.qidx = (int64_t)c;
            } else {
                S.qidx = c < *A.qlist_count ? (int64_t)A.qlist[c] : A.nq;
            }
        }
        __syncthreads();
        const int64_t qi = S.qidx;
        if (qi >= A.nq) {
            PROF(PH_IDLE);
            return;
        }
        PROF(PH_PROLOGUE);
        // stage the sorted half-distance prefixes
        {
            const KT *g1 = A.sr1 + qi * A.T, *g2 = A.sr2 + qi * A.T;
            for (int i = threadIdx.x; i < A.sr_smem; i += NT) {
                s1s[i] = g1[i];
                s2s[i] = g2[i];
            }
        }
        if constexpr (ENGINE != ENGINE_TRAVERSE) {
            const float *q = A.queries + qi * A.D;
            if constexpr (ENGINE == BPQ_ENGINE_FBPQ) {
                // fold = fine_norms - 2 * (book . q_p) (fbpq.py:140-143), from fold_kernel
                const float *fq = A.fold + (size_t)qi * M * A.K;
                if (((M * A.K) & 3) == 0) {
                    const float4 *src = reinterpret_cast<const float4 *>(fq);
                    float4 *dst = reinterpret_cast<float4 *>(tab);
                    for (int x = threadIdx.x; x < (M * A.K) / 4; x += NT) dst[x] = __ldg(src + x);
                } else {
                    for (int x = threadIdx.x; x < M * A.K; x += NT) tab[x] = __ldg(fq + x);
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
                for (int x = threadIdx.x; x < A.D; x += NT) tab[x] = __ldg(q + x);
            }
        }
        __syncthreads();
        Query<ENGINE, MT, KT, OffT, SPARSE_ONLY> Q(A, S, qi, tab, lut, s1s, s2s,
                                                   reinterpret_cast<unsigned long long *>(smem_raw + A.tk_off));
        Q.run();
        Q.finish();
        __syncthreads();
    }
}


// dynamic shared memory: Smem | per-query table | sorted-key prefixes | top-k buffer
size_t tk_offset(int tab_floats, int sr_smem, size_t kt_size) {
    return (sizeof(Smem) + (size_t)tab_floats * 4 + 2 * (size_t)sr_smem * kt_size + 15) & ~(size_t)15;
}
size_t dyn_smem_bytes(int tab_floats, int sr_smem, size_t kt_size, int tkcap) {
    return tk_offset(tab_floats, sr_smem, kt_size) + (size_t)tkcap * 8;
}
// top-k buffer: k rounded up to 256 plus one round of offers (the largest round is NT * kUnroll)
int topk_capacity(int k) { return ((k + 255) & ~255) + NT * kUnroll; }

int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 0;
        if (cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    }
    return g_num_sms;
}

template <int ENGINE, int MT, typename KT, typename OffT, bool SPARSE_ONLY = false>
int configure(size_t smem, int *n_cta_out) {
    static bool attr = false;
    auto kfn = search_kernel<ENGINE, MT, KT, OffT, SPARSE_ONLY>;
    if (!attr) {
        int dev = 0, optin = 0;
        BPQ_CUDA_TRY(cudaGetDevice(&dev));
        BPQ_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        BPQ_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
        attr = true;
    }
    int occ = 0;
    BPQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, NT, smem));
    if (occ < 1) return fail(BPQ_ERR_UNSUPPORTED, "search kernel shared memory does not fit on an SM");
    *n_cta_out = occ * num_sms();
    return BPQ_OK;
}

// the launch-independent kernel arguments (index, workspace, outputs)
template <int ENGINE, int MT>
void fill_args(Args<float, uint32_t> &A, const Index &ix, const float *queries, int64_t q0, int64_t nq,
               int64_t budget, int32_t k, const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids,
               int32_t *out_count, int64_t *out_ncand, int64_t *out_popped) {
    A.M = ix.M;
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
    A.exact = ix.exact;
    A.ids = ix.ids;
    A.codes = ix.codes;
    A.codes_rot = ix.codes_rot;
    A.books = ix.books;
    A.fine_norms = ix.fine_norms;
    A.cross1 = ix.cross1;
    A.cross2 = ix.cross2;
    A.pterm = ENGINE == BPQ_ENGINE_FBPQ ? ix.pterm : nullptr;
    A.lut_min = effective_lut_min();
    const int nb0_env = getenv("BPQ_NB0") ? atoi(getenv("BPQ_NB0")) : 0;  // A/B experiments (read per launch)
    // first sparse-traversal batch: small budgets stop within a few lines
    // first sparse-traversal batch: about 6x the populated cells the budget needs (the budget over the
    // mean entries per populated cell), 16..256 lines; without a populated count, by budget alone
    int nb0 = budget <= 2000 ? 32 : budget <= 5000 ? 64 : 128;
    if (ix.populated > 0 && ix.N_global > 0) {
        const double cells = (double)budget * (double)ix.populated / (double)ix.N_global;
        nb0 = 16;
        while (nb0 < NT && nb0 < 6.0 * cells) nb0 *= 2;
    }
    A.nb0 = nb0_env > 0 ? (nb0_env < NT ? nb0_env : NT) : nb0;
    A.bank1 = ix.bank1;
    A.bank2 = ix.bank2;
    A.rot1 = ix.rot1;
    A.rot2 = ix.rot2;
    A.n_global = (unsigned long long)ix.N_global;
    A.n_local = (uint32_t)ix.N;
    A.rho = (double)(ix.N_global > 0 ? ix.N_global : 1) / ((double)ix.T * ix.T);
    A.queries = queries;
    A.q0 = q0;
    A.nq = nq;
    A.dots1 = ws.dots1;
    A.dots2 = ws.dots2;
    A.fold = ws.fold;
    A.ru1 = ix.rowptr ? ws.ru1 : nullptr;
    A.ru2 = ix.rowptr ? ws.ru2 : nullptr;
    A.topP = ws.topP;
    A.plen = ws.topP < ix.T ? ws.plen : nullptr;
    A.retry_list = ws.retry_list;
    A.retry_count = ws.retry_count;
    A.qlist = ws.qlist;
    A.qlist_count = ws.qlist_count;
    A.sr1 = ws.sr1;
    A.sr2 = ws.sr2;
    A.ord1 = ws.ord1;
    A.ord2 = ws.ord2;
    A.pos1 = ws.pos1;
    A.pos2 = ws.pos2;
    A.rowptr = ix.rowptr;
    A.colptr = ix.colptr;
    A.rowcols = ix.rowcols;
    A.colrows = ix.colrows;
    A.L = budget;
    A.k = k;
    A.prof = g_prof_buffer;
    A.out_d = out_dist;
    A.out_ids = out_ids;
    A.out_count = out_count;
    A.out_ncand = out_ncand;
    A.out_popped = out_popped;
    A.counter = ws.counter;
    A.scratch = ws.cta_scratch;
    A.stride = ws.cta_stride;
    // point-term FBPQ with M = 8 / 16: large cells go to big_scan_kernel
    const bool defer = ENGINE == BPQ_ENGINE_FBPQ && rep_fold<MT>() && ix.pterm != nullptr && ws.big_cells != nullptr;
    A.big_cells = defer ? ws.big_cells : nullptr;
    A.big_n = ws.big_n;
    A.big_cap = ws.big_cap;
    A.tk_part = ws.tk_part;
    A.tk_n = ws.tk_n;
    A.ncand_q = ws.ncand_q;
    A.bigq_list = ws.bigq_list;
    A.bigq_count = ws.bigq_count;
    A.big_start = ws.big_start;
    A.record = ENGINE == BPQ_ENGINE_FBPQ ? ws.record : nullptr;
    A.record_n = ws.record_n;
    A.record_cap = ws.record_cap;
}

template <int ENGINE, int MT>
int launch_one(const Index &ix, const float *queries, int64_t q0, int64_t nq, int64_t budget,
               int32_t k, const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids,
               int32_t *out_count, int64_t *out_ncand, int64_t *out_popped, cudaStream_t stream) {
    Args<float, uint32_t> A{};
    fill_args<ENGINE, MT>(A, ix, queries, q0, nq, budget, k, ws, out_dist, out_ids, out_count, out_ncand, out_popped);
    // fold + per-cell LUT (exact FBPQ / generic M) or fold + the sort arrays (point-term FBPQ, whose
    // large cells are streamed by big_scan_kernel), the sort arrays aliasing the LUT
    const bool defer = A.big_cells != nullptr;
    A.tab_floats = ENGINE != BPQ_ENGINE_FBPQ ? ((ix.D + 3) & ~3) + std::max(ix.M * ix.K * 4, kSortBytes) / 4
                   : defer ? ix.M * ix.K + kSortBytes / 4
                           : ix.M * ix.K + std::max(ix.M * ix.K * 4, kSortBytes) / 4;
    A.tab_floats = (A.tab_floats + 3) & ~3;
    A.sr_smem = 0;  // sorted keys are read through L1: only active lines are probed
    A.tkcap = topk_capacity(k);
    A.tk_off = (int)tk_offset(A.tab_floats, A.sr_smem, sizeof(float));
    const size_t smem = dyn_smem_bytes(A.tab_floats, A.sr_smem, sizeof(float), A.tkcap);
    // first pass over a partially sorted sparse table: sparse traversal only
    const bool sparse_only = MT != 0 && ix.rowptr != nullptr && ws.topP < ix.T && ws.qlist == nullptr;
    int n_cta = 0;
    int rc = sparse_only ? configure<ENGINE, MT, float, uint32_t, (MT != 0)>(smem, &n_cta)
                         : configure<ENGINE, MT, float, uint32_t>(smem, &n_cta);
    if (rc) return rc;
    if (n_cta > ws.n_cta) n_cta = ws.n_cta;
    BPQ_CUDA_TRY(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned int), stream));
    if (sparse_only)
        search_kernel<ENGINE, MT, float, uint32_t, (MT != 0)><<<n_cta, NT, smem, stream>>>(A);
    else
        search_kernel<ENGINE, MT, float, uint32_t><<<n_cta, NT, smem, stream>>>(A);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

}  // namespace
}  // namespace bpq
