/*
 * bpq_b200.h -- C ABI of the B200 bilayer-PQ batch query engine.
 *
 * Plain C types only (device pointers are plain pointers, the CUDA stream is
 * passed as void*).  Every entry point returns an int status (BPQ_OK == 0);
 * on failure bpq_last_error() returns a thread-local message.  No C++
 * exception crosses this boundary, no entry point allocates device memory
 * behind the caller's back except bpq_index_create (host-copy mode, and the
 * FBPQ point-term array, see bpq_index_desc.fbpq_exact), and no
 * entry point synchronises the host except where noted.
 *
 * Reference interfaces each group replaces (paths relative to
 * /root/reference/pkg/src/bilayerpq/):
 *   - bpq_search            : the per-query loops search_baseline
 *                             (multi_index.py:358-367), search_fbpq
 *                             (fbpq.py:188-194), search_hbpq (hbpq.py:337-342)
 *                             driven by evalbench.run_engine (evalbench.py:330-354)
 *   - bpq_traverse_cells    : kernels.traverse_cells (kernels/numba_backend.py:11-146)
 *   - bpq_scan_global       : kernels.scan_global (kernels/numba_backend.py:149-180)
 *   - bpq_scan_local        : kernels.scan_local (kernels/numba_backend.py:183-213)
 *   - bpq_scan_tables       : kernels.scan_tables (kernels/numba_backend.py:216-246)
 *   - bpq_nearest_centroids : quantizer.nearest_centroids (quantizer.py:109-130)
 *   - bpq_encode_residual   : multi_index.displacements + quantizer.pq_encode_batch
 *                             (multi_index.py:181-189, quantizer.py:235-247)
 *   - bpq_encode_local      : hbpq.hbpq_encode_batch (hbpq.py:168-200)
 *   - bpq_pack_cells        : the packing tail of multi_index.build_index
 *                             (multi_index.py:224-230)
 *   - bpq_merge_topk        : no reference counterpart (per-shard top-k merge
 *                             after the NCCL all-gather)
 */
#ifndef BPQ_B200_H
#define BPQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BPQ_ABI_VERSION 3

enum {
    BPQ_OK = 0,
    BPQ_ERR_INVALID = 1,     /* bad argument (reference raises ValueError) */
    BPQ_ERR_CUDA = 2,        /* CUDA runtime failure */
    BPQ_ERR_UNSUPPORTED = 3, /* shape outside the engine's compiled range */
    BPQ_ERR_WORKSPACE = 4    /* workspace too small */
};

enum { BPQ_ENGINE_BASELINE = 0, BPQ_ENGINE_FBPQ = 1, BPQ_ENGINE_HBPQ = 2 };

/* Index arrays.  Layout matches the reference containers (multi_index.py:
 * 100-146, fbpq.py:28-66, hbpq.py:42-82) except that cell offsets are
 * uint32 (every config holds < 2^32 entries per table).  In device mode the
 * pointers are device pointers borrowed for the index lifetime; in host mode
 * they are host pointers copied into library-owned device memory. */
typedef struct bpq_index_desc {
    int32_t dim;            /* D */
    int32_t num_coarse;     /* T codewords per half, T < 65536 */
    int32_t num_parts;      /* M, even, 2..16 */
    int32_t codebook_size;  /* K, 1..256 */
    int64_t num_entries;    /* local entries (ids/codes rows) */
    int64_t num_entries_global; /* global_offsets[T*T] (== num_entries unsharded) */
    const float *coarse1, *coarse2;             /* [T, D/2] */
    const float *coarse_norms1, *coarse_norms2; /* [T] einsum('ij,ij->i') */
    const uint32_t *cell_offsets;   /* [T*T+1] local entry ranges */
    const uint32_t *global_offsets; /* [T*T+1] traversal counts; NULL = cell_offsets */
    const uint32_t *ids;            /* [N] */
    const uint8_t *codes;           /* [N, M] */
    const float *fine_books;        /* [M, K, D/M]          baseline + fbpq */
    const float *fine_norms;        /* [M, K]               fbpq */
    const float *cross1, *cross2;   /* [T, M/2, K]          fbpq */
    const float *bank1, *bank2;     /* [T, M/2, K, D/M]     hbpq */
    /* Optional populated-cell lists of the traversal table (global_offsets
     * when sharded): row i's populated columns ascending and column j's
     * populated rows ascending (bpq_build_cell_lists).  With them the
     * traversal enumerates a band segment through the list whenever the
     * line holds fewer populated cells than the segment has cells. */
    const uint32_t *row_ptr, *col_ptr;   /* [T+1] */
    const uint16_t *row_cols, *col_rows; /* [min(N_global, T*T)] capacity */
    /* Optional OPQ rotations (the paper's "optimized" variants): the coarse
     * pair's R [D, D] applied to queries as q @ R (multi_index.py:67-74), and
     * the bank's per-half R1, R2 [D/2, D/2] applied to the query
     * displacements of HBPQ (hbpq.py:328-331).  NULL = none. */
    const float *rotation, *rot1, *rot2;
    /* FBPQ scan arithmetic of bpq_search.  0 (default): the index derives a
     * query-independent point term pt[e] = sum_p 2*cross_h[row][p][code_p]
     * (f64 sum, one rounding; 4 B per entry of library-owned device memory)
     * and scores an entry as ((sum_p fold[p][code_p]) + pt[e]) + cell_base:
     * M shared-memory lookups and one 4 B load instead of M cross-table
     * gathers, within 1e-6 relative of the reference.  1: the reference's
     * exact operation order (numba_backend.py:231-242), bit-identical per
     * candidate given the same query tables.  The stage kernel
     * bpq_scan_tables is always exact.  The flag also governs Multi-D-ADC
     * and HBPQ: 0 scores cells whose GLOBAL entry count is >= 256 through a
     * per-cell residual table (per-part sums, within 1e-6 relative); 1 keeps
     * the reference's single running sum (numba_backend.py:165-176,
     * 198-210) for every candidate. */
    int32_t fbpq_exact;
} bpq_index_desc;

typedef struct bpq_index bpq_index;

const char *bpq_last_error(void);
int bpq_abi_version(void);

/* Synchronises the device when it derives the FBPQ point-term array. */
int bpq_index_create(const bpq_index_desc *desc, int copy_from_host, bpq_index **out);
int bpq_index_destroy(bpq_index *index);

/* Batched search: queries [nq, D] f32 (device).  Outputs [nq, k], each row
 * sorted by (dist asc, id asc) as select_top (multi_index.py:326-339);
 * rows with fewer than k candidates are padded with (+inf, 0xFFFFFFFF) and
 * out_count gives the valid length (reference lists are unpadded,
 * SPEC.md:472).  out_ncand (optional) receives candidates scanned per query.
 * The workspace must hold bpq_search_workspace_size() bytes. */
size_t bpq_search_workspace_size(const bpq_index *index, int engine, int64_t nq, int64_t budget,
                                 int32_t k);
int bpq_search(const bpq_index *index, int engine, const float *queries, int64_t nq,
               int64_t budget, int32_t k, float *out_dist, uint32_t *out_ids,
               int32_t *out_count, int64_t *out_ncand, void *workspace, size_t workspace_bytes,
               void *stream);

/* bpq_search plus measurement hooks: stage_events (optional) is an array of
 * 5 cudaEvent_t recorded on the stream before the first-layer kernel, after
 * it, after the row sort (+ FBPQ fold), after the fused traversal/scan
 * passes and after the large-cell stream kernel (point-term FBPQ, M = 8 /
 * 16; otherwise events 3 and 4 coincide) -- single chunk only; out_popped
 * (optional, [nq]) receives the cells the multi-sequence pops up to the
 * cutoff (empty cells included). */
int bpq_search_ex(const bpq_index *index, int engine, const float *queries, int64_t nq,
                  int64_t budget, int32_t k, float *out_dist, uint32_t *out_ids,
                  int32_t *out_count, int64_t *out_ncand, int64_t *out_popped,
                  void *const *stage_events, void *workspace, size_t workspace_bytes,
                  void *stream);

/* Stage mirrors of the reference kernel backend (device pointers, same
 * argument meaning and layout as kernels/numba_backend.py).  Traversal
 * writes the visited non-empty cells in visit order and their count to
 * *nvis_out (device int64). */
size_t bpq_traverse_workspace_size(int64_t t, int64_t budget, int64_t total_entries);
int bpq_traverse_cells(const double *sorted_r1, const double *sorted_r2, const int32_t *order1,
                       const int32_t *order2, const int64_t *offsets, int64_t t, int64_t budget,
                       int64_t total_entries, int32_t *vis_i, int32_t *vis_j, int64_t *starts,
                       int64_t *ends, int64_t *nvis_out, void *workspace, size_t workspace_bytes,
                       void *stream);
/* cand_start [nvis+1]: exclusive prefix of (ends - starts); outputs [ncand]. */
int bpq_scan_tables(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                    const int64_t *cand_start, int64_t nvis, int64_t ncand, const uint32_t *ids,
                    const uint8_t *codes, int32_t m, int32_t k, float q_norm, const float *qd1,
                    const float *qd2, const float *cn1, const float *cn2, const float *fold,
                    const float *cross1, const float *cross2, uint32_t *out_ids, float *out_d,
                    void *stream);
int bpq_scan_global(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                    const int64_t *cand_start, int64_t nvis, int64_t ncand, const uint32_t *ids,
                    const uint8_t *codes, int32_t m, int32_t k, int32_t ds, const float *e1,
                    const float *e2, const float *books, uint32_t *out_ids, float *out_d,
                    void *stream);
int bpq_scan_local(const int32_t *vis_i, const int32_t *vis_j, const int64_t *starts,
                   const int64_t *cand_start, int64_t nvis, int64_t ncand, const uint32_t *ids,
                   const uint8_t *codes, int32_t m, int32_t k, int32_t ds, const float *e1,
                   const float *e2, const float *books1, const float *books2,
                   uint32_t *out_ids, float *out_d, void *stream);

/* Encoding.  xs rows have stride ld_x floats.  out_ids (int64, optional),
 * out_d2 (optional), out_code (uint8 with row stride code_stride, optional). */
int bpq_nearest_centroids(const float *xs, int64_t n, int64_t ld_x, int32_t d,
                          const float *cents, const float *cent_norms, int32_t ncent,
                          int64_t *out_ids, float *out_d2, uint8_t *out_code,
                          int64_t code_stride, void *stream);
/* Tensor-core nearest_centroids for d = 64 (tcgen05, exact bf16 limbs of x
 * and of the centroids, f32 accumulation in TMEM, argmin fused into the
 * epilogue).  The centroids enter as a pre-swizzled limb image built once by
 * bpq_coarse_limb_image (bpq_coarse_limb_image_bytes(ncent) bytes,
 * caller-owned device memory); outputs as bpq_nearest_centroids. */
size_t bpq_coarse_limb_image_bytes(int32_t ncent);
int bpq_coarse_limb_image(const float *cents, int32_t ncent, void *img, void *stream);
int bpq_nearest_centroids_tc(const float *xs, int64_t n, int64_t ld_x, const void *img,
                             const float *cent_norms, int32_t ncent, int64_t *out_ids, float *out_d2,
                             uint8_t *out_code, int64_t code_stride, void *stream);
/* residual = x - [c1[i]; c2[j]] then per-part nearest fine codeword. The
 * workspace holds n*dim floats (the residuals). */
int bpq_encode_residual(const float *xs, int64_t n, int32_t dim, const float *coarse1,
                        const float *coarse2, const int64_t *i_idx, const int64_t *j_idx,
                        const float *books, const float *book_norms, int32_t m, int32_t k,
                        uint8_t *out_codes, void *workspace, size_t workspace_bytes,
                        void *stream);
/* HBPQ local encoding: per half, per part, nearest codeword of the entry's
 * cell-local book (bank rows i for the first half, j for the second). */
int bpq_encode_local(const float *xs, int64_t n, int32_t dim, const float *coarse1,
                     const float *coarse2, const int64_t *i_idx, const int64_t *j_idx,
                     const float *bank1, const float *bank2, int32_t m, int32_t k,
                     uint8_t *out_codes, void *stream);
size_t bpq_pack_workspace_size(int64_t n, int32_t t);
int bpq_pack_cells(const int64_t *i_idx, const int64_t *j_idx, int64_t n, int32_t t,
                   uint32_t id_offset, const uint8_t *codes_in, int32_t m,
                   uint32_t *out_offsets, uint32_t *out_ids, uint8_t *out_codes,
                   void *workspace, size_t workspace_bytes, void *stream);

/* Build the populated-cell lists of a cell table (device pointers): counts
 * per row/column, exclusive scans, ordered fills.  row_cols / col_rows need
 * capacity for every populated cell (min(entries, t*t) suffices). */
size_t bpq_cell_lists_workspace_size(int32_t t);
int bpq_build_cell_lists(const uint32_t *offsets, int32_t t, uint32_t *row_ptr, uint16_t *row_cols,
                         uint32_t *col_ptr, uint16_t *col_rows, void *workspace,
                         size_t workspace_bytes, void *stream);

/* Diagnostics: device buffer of 10 u64 cycle counters that the fused
 * search kernel fills per phase (prologue, tau search, band bounds,
 * enumeration, scan, LUT scan, top-k compaction, final select, finish,
 * idle, ...) when the library was built with -DBPQ_PHASE_PROF; returns 1 if
 * compiled in, else 0.  The buffer must hold 32 counters.  Every build adds,
 * while a buffer is set, the number of entries the large-cell stream kernel
 * scans to counter 18 (bench.py: that kernel's algorithmic bytes); a library
 * built with -DBPQ_CHECKED (csrc/build_checked.sh) counts the stream kernel's
 * bound violations into counter 19. */
int bpq_debug_set_phase_buffer(unsigned long long *dev_counters);

/* First-layer stage of coarse_scan (multi_index.py:283-288): dots1[q, t] =
 * q[:D/2] . c1[t], dots2[q, t] = q[D/2:] . c2[t] for nq device queries
 * (already rotated if the index has a coarse rotation), on the path the
 * index's searches use: the tcgen05 tensor-core GEMM over exact bf16 limbs
 * when D = 128, else the FFMA kernel.  Outputs are caller-owned f32 [nq, T]. */
int bpq_coarse_dots(const bpq_index *index, const float *queries, int64_t nq, float *dots1, float *dots2,
                    void *stream);

/* out[n, d] = x[n, d] @ R[d, d] (row-vector rotation, quantizer.py:95-96). */
int bpq_rotate(const float *x, int64_t n, int32_t d, const float *R, float *out, void *stream);

/* Merge per-shard top-k lists [g, nq, k] into [nq, k] by (dist, id). */
int bpq_merge_topk(const float *dists, const uint32_t *ids, const int32_t *counts, int32_t g,
                   int64_t nq, int32_t k, float *out_dist, uint32_t *out_ids,
                   int32_t *out_count, void *stream);

/* Query-split sharding (the traversal divided across ranks).
 * Rank r traverses only its query slice against the global cell counts and
 * records every visited non-empty cell instead of scanning it:
 * bpq_search_split_traverse writes visits [nq][cap] as int4
 * (oi * T + oj, global count, cell_base f32 bits, 0) in visit order and
 * visit_count [nq] (0xFFFFFFFF: the query failed); cap >=
 * bpq_split_visit_cap(index, budget).  After the ranks all-gather the
 * packed lists (visit_start [nq + 1] over all queries, rank order), each rank
 * streams its local entries of every query's cells with
 * bpq_search_split_scan (point-term FBPQ, M = 8 / 16), giving per-rank
 * [nq, k] lists for the usual merge.  Workspace: bpq_search_workspace_size
 * for the traversal, bpq_split_scan_workspace_size for the scan. */
int64_t bpq_split_visit_cap(const bpq_index *index, int64_t budget);
int bpq_search_split_traverse(const bpq_index *index, const float *queries, int64_t nq, int64_t budget,
                              uint32_t *visit_count, void *visits, int64_t cap, int64_t *out_ncand,
                              void *workspace, size_t workspace_bytes, void *stream);
size_t bpq_split_scan_workspace_size(const bpq_index *index, int64_t nq, int64_t total_visits);
int bpq_search_split_scan(const bpq_index *index, const float *queries, int64_t nq, int32_t k,
                          const void *visits, const uint32_t *visit_start, int64_t total_visits,
                          float *out_dist, uint32_t *out_ids, int32_t *out_count, void *workspace,
                          size_t workspace_bytes, void *stream);

/* The same merge over the packed buffer of one all-gather: shard s occupies
 * words [s * W, (s + 1) * W), W = 2 * nq * k + nq, laid out as dists f32
 * [nq, k] | ids u32 [nq, k] | counts i32 [nq]. */
int bpq_merge_topk_packed(const void *packed, int32_t g, int64_t nq, int32_t k, float *out_dist,
                          uint32_t *out_ids, int32_t *out_count, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BPQ_B200_H */
