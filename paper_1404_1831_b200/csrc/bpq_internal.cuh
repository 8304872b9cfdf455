// Internal definitions shared by the engine's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "bpq_b200.h"

namespace bpq {

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define BPQ_CUDA_TRY(expr)                                                                   \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return ::bpq::fail(BPQ_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define BPQ_CHECK(cond, code, msg)                                                           \
    do {                                                                                     \
        if (!(cond)) return ::bpq::fail((code), (msg));                                      \
    } while (0)

// Tunables of the fused traversal + scan + top-k kernel.
constexpr int kSearchThreads = 256;     // threads per CTA (one CTA per query at a time)
constexpr int kLutUnroll = 4;           // codes per thread per round in the LUT scan
constexpr int kMaxK = 1024;             // largest k the engine accepts
constexpr int kSortCap = 512;           // final-band cells sorted in shared memory
constexpr int kTopP = 1024;             // sorted prefix per half for sparse-table queries
constexpr int kMultiLines = 8;          // lines a warp evaluates per threshold in a multi-probe round
#ifndef BPQ_LUT_MIN
#define BPQ_LUT_MIN 256
#endif
constexpr int kLutMin = BPQ_LUT_MIN;    // cells with >= this many entries are scanned via a smem LUT
constexpr int kBandCap = 32768;         // max cells enumerated per band
constexpr int kMaxDim = 1024;           // queries staged in shared memory
constexpr int kStreamPad = 256;         // entries of slack after the rotated codes / point terms (masked chunk over-reads)

struct Index {
    int32_t D, T, M, K, dh, ds;
    int64_t N;
    int64_t N_global;
    const float *c1, *c2, *cn1, *cn2;
    const uint32_t *loff, *goff;
    const uint32_t *ids;
    const uint8_t *codes;
    const float *books, *fine_norms, *cross1, *cross2, *bank1, *bank2;
    const float *rot, *rot1, *rot2;  // optional rotations (see bpq_index_desc)
    const float *pterm;  // FBPQ per-entry cross term [N] (null: exact reference-order scan)
    const uint8_t *codes_rot;  // point-term FBPQ, M = 8 / 16: entry e's code bytes rotated by e % M
    // bf16 limb images of the coarse books for the tensor-core first layer (tc_dots.cu; null: FFMA)
    const uint8_t *cimg1, *cimg2;
    bool exact;          // bpq_index_desc.fbpq_exact: reference operation order, all engines
    // populated-cell lists (optional): row i -> columns j, column j -> rows i
    const uint32_t *rowptr, *colptr;
    const uint16_t *rowcols, *colrows;
    int64_t populated;  // populated cells of the traversal table (row_ptr[T]; 0: unknown)
    std::vector<void *> owned;
};

// ---- launchers implemented in the .cu files --------------------------------
int launch_point_term(const uint32_t *offsets, int32_t t, int32_t m, int32_t k, const uint8_t *codes,
                      const float *cross1, const float *cross2, float *pt, cudaStream_t s);
int launch_rotate_codes(const uint8_t *codes, int64_t n, int32_t m, uint8_t *out, cudaStream_t s);
int launch_coarse_dots(const float *queries, int64_t nq, int32_t D, const float *c1,
                       const float *c2, int32_t T, float *dots1, float *dots2,
                       cudaStream_t stream);
size_t coarse_limb_image_bytes(int32_t T);
int launch_coarse_limb_image(const float *C, int32_t T, uint8_t *img, cudaStream_t s);
int launch_nearest_tc(const float *xs, int64_t n, int64_t ld_x, const uint8_t *img, const float *cn, int32_t nc,
                      int64_t *out_ids, float *out_d2, uint8_t *out_code, int64_t code_stride, cudaStream_t s);
int launch_coarse_dots_tc(const float *queries, int64_t nq, int32_t D, const uint8_t *img1, const uint8_t *img2,
                          int32_t T, float *dots1, float *dots2, cudaStream_t s);
int launch_fold(const float *queries, int64_t nq, int32_t D, int32_t M, int32_t K, const float *books,
                const float *fine_norms, float *fold, cudaStream_t stream);
int launch_row_sort(const float *queries, int64_t nq, int32_t D, const float *dots1,
                    const float *dots2, const float *cn1, const float *cn2, int32_t T,
                    float *sr1, float *sr2, int32_t *ord1, int32_t *ord2, int32_t *pos1,
                    int32_t *pos2, float *ru1, float *ru2, const unsigned int *qlist,
                    const unsigned int *qcount, cudaStream_t stream);
int launch_row_topk(const float *queries, int64_t nq, int32_t D, const float *dots1,
                    const float *dots2, const float *cn1, const float *cn2, int32_t T, float *sr1,
                    float *sr2, int32_t *ord1, int32_t *ord2, float *ru1, float *ru2, int32_t *plen,
                    cudaStream_t stream);

struct SearchWorkspace {
    float *dots1, *dots2, *sr1, *sr2, *fold, *ru1, *ru2, *qrot;
    int32_t *ord1, *ord2, *pos1, *pos2;
    unsigned int *retry_list, *retry_count;
    int topP;                      // sorted prefix length in sr/ord for this launch (full: T)
    int32_t *plen;                 // per (query, half) prefix length of the partial sort
    const unsigned int *qlist, *qlist_count;  // indirect query list (retry pass)
    unsigned int *counter;
    // large cells deferred by the traversal kernel to the stream kernel (point-term FBPQ, M = 8 / 16)
    int4 *big_cells;               // [chunk][big_cap]
    uint32_t *big_n, *tk_n;        // [chunk]
    int big_cap;
    unsigned long long *tk_part;   // [chunk][k]
    unsigned long long *ncand_q;   // [chunk]
    unsigned int *bigq_list, *bigq_count;
    const uint32_t *big_start;     // split scan: packed per-query cell ranges [nq + 1] (else null)
    int4 *record;                  // record mode (query-split traversal): [nq][record_cap] visited cells
    uint32_t *record_n;
    int record_cap;
    char *cta_scratch;
    size_t cta_stride;
    int n_cta;
};

size_t search_cta_scratch_bytes(int32_t T, int32_t D);
int launch_rotate(const float *x, int64_t n, int32_t d, const float *R, float *out, cudaStream_t stream);
int search_grid_ctas(int engine, int M);
int effective_lut_min();
int launch_visits_to_cells(const int4 *visits, const uint32_t *visit_start, int64_t nq, const uint32_t *loff,
                           int4 *cells, uint32_t *cell_n, unsigned long long *ncand, uint32_t *tk_n,
                           unsigned int *qlist, unsigned int *qcount, cudaStream_t s);
int launch_big_scan(const Index &ix, int engine, const float *queries, int64_t q0, int64_t nq, int64_t budget,
                    int32_t k, const SearchWorkspace &ws, float *out_dist, uint32_t *out_ids, int32_t *out_count,
                    cudaStream_t stream);
int launch_search(const Index &ix, int engine, const float *queries, int64_t q0, int64_t nq,
                  int64_t budget, int32_t k, const SearchWorkspace &ws, float *out_dist,
                  uint32_t *out_ids, int32_t *out_count, int64_t *out_ncand,
                  int64_t *out_popped, cudaStream_t stream);
int launch_traverse_stage(const double *sr1, const double *sr2, const int32_t *o1,
                          const int32_t *o2, const int64_t *offsets, int64_t t, int64_t budget,
                          int64_t total, int32_t *vis_i, int32_t *vis_j, int64_t *starts,
                          int64_t *ends, int64_t *nvis_out, void *ws, size_t ws_bytes,
                          cudaStream_t stream);
size_t traverse_stage_ws_bytes(int64_t t, int64_t budget, int64_t total);

}  // namespace bpq

struct bpq_index {
    bpq::Index ix;
};
