// Batch database encoding and packing, plus the per-shard top-k merge.
//
// nearest_centroids (quantizer.py:109-130): score = |c|^2 - 2 x.c, argmin
// with ties to the lowest centroid id, d2 = max(score + |x|^2, 0).  FFMA
// tiles (64 rows x 64 centroids per CTA) with the argmin fused into the
// epilogue, so the [n, ncent] score matrix is never materialised.
// encode_residual (multi_index.py:181-189 + quantizer.py:235-247),
// encode_local (hbpq.py:168-200) and pack_cells (multi_index.py:224-230:
// stable sort by cell, counts, exclusive scan, gather) complete
// build_index / build_hbpq_index on the device.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cfloat>

#include "bpq_internal.cuh"

namespace bpq {
namespace {

constexpr int BR = 64, BC = 64, BKD = 16;

__global__ void __launch_bounds__(256) nearest_kernel(const float *__restrict__ X, int64_t n,
                                                      int64_t ldx, int d,
                                                      const float *__restrict__ C,
                                                      const float *__restrict__ cn, int nc,
                                                      int64_t *__restrict__ out_ids,
                                                      float *__restrict__ out_d2,
                                                      uint8_t *__restrict__ out_code,
                                                      int64_t code_stride) {
    __shared__ __align__(16) float Xs[BKD][BR + 4];
    __shared__ __align__(16) float Cs[BKD][BC + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t r0 = (int64_t)blockIdx.x * BR;
    const int lr = threadIdx.x >> 2, lk = (threadIdx.x & 3) * 4;
    float best[4];
    int bidx[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        best[i] = INFINITY;
        bidx[i] = 0x7fffffff;
    }
    for (int c0 = 0; c0 < nc; c0 += BC) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < d; k0 += BKD) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                int kk = k0 + lk + u;
                int64_t r = r0 + lr;
                int c = c0 + lr;
                Xs[lk + u][lr] = (r < n && kk < d) ? __ldg(X + r * ldx + kk) : 0.f;
                Cs[lk + u][lr] = (c < nc && kk < d) ? __ldg(C + (int64_t)c * d + kk) : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BKD; kk++) {
                float4 a = *reinterpret_cast<const float4 *>(&Xs[kk][ty * 4]);
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
        for (int j = 0; j < 4; j++) {
            int c = c0 + tx * 4 + j;
            if (c >= nc) continue;
            float cnv = __ldg(cn + c);
#pragma unroll
            for (int i = 0; i < 4; i++) {
                float s = __fsub_rn(cnv, __fmul_rn(2.f, acc[i][j]));
                if (s < best[i]) {
                    best[i] = s;
                    bidx[i] = c;
                }
            }
        }
    }
    // reduce across the 16 column threads of each row group (same half-warp)
#pragma unroll
    for (int i = 0; i < 4; i++) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            float ob = __shfl_xor_sync(0xffffffffu, best[i], o);
            int oi = __shfl_xor_sync(0xffffffffu, bidx[i], o);
            if (ob < best[i] || (ob == best[i] && oi < bidx[i])) {
                best[i] = ob;
                bidx[i] = oi;
            }
        }
    }
    if (tx == 0) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            int64_t r = r0 + ty * 4 + i;
            if (r >= n) continue;
            int id = bidx[i] == 0x7fffffff ? 0 : bidx[i];
            if (out_ids) out_ids[r] = id;
            if (out_code) out_code[r * code_stride] = (uint8_t)id;
            if (out_d2) {
                const float *x = X + r * ldx;
                float xn = 0.f;
                for (int u = 0; u < d; u++) xn = fmaf(x[u], x[u], xn);
                float v = __fadd_rn(best[i], xn);
                out_d2[r] = v > 0.f ? v : 0.f;
            }
        }
    }
}

__global__ void residual_kernel(const float *__restrict__ X, int64_t n, int dim,
                                const float *__restrict__ c1, const float *__restrict__ c2,
                                const int64_t *__restrict__ ii, const int64_t *__restrict__ jj,
                                float *__restrict__ out) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = n * dim;
    if (idx >= total) return;
    int64_t r = idx / dim;
    int x = (int)(idx - r * dim);
    int dh = dim / 2;
    float c = x < dh ? __ldg(c1 + ii[r] * dh + x) : __ldg(c2 + jj[r] * dh + (x - dh));
    out[idx] = __fsub_rn(X[idx], c);
}

// one warp per (row, part): nearest codeword of the cell-local book
__global__ void local_encode_kernel(const float *__restrict__ X, int64_t n, int dim,
                                    const float *__restrict__ c1, const float *__restrict__ c2,
                                    const int64_t *__restrict__ ii, const int64_t *__restrict__ jj,
                                    const float *__restrict__ bank1,
                                    const float *__restrict__ bank2, int m, int K,
                                    uint8_t *__restrict__ out_codes) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= n * m) return;
    const int64_t r = w / m;
    const int p = (int)(w - r * m);
    const int m2 = m / 2, dh = dim / 2, ds = dim / m;
    const int half = p < m2 ? 0 : 1;
    const int hp = half ? p - m2 : p;
    const int64_t cell = half ? jj[r] : ii[r];
    const float *cc = (half ? c2 : c1) + cell * dh + hp * ds;
    const float *xv = X + r * dim + half * dh + hp * ds;
    const float *book = (half ? bank2 : bank1) + ((cell * m2 + hp) * (int64_t)K) * ds;
    float best = INFINITY;
    int bi = 0x7fffffff;
    for (int c = lane; c < K; c += 32) {
        const float *bk = book + (int64_t)c * ds;
        float dot = 0.f, nn = 0.f;
        for (int u = 0; u < ds; u++) {
            float e = __fsub_rn(__ldg(xv + u), __ldg(cc + u));
            float b = __ldg(bk + u);
            dot = fmaf(e, b, dot);
            nn = fmaf(b, b, nn);
        }
        float s = __fsub_rn(nn, __fmul_rn(2.f, dot));
        if (s < best) {
            best = s;
            bi = c;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) out_codes[r * m + p] = (uint8_t)(bi == 0x7fffffff ? 0 : bi);
}

__global__ void lin_kernel(const int64_t *__restrict__ ii, const int64_t *__restrict__ jj,
                           int64_t n, int t, uint32_t *__restrict__ lin, uint32_t *__restrict__ iota,
                           uint32_t *__restrict__ counts) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    uint32_t l = (uint32_t)(ii[r] * t + jj[r]);
    lin[r] = l;
    iota[r] = (uint32_t)r;
    atomicAdd(counts + l, 1u);
}

__global__ void gather_rows_kernel(const uint32_t *__restrict__ order, int64_t n, uint32_t id_offset,
                                   const uint8_t *__restrict__ codes_in, int m,
                                   uint32_t *__restrict__ out_ids, uint8_t *__restrict__ out_codes) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    uint32_t src = order[r];
    out_ids[r] = id_offset + src;
    for (int p = 0; p < m; p++) out_codes[r * m + p] = codes_in[(int64_t)src * m + p];
}

// per query: G-way merge of sorted per-shard lists by (dist, id)
// (shard s's lists start `stride` / `cstride` elements after shard s - 1's)
__global__ void merge_kernel(const float *__restrict__ dists, const uint32_t *__restrict__ ids,
                             const int32_t *__restrict__ counts, int g, int64_t nq, int k, int64_t stride,
                             int64_t cstride, float *__restrict__ od, uint32_t *__restrict__ oi,
                             int32_t *__restrict__ oc) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    int pos[16];
    int cnt[16];
    int total = 0;
    for (int s = 0; s < g; s++) {
        pos[s] = 0;
        int c = counts[(int64_t)s * cstride + q];
        cnt[s] = c < 0 ? 0 : c;
        total += cnt[s];
    }
    int out = 0;
    for (; out < k && out < total; out++) {
        int bs = -1;
        float bd = 0.f;
        uint32_t bi = 0;
        for (int s = 0; s < g; s++) {
            if (pos[s] >= cnt[s]) continue;
            int64_t at = (int64_t)s * stride + q * k + pos[s];
            float d = dists[at];
            uint32_t id = ids[at];
            if (bs < 0 || d < bd || (d == bd && id < bi)) {
                bs = s;
                bd = d;
                bi = id;
            }
        }
        pos[bs]++;
        od[q * k + out] = bd;
        oi[q * k + out] = bi;
    }
    oc[q] = out;
    for (; out < k; out++) {
        od[q * k + out] = INFINITY;
        oi[q * k + out] = 0xFFFFFFFFu;
    }
}

struct PackLayout {
    size_t lin, lin_sorted, iota, order, counts, offs64, cub, total, cub_bytes;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

PackLayout pack_layout(int64_t n, int32_t t) {
    PackLayout L{};
    int64_t cells = (int64_t)t * t;
    size_t o = 0;
    L.lin = o; o += al(n * 4);
    L.lin_sorted = o; o += al(n * 4);
    L.iota = o; o += al(n * 4);
    L.order = o; o += al(n * 4);
    L.counts = o; o += al((cells + 1) * 4);
    L.offs64 = 0;
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs<uint32_t, uint32_t>(nullptr, a, nullptr, nullptr, nullptr, nullptr, (int)(n > 0 ? n : 1));
    cub::DeviceScan::ExclusiveSum<uint32_t *, uint32_t *>(nullptr, b, nullptr, nullptr, (int)(cells + 1));
    L.cub_bytes = a > b ? a : b;
    L.cub = o; o += al(L.cub_bytes);
    L.total = o;
    return L;
}

}  // namespace
}  // namespace bpq

using bpq::fail;

extern "C" int bpq_nearest_centroids(const float *xs, int64_t n, int64_t ld_x, int32_t d,
                                     const float *cents, const float *cent_norms, int32_t ncent,
                                     int64_t *out_ids, float *out_d2, uint8_t *out_code,
                                     int64_t code_stride, void *stream) {
    BPQ_CHECK(n >= 0 && d >= 1 && ncent >= 1 && ld_x >= d, BPQ_ERR_INVALID, "bad nearest_centroids shape");
    BPQ_CHECK(out_code == nullptr || ncent <= 256, BPQ_ERR_INVALID, "uint8 codes need ncent <= 256");
    if (n == 0) return BPQ_OK;
    unsigned grid = (unsigned)((n + bpq::BR - 1) / bpq::BR);
    bpq::nearest_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(xs, n, ld_x, d, cents, cent_norms,
                                                               ncent, out_ids, out_d2, out_code,
                                                               code_stride);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

extern "C" size_t bpq_coarse_limb_image_bytes(int32_t ncent) {
    return ncent > 0 ? bpq::coarse_limb_image_bytes(ncent) : 0;
}

extern "C" int bpq_coarse_limb_image(const float *cents, int32_t ncent, void *img, void *stream) {
    BPQ_CHECK(ncent >= 1 && cents && img, BPQ_ERR_INVALID, "bad coarse limb image arguments");
    return bpq::launch_coarse_limb_image(cents, ncent, static_cast<uint8_t *>(img), (cudaStream_t)stream);
}

extern "C" int bpq_nearest_centroids_tc(const float *xs, int64_t n, int64_t ld_x, const void *img,
                                        const float *cent_norms, int32_t ncent, int64_t *out_ids, float *out_d2,
                                        uint8_t *out_code, int64_t code_stride, void *stream) {
    BPQ_CHECK(n >= 0 && ncent >= 1 && ld_x >= 64, BPQ_ERR_INVALID, "bad nearest_centroids shape");
    BPQ_CHECK(out_code == nullptr || ncent <= 256, BPQ_ERR_INVALID, "uint8 codes need ncent <= 256");
    return bpq::launch_nearest_tc(xs, n, ld_x, static_cast<const uint8_t *>(img), cent_norms, ncent, out_ids,
                                  out_d2, out_code, code_stride, (cudaStream_t)stream);
}

extern "C" int bpq_encode_residual(const float *xs, int64_t n, int32_t dim, const float *coarse1,
                                   const float *coarse2, const int64_t *i_idx,
                                   const int64_t *j_idx, const float *books,
                                   const float *book_norms, int32_t m, int32_t k,
                                   uint8_t *out_codes, void *workspace, size_t workspace_bytes,
                                   void *stream) {
    BPQ_CHECK(m >= 2 && m % 2 == 0 && m <= 16 && dim % m == 0 && dim % 2 == 0, BPQ_ERR_INVALID,
              "bad fine-codec parameters");
    BPQ_CHECK(workspace_bytes >= (size_t)n * dim * 4, BPQ_ERR_WORKSPACE, "encode workspace too small");
    if (n == 0) return BPQ_OK;
    float *disp = static_cast<float *>(workspace);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t total = n * dim;
    bpq::residual_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(xs, n, dim, coarse1, coarse2,
                                                                        i_idx, j_idx, disp);
    BPQ_CUDA_TRY(cudaGetLastError());
    int ds = dim / m;
    for (int p = 0; p < m; p++) {
        int rc = bpq_nearest_centroids(disp + p * ds, n, dim, ds, books + (int64_t)p * k * ds,
                                       book_norms + (int64_t)p * k, k, nullptr, nullptr,
                                       out_codes + p, m, stream);
        if (rc) return rc;
    }
    return BPQ_OK;
}

extern "C" int bpq_encode_local(const float *xs, int64_t n, int32_t dim, const float *coarse1,
                                const float *coarse2, const int64_t *i_idx, const int64_t *j_idx,
                                const float *bank1, const float *bank2, int32_t m, int32_t k,
                                uint8_t *out_codes, void *stream) {
    BPQ_CHECK(m >= 2 && m % 2 == 0 && m <= 16 && dim % m == 0, BPQ_ERR_INVALID, "bad bank parameters");
    if (n == 0) return BPQ_OK;
    int64_t warps = n * m;
    unsigned grid = (unsigned)((warps * 32 + 255) / 256);
    bpq::local_encode_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        xs, n, dim, coarse1, coarse2, i_idx, j_idx, bank1, bank2, m, k, out_codes);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

extern "C" size_t bpq_pack_workspace_size(int64_t n, int32_t t) {
    return bpq::pack_layout(n, t).total;
}

extern "C" int bpq_pack_cells(const int64_t *i_idx, const int64_t *j_idx, int64_t n, int32_t t,
                              uint32_t id_offset, const uint8_t *codes_in, int32_t m,
                              uint32_t *out_offsets, uint32_t *out_ids, uint8_t *out_codes,
                              void *workspace, size_t workspace_bytes, void *stream) {
    BPQ_CHECK(t >= 1 && t < 65536, BPQ_ERR_UNSUPPORTED, "num_coarse must be < 65536");
    BPQ_CHECK(n >= 0 && n < (int64_t)1 << 31, BPQ_ERR_UNSUPPORTED, "pack handles < 2^31 rows per call");
    BPQ_CHECK(n == 0 || (uint64_t)id_offset + (uint64_t)(n - 1) <= 0xFFFFFFFFull, BPQ_ERR_INVALID,
              "point ids must fit in 32 bits");
    bpq::PackLayout L = bpq::pack_layout(n, t);
    BPQ_CHECK(workspace_bytes >= L.total, BPQ_ERR_WORKSPACE, "pack workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    char *w = static_cast<char *>(workspace);
    uint32_t *lin = reinterpret_cast<uint32_t *>(w + L.lin);
    uint32_t *lin_sorted = reinterpret_cast<uint32_t *>(w + L.lin_sorted);
    uint32_t *iota = reinterpret_cast<uint32_t *>(w + L.iota);
    uint32_t *order = reinterpret_cast<uint32_t *>(w + L.order);
    uint32_t *counts = reinterpret_cast<uint32_t *>(w + L.counts);
    int64_t cells = (int64_t)t * t;
    BPQ_CUDA_TRY(cudaMemsetAsync(counts, 0, (cells + 1) * 4, s));
    if (n > 0) {
        bpq::lin_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(i_idx, j_idx, n, t, lin, iota, counts);
        BPQ_CUDA_TRY(cudaGetLastError());
        int end_bit = 1;
        while (end_bit < 32 && ((uint64_t)1 << end_bit) < (uint64_t)cells) end_bit++;
        size_t cb = L.cub_bytes;
        BPQ_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w + L.cub, cb, lin, lin_sorted, iota, order, (int)n, 0,
                                                     end_bit, s));
    }
    size_t cb = L.cub_bytes;
    BPQ_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w + L.cub, cb, counts, out_offsets, (int)(cells + 1), s));
    if (n > 0) {
        bpq::gather_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(order, n, id_offset, codes_in, m,
                                                                          out_ids, out_codes);
        BPQ_CUDA_TRY(cudaGetLastError());
    }
    return BPQ_OK;
}

extern "C" int bpq_merge_topk(const float *dists, const uint32_t *ids, const int32_t *counts, int32_t g,
                              int64_t nq, int32_t k, float *out_dist, uint32_t *out_ids,
                              int32_t *out_count, void *stream) {
    BPQ_CHECK(g >= 1 && g <= 16 && k >= 1, BPQ_ERR_INVALID, "merge needs 1 <= shards <= 16, k >= 1");
    if (nq == 0) return BPQ_OK;
    bpq::merge_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        dists, ids, counts, g, nq, k, nq * k, nq, out_dist, out_ids, out_count);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}

extern "C" int bpq_merge_topk_packed(const void *packed, int32_t g, int64_t nq, int32_t k, float *out_dist,
                                     uint32_t *out_ids, int32_t *out_count, void *stream) {
    BPQ_CHECK(g >= 1 && g <= 16 && k >= 1, BPQ_ERR_INVALID, "merge needs 1 <= shards <= 16, k >= 1");
    if (nq == 0) return BPQ_OK;
    const int64_t words = 2 * nq * k + nq;  // per shard: dists [nq, k] | ids [nq, k] | counts [nq]
    const uint32_t *w = static_cast<const uint32_t *>(packed);
    bpq::merge_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float *>(w), w + nq * k, reinterpret_cast<const int32_t *>(w + 2 * nq * k), g, nq, k,
        words, words, out_dist, out_ids, out_count);
    BPQ_CUDA_TRY(cudaGetLastError());
    return BPQ_OK;
}
